import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2602_04789_b200 as lf
from oracle import lf_oracle as O
for lq, lk, d in [(128, 128, 64), (128, 512, 64), (256, 1024, 128), (700, 3000, 128)]:
    q, k, v = O.synthetic_qkv(1, lq, lk, d)
    ref = O.dense_attention(q[0], k[0], v[0])
    for sp in ("1", "2", "3", "4"):
        os.environ["LF_ATTN_SPLIT"] = sp
        out = lf.dense_attention(q[0], k[0], v[0])
        rel = np.linalg.norm(out - ref) / np.linalg.norm(ref)
        print(lq, lk, d, "split", sp, "rel", f"{rel:.3e}", flush=True)
