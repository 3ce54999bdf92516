"""One rollout step's query pooling at c2 (12 heads, 3 x 1560 rows, d 128) between
cudaProfilerStart/Stop, for `ncu --profile-from-start off` (profiling aid).

    ncu --profile-from-start off --set full -k regex:pool_frames_tma -o x python scripts/ncu_qpool.py
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_04789_b200 as lf  # noqa: E402
from paper_2602_04789_b200 import device as D  # noqa: E402
from paper_2602_04789_b200.selection import tilings  # noqa: E402

H, f, n, d, i = 12, 3, 1560, 128, 7
lay = lf.ChunkLayout(f=f, n=n, b_q=64, b_kv=64, d=d, N=7)
q = torch.randn((H, f * n, d), device="cuda").to(torch.bfloat16)
qt, _ = tilings(lay, i, True)
for _ in range(3):
    D.pool_blocks(q, qt)
torch.cuda.synchronize()
torch.cuda.profiler.start()
D.pool_blocks(q, qt)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("ok")
