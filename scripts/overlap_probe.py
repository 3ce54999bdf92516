"""Where the rollout step's time goes at one config (GPU): graph-timed
(A) attention only, (B) prepare + attend serial on one stream, (C) the bench's
overlapped flow (prepare of call s+1 on a side stream while call s attends).

    python scripts/overlap_probe.py [config]
"""
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2602_04789_b200 as lf  # noqa: E402
from oracle import lf_oracle as O  # noqa: E402
from paper_2602_04789_b200.rollout import HsaRollout  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
c = bench.CONFIGS[name]
H, d, n, f, i, T = c["heads"], c["d"], c["n"], c["f"], c["chunk"], 4
lay = lf.ChunkLayout(f=f, n=n, b_q=64, b_kv=64, d=d, N=c["N"])
plan = lf.allocate(c["plan"][0], c["plan"][1], c["N"], 4, lay) if c["plan"] else None
s_host = float(plan.s[i - 1]) if plan else c["s"]
cfg = lf.SelectionConfig(topk_frames=c["topk"])
dev = torch.device("cuda")
lq = f * n
ro = HsaRollout(lay, H, plan, cfg, framewise=True)
for t in range(1, i):
    q, k, v = O.synthetic_qkv(t, lq, lq, d, heads=H)
    ro.commit(*(torch.from_numpy(a).to(dev, torch.bfloat16) for a in (k, v)), t)
Q = [torch.randn(H, lq, d, device=dev).to(torch.bfloat16) for _ in range(T)]
ro.kv_slot(i)[0].copy_(torch.randn(H, lq, d, device=dev).to(torch.bfloat16))
ro.kv_slot(i)[1].copy_(torch.randn(H, lq, d, device=dev).to(torch.bfloat16))
s_dev = torch.tensor([s_host], dtype=torch.float64, device=dev)
outs = [torch.empty(H, lq, d, dtype=torch.bfloat16, device=dev) for _ in range(T)]
plans = [ro.prepare(Q[s], i, s_i=s_dev, s_host=s_host) for s in range(T)]
side = torch.cuda.Stream()
evs = [torch.cuda.Event() for _ in range(T)]


def attn_only():
    for s in range(T):
        ro.attend(plans[s], out=outs[s])


def serial():
    for s in range(T):
        p = ro.prepare(Q[s], i, s_i=s_dev, s_host=s_host)
        ro.attend(p, out=outs[s])


def prep_only():
    for s in range(T):
        ro.prepare(Q[s], i, s_i=s_dev, s_host=s_host)


def overlapped():
    main = torch.cuda.current_stream()
    side.wait_stream(main)
    pl = [None] * T

    def prep(s):
        with torch.cuda.stream(side):
            pl[s] = ro.prepare(Q[s], i, s_i=s_dev, s_host=s_host)
            evs[s].record(side)
    prep(0)
    for s in range(T):
        if s + 1 < T:
            prep(s + 1)
        main.wait_event(evs[s])
        ro.attend(pl[s], out=outs[s])
    main.wait_stream(side)


def commit_only():
    ro.commit(None, None, i - 1, overwrite=True)


for nm, fn in (("attention x4", attn_only), ("prepare x4", prep_only), ("serial x4", serial),
               ("overlapped x4", overlapped), ("commit", commit_only)):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    print(f"{name} {nm}: {e0.elapsed_time(e1) / 50 * 1e3:.1f} us")
