"""Do kernels launched on another stream while the persistent attention kernel
runs get SM resources?  Attention (dense, c2-sized) on stream A; on stream B a
spin of ~30 us then (a) a trivial fill, (b) the selection kernel.  Prints the
device timeline (torch.profiler / CUPTI)."""
import sys
import torch
from torch.profiler import ProfilerActivity, profile
from paper_2602_04789_b200 import device as D

dev = torch.device("cuda")
H, n, f, d = 12, 1560, 3, 128
L = 7 * f * n
lq = f * n
q = torch.randn((H, lq, d), device=dev, dtype=torch.bfloat16)
k = torch.randn((H, L, d), device=dev, dtype=torch.bfloat16)
v = torch.randn((H, L, d), device=dev, dtype=torch.bfloat16)
qt = D.TilingSpec(lq, n, 64)
qb = torch.randn((H, 75, d), device=dev) * 0.125
kb = torch.randn((H, 525, d), device=dev) * 0.125
kf = torch.randn((H, 18, d), device=dev) * 0.05
A, B = torch.cuda.Stream(), torch.cuda.Stream()
buf = torch.empty(1 << 20, device=dev)


def run(kind):
    with torch.cuda.stream(A):
        D.attention(q, k, v, qt, None, 0, L, out_dtype=torch.bfloat16)
    with torch.cuda.stream(B):
        torch.cuda._sleep(60000)  # ~30 us on one SM
        if kind == "fill":
            buf.fill_(1.0)
        else:
            D.select(qb, kb, kf, 25, 7, 3, 6, False, 0.7)
    torch.cuda.synchronize()


for kind in ("fill", "select"):
    run(kind)
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        run(kind)
    evs = sorted((e.time_range.start, e.time_range.end, e.name[:50]) for e in prof.events()
                 if e.device_type.name == "CUDA")
    t0 = evs[0][0]
    print(kind)
    for s, e_, nm in evs:
        print(f"  {s - t0:8.1f} {e_ - t0:8.1f}  {nm}")
