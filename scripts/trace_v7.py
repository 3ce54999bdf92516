"""Print the v7 attention event trace.

Build with LF_NVCC_FLAGS=-DLF_V7_TRACE, run with LF_ATTN_DEBUG=2 (optionally
LF_ATTN_TRACE_CTA=<cta>); the library writes gpurun_out/attn_trace.txt.
Layout: see the LF_T7 comment in paper_2602_04789_b200/csrc/attn_sm100_v7.cuh.
"""
import sys

t = [int(x) for x in open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/attn_trace.txt")]
vals = [x for x in t[:1536 + 128] if x > 0]
base = min(vals)
r = lambda x: x - base if x > 0 else None
print("softmax per set: k | wait S ready stats P0 P1 | durations: S-wait, stats, exp+P")
for X in range(2):
    prev_end = None
    gaps = []
    for k in range(60):
        e = [t[X * 512 + k * 8 + i] for i in range(5)]
        if not e[1]:
            break
        w, s, st, p0, p1 = e
        gaps.append((s - w, st - s, p1 - st))
        if k < 12:
            print(X, k, [r(y) for y in e], (s - w, st - s, p1 - st))
    if gaps:
        n = len(gaps)
        print(f"set {X}: {n} tiles, mean S-wait {sum(g[0] for g in gaps) / n:.0f}, "
              f"stats {sum(g[1] for g in gaps) / n:.0f}, exp+P {sum(g[2] for g in gaps) / n:.0f} clk")
print("MMA per key tile: kit | QK issued, PV wait start, PV issued, K wait start, K ready")
qk = []
for kit in range(120):
    e = [t[1024 + kit * 4 + i] for i in range(4)] + [t[3072 + kit]]
    if not e[0]:
        break
    qk.append(e[0])
    if kit < 16:
        print(kit, [r(x) for x in e])
if len(qk) > 2:
    d = [b - a for a, b in zip(qk, qk[1:])]
    print(f"QK issue interval: mean {sum(d) / len(d):.0f} clk over {len(d)} (ideal 1024 per tile at peak)")
print("items: Q issue, MMA start, set0 tail/O ready/done, set1 tail/O ready/done")
for n in range(16):
    e = [t[1536 + n * 8 + i] for i in range(8)]
    if any(e):
        print(n, [r(x) for x in e])
