"""Print the v5 attention event trace (LF_ATTN_DEBUG=2 writes gpurun_out/attn_trace.txt)."""
import sys
t = [int(x) for x in open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/attn_trace.txt")]
base = min(x for x in t if x > 0)
r = lambda x: x - base if x > 0 else None
print("tile | X: wait S ldS max Ph0 Ph1 | MMA: X P0seen issued")
for k in range(44):
    row = []
    for X in range(2):
        row.append([r(t[X * 512 + k * 8 + i]) for i in range(6)])
    m = [r(t[1024 + k * 4 + i]) for i in range(4)]
    print(k, row[0], row[1], m)
for X in range(2):
    for u in range(4):
        print("unit", u, "X", X, "epilogue (start, O ready, done):", [r(t[X * 512 + 400 + u * 4 + i]) for i in range(3)])
# per-CTA start/end (globaltimer ns)
st = [t[1536 + 2 * b] for b in range(148)]
en = [t[1537 + 2 * b] for b in range(148)]
if all(st):
    g0 = min(st)
    d = sorted(((en[b] - g0) / 1e3, b, (st[b] - g0) / 1e3) for b in range(148))
    print("CTA end times (us): min", d[0], "median", d[74], "max", d[-1])
    print("slowest 10:", [(round(x, 1), b) for x, b, _ in d[-10:]])
if t[1840] and t[1841]:
    b = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    dur_ns = t[1537 + 2 * b] - t[1536 + 2 * b]
    print("traced CTA clk span", t[1841] - t[1840], "ns", dur_ns, "-> GHz", (t[1841] - t[1840]) / dur_ns)
    print("first event after kernel start (clk)", base - t[1840], " kernel end after last event", t[1841] - max(x for x in t[:1536] if x > 0))
for X in range(2):
    for u in range(4):
        v = [t[X * 512 + 460 + u * 4 + i] for i in range(4)]
        if any(v):
            print("unit", u, "X", X, "split (partial written, counter done, merge done, last?):", [r(x) for x in v[:3]], v[3])
for X in range(2):
    v = [t[X * 512 + 480 + i] for i in range(11)]
    if v[0]:
        print("merge X", X, "deltas:", [v[i] - v[0] if v[i] else None for i in range(11)])
