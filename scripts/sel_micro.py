"""Selection-kernel micro timing: D.select alone (CUDA events, 200 launches) on
synthetic N(0,1)/8 summaries at the bench shapes, for 1..12 heads; with and
without the exact option.  Prints us per launch."""
import sys
import numpy as np
import torch
from paper_2602_04789_b200 import device as D, _lib as L

dev = torch.device("cuda")


def run(H, chunk, s_i, topk=6, f=3, bpf=25, d=128, exact=0, reps=200):
    nqb = f * bpf
    P = (chunk - 1) * f
    g = torch.Generator(device=dev).manual_seed(0)
    qb = torch.randn((H, nqb, d), device=dev, generator=g) * 0.125
    kb = torch.randn((H, chunk * f * bpf, d), device=dev, generator=g) * 0.125
    kf = torch.randn((H, max(P, 1), d), device=dev, generator=g) * 0.05
    st = torch.tensor([float(s_i)], dtype=torch.float64, device=dev)
    D.select_fallbacks(reset=True)
    with L.option("select_exact", exact):
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            for _ in range(3):
                D.select(qb, kb, kf, bpf, chunk, f, topk, False, st)
        torch.cuda.current_stream().wait_stream(s)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            for _ in range(20):
                D.select(qb, kb, kf, bpf, chunk, f, topk, False, st)
        graph.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps // 20):
            graph.replay()
        e1.record()
        torch.cuda.synchronize()
    fb = D.select_fallbacks(reset=True)
    nl = reps // 20 * 20 + 24
    print(f"   (undecided per launch over {H * nqb} lists: frames {fb[0] / nl:.2f} "
          f"({fb[2] / nl:.2f} partial), blocks {fb[1] / nl:.2f} ({fb[3] / nl:.2f} partial))")
    return e0.elapsed_time(e1) / (reps // 20 * 20) * 1e3


if len(sys.argv) > 1 and sys.argv[1] != "plan":  # one case, a few plain launches (for ncu): name H
    cfg = {"c2": (7, 6 / 7), "c5_s70": (7, 0.7), "c3": (14, 0.9046)}[sys.argv[1]]
    H = int(sys.argv[2])
    nqb, P = 75, (cfg[0] - 1) * 3
    qb = torch.randn((H, nqb, 128), device=dev) * 0.125
    kb = torch.randn((H, cfg[0] * 75, 128), device=dev) * 0.125
    kf = torch.randn((H, P, 128), device=dev) * 0.05
    for _ in range(3):
        D.select(qb, kb, kf, 25, cfg[0], 3, 6, False, cfg[1])
    torch.cuda.synchronize()
    sys.exit(0)

for chunk, s_i, name in [] if len(sys.argv) > 1 else [(7, 6 / 7, "c2"), (7, 0.7, "c5_s70"), (14, 0.9046, "c3")]:
    for H in (1, 4, 12):
        print(name, "H", H, "screened %.1f us" % run(H, chunk, s_i), "exact %.1f us" % run(H, chunk, s_i, exact=1))


def graph_time(fn, reps=200):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(3):
            fn()
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(20):
            fn()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps // 20):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / (reps // 20 * 20) * 1e3


def plan_pair(chunk, s_i, H=12, f=3, n=1560, d=128, topk=6):
    """pairing and plan-kernel times on the selections of random summaries"""
    qt = D.TilingSpec(f * n, n, 64)
    kt = D.TilingSpec(chunk * f * n, n, 64)
    bpf = -(-n // 64)
    P = (chunk - 1) * f
    qb = torch.randn((H, qt.count, d), device=dev) * 0.125
    kb = torch.randn((H, kt.count, d), device=dev) * 0.125
    kf = torch.randn((H, P, d), device=dev) * 0.05
    sel = D.select(qb, kb, kf, bpf, chunk, f, topk, False, s_i)
    lb = P * bpf
    qperm = D.pair_qblocks(sel.blocks, sel.count, lb)
    tp = graph_time(lambda: D.pair_qblocks(sel.blocks, sel.count, lb))
    out = {"pair": tp}
    for mode in (0, 1, 2):
        with D.qtile_scope(mode):
            out[f"plan{mode}"] = graph_time(
                lambda: D.plan_tiles(sel.blocks, sel.count, qt, kt, lb,
                                     qperm=qperm if mode == 2 else None))
    return out


if len(sys.argv) == 1 or sys.argv[1] == "plan":
    for chunk, s_i, name in [(7, 0.5, "c5_s50"), (7, 0.7, "c5_s70"), (14, 0.9046, "c3")]:
        print(name, {k: round(v, 1) for k, v in plan_pair(chunk, s_i).items()}, "us")
