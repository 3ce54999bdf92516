#!/usr/bin/env python
"""Benchmark of the Light Forcing sparse-attention hot path on B200.

One *step* = one chunk of one layer, all heads.  Headline (`value`): the
rollout driver (HsaRollout) -- commit of the previous clean chunk (its key
summaries pooled once) + the T = 4 denoising-step calls of chunk i (pool Q ->
hierarchical selection -> tile plan -> tcgen05 block-sparse attention) over a
device KV cache of i chunks.  `stateless`: the same T calls through the
per-call pipeline (lf_hsa_forward, the reference's hsa_attention contract),
which re-pools the whole key context every call.  Inputs are synthetic bf16
N(0,1) (seeded); the CAG plan is solved on device and s_i is read from device
memory by the selection kernel.

    python bench.py [--gpus N --steps K --warmup W] [--config c2] [--impl reference]

LF_BENCH_TRACE=1 prints the per-iteration device times of the timed legs to
stderr (diagnosing outliers, e.g. of the PCIe-bound e2e leg).
LF_BENCH_TIMELINE=path writes the device timeline (kernel intervals per
stream) of three headline replays, and of one eager chunk, as CSV.

Multi-GPU (torchrun, one rank per GPU): heads are sharded when H % N == 0 and
the per-head outputs are all-gathered over NCCL (strong scaling); otherwise
every rank runs an independent video (replicas, weak scaling, no collective).
Prints ONE JSON line on rank 0.
"""

from __future__ import annotations

import argparse
import gc
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")

METRIC = "sparse-attn ms/chunk & effective TFLOPS (1.3B 480p) at 1/2/4/8 B200 vs CPU ref"
UNIT = "effective TFLOP/s"

CONFIGS = {
    # BASELINE.json configs[1]: Self-Forcing 1.3B 480p, chunk 7 of a 7-chunk rollout, CAG plan
    "c2": dict(heads=12, d=128, n=1560, f=3, N=7, chunk=7, plan=(0.9, 0.98), s=None, topk=6,
               mode="global", T=4),
    # configs[2]: long rollout, chunk 14 of 21 (42 frames of KV), CAG plan -> past blocks selected
    "c3": dict(heads=12, d=128, n=1560, f=3, N=21, chunk=14, plan=(0.9, 0.98), s=None, topk=6,
               mode="global", T=4),
    # load-balance probes (diagnostics): 8 / 16 heads = exactly 1 / 2 work items per CTA
    "c2h8": dict(heads=8, d=128, n=1560, f=3, N=7, chunk=7, plan=(0.9, 0.98), s=None, topk=6,
                 mode="global", T=4),
    "c2h16": dict(heads=16, d=128, n=1560, f=3, N=7, chunk=7, plan=(0.9, 0.98), s=None, topk=6,
                  mode="global", T=4),
    # configs[3]: Wan-14B attention shape (40 heads)
    "c4": dict(heads=40, d=128, n=1560, f=3, N=7, chunk=7, plan=(0.9, 0.98), s=None, topk=6,
               mode="global", T=4),
    # configs[4] sweep points: fixed sparsity s at chunk 7 (0.0 = dense through the same kernel)
    "c5_s50": dict(heads=12, d=128, n=1560, f=3, N=7, chunk=7, plan=None, s=0.5, topk=6,
                   mode="global", T=4),
    "c5_s70": dict(heads=12, d=128, n=1560, f=3, N=7, chunk=7, plan=None, s=0.7, topk=6,
                   mode="global", T=4),
    "c5_s85": dict(heads=12, d=128, n=1560, f=3, N=7, chunk=7, plan=None, s=0.85, topk=6,
                   mode="global", T=4),
    "c5_dense": dict(heads=12, d=128, n=1560, f=3, N=7, chunk=7, plan=None, s=0.0, topk=18,
                     mode="global", T=4),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--profile-launch", action="store_true",
                    help="run 2 eager steps only (for ncu launch lists)")
    return ap.parse_args()


# ---------------------------------------------------------------------------- helpers


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms in the background."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits", "-lms",
                 "50", "-i", str(self.index)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
                text=True)
        except OSError:
            return self
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 9:
                self.rows.append(parts)

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        return self.summary()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[5 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def cpu_desc():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def make_layout(lf, c):
    return lf.ChunkLayout(f=c["f"], n=c["n"], b_q=64, b_kv=64, d=c["d"], N=c["N"])


def host_s(lf, c, lay):
    """s_i for the config (host value, for the CPU legs)."""
    if c["plan"] is None:
        return float(c["s"])
    from oracle import lf_oracle as O
    p = O.allocate(c["plan"][0], c["plan"][1], c["N"], c["T"], c["f"], c["n"], 64, c["d"])
    return p.s[c["chunk"] - 1]


def job_config(args, c, s_i, world):
    """The workload's config dict, identical in both arms (ours / --impl reference)."""
    from paper_2602_04789_b200.sharding import partition_heads
    H, d, n, f, i, T = c["heads"], c["d"], c["n"], c["f"], c["chunk"], c["T"]
    lk = i * f * n
    return {"workload": f"{args.config}: {H} heads x d{d}, n={n} tokens/frame (framewise "
                        f"b=64), f={f}, chunk {i} of {c['N']}, T={T} calls/step",
            "heads": H, "d": d, "n": n, "f": f, "chunk": i, "N": c["N"], "T": T,
            "plan": list(c["plan"]) if c["plan"] else None, "s_i": s_i,
            "topk_frames": c["topk"], "mode": c["mode"],
            "parallelism": partition_heads(H, world, 0).mode,
            "l2": f"inputs larger than L2 (K+V per call {2 * H * lk * d * 2 / 1e6:.0f} MB "
                  f"over all heads)"}


# ---------------------------------------------------------------------------- CPU legs


def oracle_sample(c, s_i, seed, threads):
    """Time the CPU oracle (framewise port of chunkattn.hsa_attention) on one head."""
    import numpy as np
    from oracle import lf_oracle as O
    i, f, n, d = c["chunk"], c["f"], c["n"], c["d"]
    q, k, v = O.synthetic_qkv(seed, f * n, i * f * n, d)
    t0 = time.perf_counter()
    out, sel, _ = O.hsa_attention(q[0], k[0], v[0], i, s_i, f, n, 64, 64, c["topk"], c["mode"],
                                  framewise=True, threads=threads)
    dt = time.perf_counter() - t0
    flops = O.effective_flops(sel.bits, O.q_tiling(f, n, 64, True), O.k_tiling(i, f, n, 64, True), d)
    assert np.isfinite(out).all()
    return dt, flops


def ref_aligned_sample(c, s_i, seed, threads):
    """Time the REAL reference (chunkattn.hsa_attention, staged unmodified in
    oracle/_ref) on one head at the aligned n = 1536 form of the workload (the
    reference rejects n = 1560, selection.py:88-92).  None if not staged."""
    import numpy as np
    from oracle import lf_oracle as O
    from oracle.make_ref import import_reference
    try:
        R = import_reference()
    except ImportError:
        return None
    i, f, d = c["chunk"], c["f"], c["d"]
    n = c["n"] - c["n"] % 64
    lay = R.ChunkLayout(f=f, n=n, b_q=64, b_kv=64, d=d, N=c["N"])
    cfg = R.SelectionConfig(topk_frames=c["topk"], block_budget_mode=c["mode"])
    q, k, v = O.synthetic_qkv(seed, f * n, i * f * n, d)
    t0 = time.perf_counter()
    out, st, _ = R.hsa_attention(q[0], k[0], v[0], i, s_i, cfg, lay, threads=threads)
    dt = time.perf_counter() - t0
    assert np.isfinite(out).all()
    return dt, 2 * st.flop_estimate, n  # aligned 64x64 tiles: effective = 2 x MAC count


def run_reference(args, c):
    """The reference arm: the reference's own CPU implementation of the path on
    this box's host cores -- the unmodified chunkattn.hsa_attention staged in
    oracle/_ref, at the aligned n = 1536 form of the workload (it rejects
    n = 1560, selection.py:88-92), one head-call per step, all host threads;
    the framewise oracle port at the workload's own n is timed beside it.
    Without a staged reference the port is the arm's value."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    import paper_2602_04789_b200 as lf  # layout helper only (no GPU use)
    lay = make_layout(lf, c)
    s_i = host_s(lf, c, lay)
    threads = os.cpu_count() or 1
    real = ref_aligned_sample(c, s_i, 99, threads) is not None  # also the first warm-up
    for w in range(args.warmup):
        if real:
            ref_aligned_sample(c, s_i, 100 + w, threads)
        else:
            oracle_sample(c, s_i, 100 + w, threads)
    times, flops = [], []
    for st in range(args.steps):
        if real:
            dt, fl, n_al = ref_aligned_sample(c, s_i, 1000 + st, threads)
        else:
            dt, fl = oracle_sample(c, s_i, 1000 + st, threads)
        times.append(dt)
        flops.append(fl)
    value = sum(flops) / sum(times) / 1e12
    ms_chunk = statistics.mean(times) * c["heads"] * c["T"] * 1e3
    if real:
        kind = "reference"
        sample = (f"1 head of 1 denoising-step call of chunk {c['chunk']} per step through the "
                  f"unmodified chunkattn.hsa_attention (oracle/_ref) at the aligned n={n_al} "
                  f"(the reference rejects n={c['n']}), OPENBLAS_NUM_THREADS=1, "
                  f"threads={threads}; ms/chunk extrapolated x{c['heads']} heads x{c['T']} steps")
    else:
        kind = "port"
        sample = (f"1 head of 1 denoising-step call of chunk {c['chunk']} per step (oracle port "
                  f"of chunkattn.hsa_attention, framewise n={c['n']}), OPENBLAS_NUM_THREADS=1, "
                  f"threads={threads}; ms/chunk extrapolated x{c['heads']} heads x{c['T']} steps")
    port = None
    if real:  # the framewise port at the workload's own n, beside it
        pt, pf = 0.0, 0
        for j in range(max(1, min(args.steps, 3))):
            dt, fl = oracle_sample(c, s_i, 2000 + j, threads)
            pt += dt
            pf += fl
        port = {"value": pf / pt / 1e12, "unit": UNIT, "cores": threads, "kind": "port",
                "sample": f"framewise oracle port at n={c['n']}, "
                          f"{max(1, min(args.steps, 3))} head-call(s)"}
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": statistics.mean(times) * 1e3, "ms_per_chunk": ms_chunk,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32/f64",
        "data": "synthetic",
        "config": job_config(args, c, s_i, world),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": kind,
                         "sample": sample, "cpu": cpu_desc()},
        "port_framewise": port,
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------- GPU leg


def issued_mma_flops(plan, d):
    """FLOPs the tensor cores execute for one attention call under its tile
    plan: every (128-row query tile, 128-key tile) the kernel computes costs
    4*128*128*d (QK^T + PV), whatever part of it the selection needs (rows of
    a tile share the union of their query blocks' key blocks)."""
    import numpy as np
    from paper_2602_04789_b200 import device as dv
    qt = plan.qt
    H = plan.q.shape[0]
    mode = getattr(plan, "qmode", None)
    mode = dv.qtile_mode(qt) if mode is None else mode
    nq = -(-qt.count // 2) if mode else -(-qt.total // 128)
    tq = -(-qt.total // 128)
    dense = nq * tq * H  # the current chunk: every query tile x every chunk key tile
    if plan.tiles is None:  # chunk 1: no past
        return dense * 4 * 128 * 128 * d
    segs = plan.tiles.segs.cpu().numpy()
    cnt = plan.tiles.seg_count.cpu().numpy()
    ntiles = cnt.shape[1]
    total = 0
    for t in range(ntiles):
        if mode == 2:  # paired tiles: plan bits 0, 1 = query tile 2t, bits 2, 3 = 2t + 1
            ma, mb = 0b0011, 0b1100
        else:
            q0, mid = dv.qtile_rows(qt, mode, 2 * t)
            q1 = dv.qtile_rows(qt, mode, 2 * t + 1)[1] if 2 * t + 1 < nq else mid
            qb0 = qt.block_of(q0)

            def bits(r0, r1):
                if r0 >= r1:
                    return 0
                lo, hi = qt.block_of(r0) - qb0, min(qt.block_of(r1 - 1) - qb0, 31)
                return ((2 << hi) - 1) & ~((1 << lo) - 1)
            ma, mb = bits(q0, mid), bits(mid, q1)
        for h in range(H):
            n = int(cnt[h, t])
            m = segs[h, t, :n, 2].astype(np.int64)
            if n & 1:
                m = np.append(m, 0)
            pm = m[0::2] | m[1::2]
            total += int(((pm & ma) != 0).sum()) + int(((pm & mb) != 0).sum())
    return (total + dense) * 4 * 128 * 128 * d


def run_ours(args, c):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2602_04789_b200 as lf
    from paper_2602_04789_b200 import device as D
    from paper_2602_04789_b200.selection import tilings
    from paper_2602_04789_b200.sharding import (gather_heads, gather_heads_overlapped,
                                                partition_heads)

    rank, world, local = dist_env()
    # LF_BENCH_DIST_CHECK=1 (under torchrun): a functional check of the N-rank
    # flow (head shards, eager gathers between step graphs, max-over-ranks
    # timing, the JSON line) with every rank on the node's first GPUs and gloo
    # for the collectives; not a measurement (the line says so)
    dist_check = world > 1 and os.environ.get("LF_BENCH_DIST_CHECK") == "1"
    if dist_check:
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if dist_check:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    H, d, f, n, i, T = c["heads"], c["d"], c["f"], c["n"], c["chunk"], c["T"]
    lay = make_layout(lf, c)
    cfg = lf.SelectionConfig(topk_frames=c["topk"], block_budget_mode=c["mode"])
    shard = partition_heads(H, world, rank)
    mode, h_local, h0 = shard.mode, shard.local_heads, shard.h0
    scaling = "strong" if mode == "headshard" else "weak"

    # CAG plan solved on device; the selection kernel reads s_i from device memory
    if c["plan"] is not None:
        plan = lf.allocate(c["plan"][0], c["plan"][1], c["N"], T, lay)
        s_dev = plan.device.s[i - 1:i]
        s_host = plan.s[i - 1]
    else:
        s_host = float(c["s"])
        s_dev = torch.tensor([s_host], dtype=torch.float64, device=dev)

    lq, lk = f * n, i * f * n
    video = rank if mode == "replica" else 0

    def gen(step, rows, h_start):
        g = torch.Generator(device=dev)
        out = torch.empty((h_local, rows, d), dtype=torch.bfloat16, device=dev)
        for h in range(h_local):
            g.manual_seed(((video * 64 + step) * 1024 + h_start + h) * 7 + rows)
            out[h] = torch.randn((rows, d), generator=g, device=dev).to(torch.bfloat16)
        return out

    Q = [gen(s, lq, h0) for s in range(T)]
    K = [gen(s + 100, lk, h0) for s in range(T)]
    V = [gen(s + 200, lk, h0) for s in range(T)]
    # the per-call contract returns the output (hsa_attention's mask comes from the
    # blocks): no frame lists, so a call with past budget 0 skips the frame ranking
    pipes = [lf.HsaPipeline(lay, h_local, i, cfg, framewise=True, out_dtype=torch.bfloat16,
                            keep_frames=False)
             for _ in range(T)]
    outs = [p.bind(Q[s], K[s], V[s], s_dev, s_host=s_host) for s, p in enumerate(pipes)]
    full = [torch.empty((H, lq, d), dtype=torch.bfloat16, device=dev) for _ in range(T)] \
        if mode == "headshard" else None

    def gather(s):
        if mode == "headshard":
            gather_heads(outs[s], shard, out=full[s])

    if args.profile_launch:
        for _ in range(2):
            for s in range(T):
                pipes[s].launch()
        torch.cuda.synchronize()
        return

    clocks = ClockSampler(local).start()
    for _ in range(max(args.warmup, 3)):
        for s in range(T):
            pipes[s].launch()
            gather(s)
    torch.cuda.synchronize()
    for p in pipes:
        p.capture()
    for _ in range(2):
        for s in range(T):
            pipes[s].replay()
            gather(s)
    torch.cuda.synchronize()
    errs = sum(p.errors() for p in pipes)

    # effective (selected) FLOPs of one step = T calls, summed over ranks
    flops_local = sum(p.effective_flops() for p in pipes)
    fl = torch.tensor([float(flops_local)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(fl)
    flops_step = float(fl.item())

    # ---- timed region: K steps of graph replays (+ all-gather when sharded)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        for s in range(T):
            pipes[s].replay()
            gather(s)
    e1.record()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = e0.elapsed_time(e1) / args.steps
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_step = float(t.item())
    value_stateless = flops_step / (ms_step * 1e-3) / 1e12

    # ---- the same chunk through the rollout driver (device KV cache, past
    # summaries pooled once per committed chunk): one step = commit of chunk
    # i-1 (re-pooled, as a real rollout does once per chunk) + T denoising calls
    from paper_2602_04789_b200.rollout import HsaRollout
    past = (i - 1) * lq
    ro = HsaRollout(lay, h_local, plan if c["plan"] is not None else None, cfg, framewise=True)
    for t in range(1, i):
        sl = slice((t - 1) * lq, t * lq)
        ro.commit(K[0][:, sl], V[0][:, sl], t)
    Kc = [K[s][:, past:].contiguous() for s in range(T)]
    Vc = [V[s][:, past:].contiguous() for s in range(T)]
    Kprev = K[0][:, past - lq:past].contiguous() if i > 1 else None
    Vprev = V[0][:, past - lq:past].contiguous() if i > 1 else None
    r_out = [torch.empty((h_local, lq, d), dtype=torch.bfloat16, device=dev) for _ in range(T)]

    # the producer writes K/V projections straight into the cache slot; the
    # current chunk's K/V of step 0 stand in for every step (selection only
    # reads past summaries, and attention cost does not depend on the values)
    ro.kv_slot(i)[0].copy_(Kc[0])
    ro.kv_slot(i)[1].copy_(Vc[0])

    # Step order (LF_BENCH_FLOW).  serial (the headline): each call's pool q ->
    # select -> plan -> attention in order on one stream, call after call -- what
    # a denoiser allows, whose query of step s+1 depends on the output of step s.
    # overlap (A/B only, rounds 1-2's headline): the selection half of step s+1
    # enqueued on a side stream while step s attends, which a real denoiser
    # cannot do (profiles/r02/flow_ab.txt; two stream-priority variants measured
    # there were dropped)
    flow = os.environ.get("LF_BENCH_FLOW", "serial")
    if flow not in ("serial", "overlap"):
        raise SystemExit(f"LF_BENCH_FLOW={flow}: serial | overlap")
    side = torch.cuda.Stream()
    comm = torch.cuda.Stream()
    ev_prep = [torch.cuda.Event() for _ in range(T)]

    def chunk_flow():
        main = torch.cuda.current_stream()
        if i > 1:
            ro.commit(None, None, i - 1, overwrite=True)
        plans = [None] * T
        if flow == "serial":
            for s in range(T):
                plans[s] = ro.prepare(Q[s], i, s_i=s_dev, s_host=s_host)
                ro.attend(plans[s], out=r_out[s])
                if mode == "headshard":
                    gather_heads_overlapped(r_out[s], shard, full[s], comm)
            if mode == "headshard":
                main.wait_stream(comm)
            return plans
        side.wait_stream(main)

        def prep(s):
            with torch.cuda.stream(side):
                plans[s] = ro.prepare(Q[s], i, s_i=s_dev, s_host=s_host)
                ev_prep[s].record(side)
        prep(0)
        for s in range(T):
            if s + 1 < T:
                prep(s + 1)
            main.wait_event(ev_prep[s])
            ro.attend(plans[s], out=r_out[s])
            if mode == "headshard":  # all-gather of call s overlaps the compute of s+1
                gather_heads_overlapped(r_out[s], shard, full[s], comm)
        main.wait_stream(side)
        if mode == "headshard":
            main.wait_stream(comm)
        return plans

    flops_r = 0
    mma_r = 0
    for s in range(T):
        pl = ro.prepare(Q[s], i, s_i=s_dev, s_host=s_host)
        ro.attend(pl, out=r_out[s])
        flops_r += ro.selection_flops()
        mma_r += issued_mma_flops(pl, d)
    for _ in range(max(args.warmup, 3)):
        chunk_flow()
    torch.cuda.synchronize()
    if mode == "headshard" and flow == "serial":
        # NCCL stays out of the graphs: one graph per step (compute only), the
        # all-gather of step s launched eagerly on the comm stream after it
        # (overlapping step s+1), so a rank never replays a captured collective
        g_steps = []
        for s in range(T):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                if s == 0 and i > 1:
                    ro.commit(None, None, i - 1, overwrite=True)
                ro.attend(ro.prepare(Q[s], i, s_i=s_dev, s_host=s_host), out=r_out[s])
            g_steps.append(g)

        def run_chunk():
            for s in range(T):
                g_steps[s].replay()
                gather_heads_overlapped(r_out[s], shard, full[s], comm)
            torch.cuda.current_stream().wait_stream(comm)
    else:
        g_chunk = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g_chunk):
            chunk_flow()
        run_chunk = g_chunk.replay
    run_chunk()
    torch.cuda.synchronize()
    fl = torch.tensor([float(flops_r)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(fl)
        dist.barrier()
    flops_r_step = float(fl.item())
    torch.cuda.synchronize()
    e0.record()
    for _ in range(args.steps):
        run_chunk()
    e1.record()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t = torch.tensor([e0.elapsed_time(e1) / args.steps], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_chunk_r = float(t.item())
    clk = clocks.stop()
    if os.environ.get("LF_BENCH_TIMELINE") and rank == 0:
        timeline_dump(run_chunk, os.environ["LF_BENCH_TIMELINE"])
        timeline_dump(chunk_flow, os.environ["LF_BENCH_TIMELINE"] + ".eager.csv")
    value = flops_r_step / (ms_chunk_r * 1e-3) / 1e12
    if os.environ.get("LF_BENCH_PROBE") and rank == 0:
        # profiling aid: the rollout's attention calls alone (plans prepared once),
        # each in its own graph, replayed back to back -- against the stage timing
        pls = [ro.prepare(Q[s], i, s_i=s_dev, s_host=s_host) for s in range(T)]
        gA = []
        for s in range(T):
            ro.attend(pls[s], out=r_out[s])
        torch.cuda.synchronize()
        for s in range(T):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                ro.attend(pls[s], out=r_out[s])
            gA.append(g)
        for variant in ("rotate", "same"):
            a_, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            for s in range(T):
                gA[s].replay()
            a_.record()
            for _ in range(10):
                for s in range(T):
                    gA[s if variant == "rotate" else 0].replay()
            b_.record()
            torch.cuda.synchronize()
            sys.stderr.write(f"probe: rollout attention alone ({variant}) "
                             f"{a_.elapsed_time(b_) / (10 * T) * 1e3:.1f} us/call\n")
    errs += int(ro.err.item())

    # ---- kernel-level timing for the roofline: the same kernels on the same
    # inputs, each stage captured in its own CUDA graph so that no host launch
    # gap is timed; events bracket graph replays on the current stream
    qt, kt = tilings(lay, i, True)
    bpf = lay.frame_kv_blocks
    P = (i - 1) * f
    hint = D.past_tiles_hint(s_host, i, f, bpf, c["topk"], qt)
    qmode = D.auto_qtile_mode(s_host, i, f, bpf, c["topk"])  # as HsaRollout.prepare picks it
    from paper_2602_04789_b200 import _lib as LL
    stage = {"pool": [], "select": [], "attn": []}
    graphs = []
    for s in range(T):
        st = {}

        def run_pool(s=s, st=st):
            st["views"] = D.compress(Q[s], K[s], qt, kt, bpf, P)

        def run_sel(s=s, st=st):
            qb, kb, kf = st["views"]
            with D.qtile_scope(qmode):
                # as the per-call pipeline runs it (no frame lists: skip_frames)
                _, st["tiles"], _ = D.select_plan(qb, kb, kf, bpf, i, f, c["topk"],
                                                  c["mode"] == "per-frame", s_dev, qt, kt, P * bpf,
                                                  want_frames=False)

        def run_attn(s=s, st=st):
            with D.qtile_scope(qmode):
                D.attention(Q[s], K[s], V[s], qt, st["tiles"], P * n, lk, out=outs[s],
                            past_tiles=hint, qperm=st["tiles"].qperm if st["tiles"] else None)

        fns = (run_pool, run_sel, run_attn)
        for fn in fns:  # warm (allocates the static buffers the graphs reuse)
            fn()
        torch.cuda.synchronize()
        gs = []
        for fn in fns:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                fn()
            gs.append(g)
        graphs.append(gs)
    torch.cuda.synchronize()
    # each stage's graphs replayed back to back (T different inputs in rotation,
    # > L2 in total) between two events on this stream: per-launch device time
    # with the host launch latency of the graph hidden behind the previous replay
    reps = max(5, min(args.steps, 50))
    for si, name in enumerate(("pool", "select", "attn")):
        ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for s in range(T):  # warm
            graphs[s][si].replay()
        ea.record()
        for r in range(reps):
            for s in range(T):
                graphs[s][si].replay()
        eb.record()
        torch.cuda.synchronize()
        stage[name].append(ea.elapsed_time(eb) / (reps * T))
    attn_ms = statistics.mean(stage["attn"])
    if os.environ.get("LF_BENCH_PROBE") and rank == 0:
        sys.stderr.write(f"probe: stage attention (stateless inputs) {attn_ms * 1e3:.1f} us/call\n")
    pool_ms = statistics.mean(stage["pool"])
    sel_ms = statistics.mean(stage["select"])
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except (OSError, ValueError):
        pass
    tf_peak = peaks.get("bf16_tflops")
    hbm_peak = peaks.get("hbm_gbs")
    tf_src = "MEASURED_PEAKS.json bf16_tflops (burst), of measured"
    hbm_src = "MEASURED_PEAKS.json hbm_gbs, of measured"
    if tf_peak is None:  # B200_PROFILING.md fallback when the driver file is absent
        tf_peak, tf_src = 1590.0, "B200_PROFILING.md fallback 1.59 PFLOP/s burst, of fallback"
    if hbm_peak is None:
        hbm_peak, hbm_src = 6650.0, "B200_PROFILING.md fallback 6.65 TB/s, of fallback"
    traffic = {}
    try:
        traffic = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
    except (OSError, ValueError):
        pass
    flops_call = flops_local / T
    mma_call = mma_r / T
    achieved_tf = flops_call / (attn_ms * 1e-3) / 1e12
    pool_bytes = h_local * (lq + lk) * d * 2 + h_local * (qt.count + kt.count + P) * d * 4
    achieved_gbs = pool_bytes / (pool_ms * 1e-3) / 1e9
    stage_gbs = pool_bytes / ((pool_ms + sel_ms) * 1e-3) / 1e9

    # ---- end to end through the public API with pinned host buffers, H2D of
    # every step's inputs and D2H of its output inside the timed region
    e2e_steps = max(3, min(args.steps, 20))

    def timed(fn, reps, no_gc=False):
        for _ in range(max(args.warmup, 3)):  # the same W >= 3 warm-up steps as the headline
            fn()
        torch.cuda.synchronize()
        gc_was = gc.isenabled()
        if no_gc:
            gc.collect()
            gc.disable()
        if world > 1:
            dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        marks = [torch.cuda.Event(enable_timing=True) for _ in range(reps)] \
            if os.environ.get("LF_BENCH_TRACE") else None
        ms0 = torch.cuda.memory_stats() if marks else None
        h0 = time.perf_counter()
        a.record()
        for r in range(reps):
            fn()
            if marks:
                marks[r].record()
        b.record()
        h1 = time.perf_counter()
        torch.cuda.synchronize()
        if marks:
            ms1 = torch.cuda.memory_stats()
            sys.stderr.write("host enqueue ms/iter %.3f; allocator: %s\n" % (
                (h1 - h0) * 1e3 / reps, {k: ms1.get(k, 0) - ms0.get(k, 0) for k in (
                    "num_device_alloc", "num_device_free", "num_alloc_retries",
                    "num_sync_all_streams")}))
        if no_gc and gc_was:
            gc.enable()
        if marks:
            per = [a.elapsed_time(marks[0])] + [marks[r - 1].elapsed_time(marks[r])
                                                for r in range(1, reps)]
            sys.stderr.write("timed: " + " ".join(f"{x:.2f}" for x in per) + "\n")
        tt = torch.tensor([a.elapsed_time(b) / reps], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        return float(tt.item())

    # (a) stateless per-call pipeline (lf_hsa_forward): full Q/K/V per call
    hq = [x.cpu().pin_memory() for x in Q]
    hk = [x.cpu().pin_memory() for x in K]
    hv = [x.cpu().pin_memory() for x in V]
    ho = [torch.empty(outs[s].shape, dtype=outs[s].dtype).pin_memory() for s in range(T)]
    h2d_sl = sum(x.numel() * 2 for x in hq + hk + hv)
    d2h = sum(x.numel() * 2 for x in ho)

    def e2e_stateless():
        for s in range(T):
            Q[s].copy_(hq[s], non_blocking=True)
            K[s].copy_(hk[s], non_blocking=True)
            V[s].copy_(hv[s], non_blocking=True)
            pipes[s].replay()
            gather(s)
            ho[s].copy_(outs[s], non_blocking=True)

    e2e_ms_sl = timed(e2e_stateless, e2e_steps, no_gc=True)

    # (b) rollout driver (HsaRollout): per chunk the previous clean chunk's K/V
    # (commit) and, per denoising step, the current chunk's q, k, v
    hkc = [x.cpu().pin_memory() for x in Kc]
    hvc = [x.cpu().pin_memory() for x in Vc]
    hkp = Kprev.cpu().pin_memory() if i > 1 else None
    hvp = Vprev.cpu().pin_memory() if i > 1 else None
    hro = [torch.empty(r_out[s].shape, dtype=r_out[s].dtype).pin_memory() for s in range(T)]
    h2d = sum(x.numel() * 2 for x in hq + hkc + hvc) + (2 * hkp.numel() * 2 if i > 1 else 0)

    # copies overlap compute: H2D of step s+1 into a staging pair on a copy
    # stream while step s runs, a device copy into the cache slot (HBM, ~10 us),
    # D2H of each output on a third stream; PCIe H2D is the e2e bound
    s_h2d, s_d2h = torch.cuda.Stream(), torch.cuda.Stream()
    stg_q = [torch.empty_like(Q[0]) for _ in range(2)]
    stg_k = [torch.empty_like(Kc[0]) for _ in range(2)]
    stg_v = [torch.empty_like(Vc[0]) for _ in range(2)]
    ev_in = [torch.cuda.Event() for _ in range(2)]
    ev_free = [torch.cuda.Event() for _ in range(2)]
    ev_out = [torch.cuda.Event() for _ in range(T)]

    stg_kp = torch.empty_like(Kprev) if i > 1 else None  # previous clean chunk's K/V
    stg_vp = torch.empty_like(Vprev) if i > 1 else None

    # One chunk through the public API, captured in a CUDA graph together with
    # its copies (an eager host loop of these calls took 2-8 ms per chunk on a
    # loaded host and grew the caching allocator inside the timed region --
    # e2e swung 2x between runs).  Software-pipelined across replays: a replay
    # finds step 0's q, k, v and the previous clean chunk's K/V already in
    # staging (loaded by the previous replay's tail, or by the prologue below)
    # and ends by loading them for the next one while its last step computes,
    # so every replay moves exactly one chunk's inputs over PCIe and the link
    # does not idle at the chunk boundary.  Each call's pool q -> select ->
    # plan -> attention runs in order on the compute stream (as the headline);
    # the H2D of step s+1 overlaps step s, the D2H of each output follows it.
    def h2d_step(s, wait_free):
        b = s & 1
        with torch.cuda.stream(s_h2d):
            if wait_free:
                s_h2d.wait_event(ev_free[b])  # staging b no longer read by compute
            stg_q[b].copy_(hq[s], non_blocking=True)
            stg_k[b].copy_(hkc[s], non_blocking=True)
            stg_v[b].copy_(hvc[s], non_blocking=True)

    def h2d_prev():
        with torch.cuda.stream(s_h2d):
            stg_kp.copy_(hkp, non_blocking=True)
            stg_vp.copy_(hvp, non_blocking=True)

    ev_kv = torch.cuda.Event()

    def e2e_chunk():
        cur = torch.cuda.current_stream()
        for st in (s_h2d, s_d2h):
            st.wait_stream(cur)
        if i > 1:  # previous clean chunk: staging -> its cache slot, pooled once
            kp, vp = ro.kv_slot(i - 1)
            kp.copy_(stg_kp)
            vp.copy_(stg_vp)
            ev_kv.record(cur)
            ro.commit(None, None, i - 1, overwrite=True)
        last_even = (T - 1) & ~1  # the last step reading staging 0
        for s in range(T):
            b = s & 1
            if s + 1 < T:
                h2d_step(s + 1, wait_free=s >= 1)  # staging (s+1)&1 last read by step s-1
                ev_in[(s + 1) & 1].record(s_h2d)
            if s > 0:
                cur.wait_event(ev_in[b])
            kc, vc = ro.kv_slot(i)
            kc.copy_(stg_k[b])
            vc.copy_(stg_v[b])
            pl = ro.prepare(stg_q[b], i, s_i=s_dev, s_host=s_host)
            ro.attend(pl, out=r_out[s])
            ev_free[b].record(cur)
            ev_out[s].record(cur)
            with torch.cuda.stream(s_d2h):
                s_d2h.wait_event(ev_out[s])
                hro[s].copy_(r_out[s], non_blocking=True)
            if s == last_even:  # the next replay's inputs, behind this chunk's last steps
                h2d_step(0, wait_free=True)
                if i > 1:
                    with torch.cuda.stream(s_h2d):
                        s_h2d.wait_event(ev_kv)
                    h2d_prev()
        cur.wait_stream(s_h2d)
        cur.wait_stream(s_d2h)  # the chunk ends when its outputs are on the host

    # prologue: the first replay's inputs
    h2d_step(0, wait_free=False)
    if i > 1:
        h2d_prev()
    torch.cuda.current_stream().wait_stream(s_h2d)
    for _ in range(2):
        e2e_chunk()
    torch.cuda.synchronize()
    g_e2e = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g_e2e):
        e2e_chunk()
    torch.cuda.synchronize()

    def e2e_replay():
        g_e2e.replay()
        if mode == "headshard":  # the chunk's all-gathers, eager (NCCL stays out of graphs)
            for s in range(T):
                gather_heads_overlapped(r_out[s], shard, full[s], comm)
            torch.cuda.current_stream().wait_stream(comm)
    e2e_ms = timed(e2e_replay, e2e_steps, no_gc=True)

    # ---- CPU baseline (rank 0, N = 1 only): the oracle on a bounded sample of
    # the same workload -- head-calls of this chunk until ~10 s of CPU work or
    # the whole chunk (H heads x T calls), whichever comes first
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        # the real reference (oracle/_ref) at the aligned n, ~10 s of head-calls
        real = ref_aligned_sample(c, s_host, 4141, threads)
        if real is not None:
            tot_t, tot_f, calls = real[0], real[1], 1
            while calls < H * T and tot_t < 10.0:
                dt, fl, n_al = ref_aligned_sample(c, s_host, 4242 + calls, threads)
                tot_t += dt
                tot_f += fl
                calls += 1
            cpu = {"value": tot_f / tot_t / 1e12, "unit": UNIT, "cores": threads,
                   "kind": "reference",
                   "sample": (f"{calls} of the {H * T} head-calls of one chunk-{i} step through "
                              f"the unmodified chunkattn.hsa_attention (oracle/_ref) at the "
                              f"aligned n={real[2]} (it rejects n={n}), {tot_t:.1f} s; "
                              f"OPENBLAS_NUM_THREADS=1, threads={threads}"),
                   "ms_per_chunk": tot_t / calls * H * T * 1e3,
                   "ms_per_chunk_is_extrapolated": calls < H * T, "cpu": cpu_desc()}
        # the framewise oracle port at the workload's own n (the value when no
        # reference is staged, else beside it on a smaller sample)
        tot_t, tot_f, calls = 0.0, 0, 0
        budget_s = 10.0 if cpu is None else 3.0
        while calls < H * T and tot_t < budget_s:
            dt, cflops = oracle_sample(c, s_host, 4242 + calls, threads)
            tot_t += dt
            tot_f += cflops
            calls += 1
        port = {"value": tot_f / tot_t / 1e12, "unit": UNIT, "cores": threads, "kind": "port",
                "sample": (f"{calls} of the {H * T} head-calls of one chunk-{i} step (framewise "
                           f"oracle port of chunkattn.hsa_attention), {tot_t:.1f} s; "
                           f"OPENBLAS_NUM_THREADS=1, threads={threads}"),
                "ms_per_chunk": tot_t / calls * H * T * 1e3,
                "ms_per_chunk_is_extrapolated": calls < H * T, "cpu": cpu_desc()}
        if cpu is None:
            cpu = port
        else:
            cpu["port_framewise"] = port

    # PCIe bound of the e2e leg: the step's H2D copies alone (same pinned
    # buffers, same order), timed on the device
    def h2d_only():
        if i > 1:
            kp, vp = ro.kv_slot(i - 1)
            kp.copy_(hkp, non_blocking=True)
            vp.copy_(hvp, non_blocking=True)
        for s in range(T):
            stg_q[s & 1].copy_(hq[s], non_blocking=True)
            stg_k[s & 1].copy_(hkc[s], non_blocking=True)
            stg_v[s & 1].copy_(hvc[s], non_blocking=True)
    h2d_only_ms = timed(h2d_only, 3)
    h2d_gbs = h2d / (h2d_only_ms * 1e-3) / 1e9

    # pool(Q+K), pool(k_frame), select, plan_tiles, attention; chunk 1 has no past stages
    # rollout flow per chunk: commit (2 pool launches) + T x (pool Q, select,
    # plan tiles, attention); chunk 1 has no past (no commit, no tile plan)
    # (+ the two pairing kernels per step under query-tile geometry 2)
    paired = int(getattr(pl, "qmode", 0) or 0) == 2
    launches_per_chunk = T * ((4 if P > 0 else 3) + (2 if paired else 0)) + (2 if i > 1 else 0)
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_chunk_r,
            "ms_per_chunk": ms_chunk_r, "higher_is_better": True, "scaling": scaling,
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": job_config(args, c, s_host, world),
            **({"dist_check": "functional check: all ranks on one GPU, gloo; not a measurement"}
               if dist_check else {}),
            "query_tiles": {0: "128-row", 1: "block-aligned (2 query blocks)",
                            2: "2 query blocks paired by selection overlap"}.get(
                                int(getattr(pl, "qmode", 0) or 0), "128-row"),
            "step_order": flow + (" (each call's pool q -> select -> plan -> attention in order,"
                                  " call after call)" if flow == "serial" else " (A/B variant)"),
            "e2e": {"value": flops_r_step / (e2e_ms * 1e-3) / 1e12, "unit": UNIT,
                    "ms_per_chunk": e2e_ms, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "api": "HsaRollout.commit + prepare/attend (C ABI underneath) with the chunk's H2D/D2H copies from/to pinned host memory, one CUDA graph per chunk; H2D of step s+1 and of the next chunk's first inputs overlap compute",
                    "h2d_gbs_measured": h2d_gbs,
                    "pcie_bound_ms_per_chunk": h2d_only_ms},
            "stateless": {"value": value_stateless, "unit": UNIT, "ms_per_chunk": ms_step,
                          "api": "HsaPipeline / lf_hsa_forward, full K/V per call",
                          "e2e_value": flops_step / (e2e_ms_sl * 1e-3) / 1e12,
                          "e2e_ms_per_chunk": e2e_ms_sl, "e2e_h2d_bytes_per_step": h2d_sl},
            "roofline": {"bound": "tensor",
                         "kernel": "attn_fwd_v7_kernel<128> (query tile, two softmax sets)",
                         "achieved": achieved_tf, "peak": tf_peak, "unit": "TFLOP/s",
                         "frac": achieved_tf / tf_peak,
                         "traffic": (traffic.get("attn_fwd", {}).get("bytes")
                                     if args.config == "c2" else None),
                         "traffic_source": traffic.get("attn_fwd", {}).get("source"),
                         "peak_source": tf_src,
                         "attn_ms_per_call": attn_ms, "flops_per_call": flops_call,
                         "issued_mma_flops_per_call": mma_call,
                         "issued_tflops": mma_call / (attn_ms * 1e-3) / 1e12,
                         "issued_frac": mma_call / (attn_ms * 1e-3) / 1e12 / tf_peak,
                         "note": "achieved counts the selection's FLOPs; issued counts the "
                                 "128x128 tiles the tile plan makes the kernel compute"},
            "roofline_select": {"bound": "hbm",
                                "kernel": "mask-selection stage: pool_frames_tma_kernel (Q+K block "
                                          "pooling) + select_cta_kernel + plan_tiles_cta_kernel",
                                "achieved": stage_gbs, "peak": hbm_peak, "unit": "GB/s",
                                "frac": stage_gbs / hbm_peak, "peak_source": hbm_src,
                                "traffic": (traffic.get("pool", {}).get("bytes")
                                            if args.config == "c2" else None),
                                "bytes_per_call": pool_bytes,
                                "stage_ms_per_call": pool_ms + sel_ms,
                                "pool_ms_per_call": pool_ms, "select_plan_ms_per_call": sel_ms,
                                "pool_gbs": achieved_gbs, "pool_frac": achieved_gbs / hbm_peak,
                                "note": "achieved = the stage's algorithmic HBM bytes (bf16 Q and "
                                        "K reads + fp32 summary writes) / (pool + select + plan "
                                        "time); selection and plan read the summaries from L2"},
            "cpu_baseline": cpu,
            "clocks": clk,
            "gpu_launches": launches_per_chunk * args.steps,
            "device_errors": errs,
            "effective_flops_per_step": flops_step,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def timeline_dump(fn, path: str, reps: int = 3) -> None:
    """LF_BENCH_TIMELINE=path: the device timeline of `reps` replays (kernel and
    copy intervals per stream, CUPTI via torch.profiler) as CSV -- where the
    rollout step's time goes beyond the attention kernel (profiling aid; not a
    bench number)."""
    import torch
    from torch.profiler import ProfilerActivity, profile
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(reps):
            fn()
        torch.cuda.synchronize()
    rows = []
    for ev in prof.events():
        if ev.device_type.name != "CUDA":
            continue
        rows.append((ev.time_range.start, ev.time_range.end - ev.time_range.start,
                     getattr(ev, "device_resource_id", -1), ev.name[:90]))
    rows.sort()
    t0 = rows[0][0] if rows else 0
    with open(path, "w") as fh:
        fh.write("start_us,dur_us,stream,name\n")
        for st, du, sid, nm in rows:
            fh.write(f"{st - t0:.2f},{du:.2f},{sid},\"{nm}\"\n")


def self_launch(args) -> int:
    """`bench.py --gpus N` outside torchrun: start N ranks (one per GPU) through
    torch.distributed.run on 127.0.0.1 with the same arguments; rank 0 prints
    the line.  Refuses (non-zero exit, reason on stderr) when the node has
    fewer than N GPUs -- never a silent single-GPU run."""
    n = args.gpus
    if args.impl == "ours":
        import torch
        have = torch.cuda.device_count()
        if have < n:
            sys.stderr.write(f"bench.py: --gpus {n} needs {n} CUDA devices, this node has {have}\n")
            return 2
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    args = parse()
    c = CONFIGS[args.config]
    world = int(os.environ.get("WORLD_SIZE", "0"))
    if world == 0 and args.gpus > 1:
        sys.exit(self_launch(args))
    if world and world != args.gpus:
        sys.stderr.write(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}\n")
        sys.exit(2)
    if args.impl == "reference":
        run_reference(args, c)
    else:
        run_ours(args, c)


if __name__ == "__main__":
    main()
