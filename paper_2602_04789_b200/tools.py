"""Report tooling in the reference CLI's formats, on the GPU kernels.

* ``bench_sweep`` -- the kernel timing sweep of ``chunkattn bench``
  (cli.py:125-178): dense vs block-sparse attention on random row masks, one
  RFC-4180 CSV row per density with the run's config hash, under a
  ``# config:`` comment line (cli.py:71-78).  Masks, config, hash and the
  deterministic columns are the reference's; times are CUDA-event medians of
  the GPU kernels, ``max_abs_err_vs_dense`` compares the GPU sparse and dense
  outputs.
* ``mask_dump`` -- ``chunkattn mask-dump`` (cli.py:220-266): one hierarchical
  selection on seeded inputs, the mask as a binary PGM (attention.py:133-138)
  and optionally the canonical-JSON selection trace (selection.py:234-249).

    python -m paper_2602_04789_b200.tools bench --seq 8192 --dim 64 --out bench.csv
    python -m paper_2602_04789_b200.tools mask-dump --chunk 7 --out mask.pgm --trace t.json

The CLI itself (argument handling, exit codes) is outside the hot path (DESIGN
§8); these entry points exist so reports made with the GPU kernels can be
diffed against the reference's.
"""

from __future__ import annotations

import argparse
import statistics
import sys

import numpy as np

from .attention import block_sparse_attention, dense_attention
from .layout import BlockMask, ChunkLayout
from .planner import chunk_block_budget
from .reports import canonical_json, config_hash, write_csv
from .selection import (SelectionConfig, build_mask, compress, frame_scores, select_blocks,
                        select_frames, selection_trace)

BENCH_HEADER = ["config_hash", "seq", "d", "b_q", "b_kv", "density", "sparsity", "active_tiles",
                "total_tiles", "flops", "wall_time_dense", "wall_time_sparse", "speedup",
                "max_abs_err_vs_dense"]


def bench_mask(n_q: int, n_k: int, density: float, seed: int) -> BlockMask:
    """cli.py:93-100: round-half-up(density * n_k) random active blocks per row."""
    per_row = min(n_k, max(1, int(np.floor(density * n_k + 0.5))))
    rng = np.random.default_rng([seed, 23])
    bits = np.zeros((n_q, n_k), dtype=bool)
    for r in range(n_q):
        bits[r, rng.choice(n_k, size=per_row, replace=False)] = True
    return BlockMask(bits)


def bench_config(seq, dim, block, kv_block, densities, repeats, seed, threads):
    """The reference's bench config dict (cli.py:145-147) and its densities list
    (1.0 always first, cli.py:127-133)."""
    densities = [float(x) for x in densities]
    if any(not 0.0 < x <= 1.0 for x in densities):
        raise ValueError(f"densities must lie in (0, 1]: {densities}")
    if 1.0 not in densities:
        densities.insert(0, 1.0)
    b_kv = kv_block or block
    return densities, {"command": "bench", "seq": seq, "d": dim, "b_q": block, "b_kv": b_kv,
                       "densities": densities, "repeats": repeats, "seed": seed,
                       "threads": threads}


def _median_gpu_time(fn, repeats: int) -> float:
    """Median device time (s) over ``repeats`` runs after one discarded warmup."""
    import torch
    fn()
    torch.cuda.synchronize()
    times = []
    for _ in range(repeats):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        times.append(a.elapsed_time(b) * 1e-3)
    return statistics.median(times)


def bench_sweep(seq=8192, dim=64, block=64, kv_block=None, densities=(1.0, 0.5, 0.25, 0.1),
                repeats=5, seed=0, threads=1, out=None):
    """cmd_bench (cli.py:125-178) on the GPU kernels; returns (header, rows, config)."""
    import torch
    if repeats < 3:
        raise ValueError(f"--repeats must be >= 3, got {repeats}")
    densities, config = bench_config(seq, dim, block, kv_block, list(densities), repeats, seed,
                                     threads)
    b_kv = config["b_kv"]
    layout = ChunkLayout(f=1, n=seq, b_q=block, b_kv=b_kv, d=dim, N=1)
    rng = np.random.default_rng([seed, 17])
    q = rng.standard_normal((seq, dim)).astype(np.float32)
    k = rng.standard_normal((seq, dim)).astype(np.float32)
    v = rng.standard_normal((seq, dim)).astype(np.float32)
    dev = torch.device("cuda")
    qd, kd, vd = (torch.from_numpy(a).to(dev) for a in (q, k, v))
    dense_out = dense_attention(qd, kd, vd).double()
    t_dense = _median_gpu_time(lambda: dense_attention(qd, kd, vd), repeats)
    chash = config_hash(config)
    n_q, n_k = layout.q_blocks, layout.k_blocks(1)
    rows = []
    for density in densities:
        mask = bench_mask(n_q, n_k, density, seed)
        sparse_out, stats = block_sparse_attention(qd, kd, vd, mask, layout)
        t_sparse = _median_gpu_time(lambda: block_sparse_attention(qd, kd, vd, mask, layout),
                                    repeats)
        err = float((sparse_out.double() - dense_out).abs().max())
        rows.append([chash, seq, dim, block, b_kv, repr(density),
                     repr(1.0 - stats.active_tiles / stats.total_tiles), stats.active_tiles,
                     stats.total_tiles, stats.flop_estimate, repr(t_dense), repr(t_sparse),
                     repr(t_dense / t_sparse), repr(err)])
    if out:
        write_csv(out, BENCH_HEADER, rows, config)
    return BENCH_HEADER, rows, config


def mask_dump(frames=3, tokens=128, block=64, kv_block=None, dim=32, chunks=7, chunk=7,
              sparsity=0.9, topk=6, mode="global", seed=0, out=None, trace=None):
    """cmd_mask_dump (cli.py:220-266) on the GPU selection; returns (mask, trace rows)."""
    layout = ChunkLayout(f=frames, n=tokens, b_q=block, b_kv=kv_block or block, d=dim, N=chunks)
    i = chunk
    if not 0.0 <= sparsity < 1.0:
        raise ValueError(f"--sparsity must lie in [0, 1), got {sparsity}")
    cfg = SelectionConfig(topk_frames=topk, block_budget_mode=mode)
    rng = np.random.default_rng([seed, 29])
    q = rng.standard_normal((layout.chunk_tokens, layout.d)).astype(np.float32)
    k = rng.standard_normal((layout.context_tokens(i), layout.d)).astype(np.float32)
    views = compress(q, k, i, layout)
    current = layout.f * layout.frame_kv_blocks
    total = current if i == 1 else chunk_block_budget(sparsity, i, layout)
    past_budget = max(0, total - current)
    selections, score_rows = [], []
    for r in range(views.q_block.shape[0]):
        p = frame_scores(views, r)
        selections.append(select_blocks(views, r, select_frames(p, cfg, i, layout), past_budget,
                                         cfg))
        score_rows.append(p)
    mask = build_mask(selections, i, layout)
    if out:
        mask.to_pgm(out)
    rows = selection_trace(selections, score_rows)
    if trace:
        payload = {"config": {"command": "mask-dump", "f": layout.f, "n": layout.n,
                              "b_q": layout.b_q, "b_kv": layout.b_kv, "d": layout.d,
                              "N": layout.N, "chunk": i, "sparsity": sparsity,
                              "topk_frames": topk, "mode": mode, "seed": seed},
                   "rows": rows}
        with open(trace, "w", encoding="utf-8") as fh:
            fh.write(canonical_json(payload))
    return mask, rows


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_2602_04789_b200.tools")
    sub = ap.add_subparsers(dest="command", required=True)
    b = sub.add_parser("bench")
    b.add_argument("--seq", type=int, default=8192)
    b.add_argument("--dim", type=int, default=64)
    b.add_argument("--block", type=int, default=64)
    b.add_argument("--kv-block", type=int, default=None)
    b.add_argument("--densities", type=str, default="1.0,0.5,0.25,0.1")
    b.add_argument("--repeats", type=int, default=5)
    b.add_argument("--seed", type=int, default=0)
    b.add_argument("--out", type=str, default="bench.csv")
    m = sub.add_parser("mask-dump")
    m.add_argument("--frames", type=int, default=3)
    m.add_argument("--tokens", type=int, default=128)
    m.add_argument("--block", type=int, default=64)
    m.add_argument("--kv-block", type=int, default=None)
    m.add_argument("--dim", type=int, default=32)
    m.add_argument("--chunks", type=int, default=7)
    m.add_argument("--chunk", type=int, default=7)
    m.add_argument("--sparsity", type=float, default=0.9)
    m.add_argument("--topk", type=int, default=6)
    m.add_argument("--mode", type=str, default="global", choices=["global", "per-frame"])
    m.add_argument("--seed", type=int, default=0)
    m.add_argument("--out", type=str, default="mask.pgm")
    m.add_argument("--trace", type=str, default=None)
    args = ap.parse_args(argv)
    try:
        if args.command == "bench":
            _, rows, _ = bench_sweep(args.seq, args.dim, args.block, args.kv_block,
                                     [float(x) for x in args.densities.split(",") if x],
                                     args.repeats, args.seed, 1, args.out)
            print(f"wrote {args.out} ({len(rows)} rows)")
        else:
            mask, _ = mask_dump(args.frames, args.tokens, args.block, args.kv_block, args.dim,
                                args.chunks, args.chunk, args.sparsity, args.topk, args.mode,
                                args.seed, args.out, args.trace)
            print(f"mask {mask.n_q}x{mask.n_k}, active {mask.popcount()}, wrote {args.out}")
    except (ValueError, OSError, KeyError, IndexError) as exc:  # cli.py:329-340
        print(f"error: {exc}", file=sys.stderr)
        return 2
    return 0


if __name__ == "__main__":
    sys.exit(main())
