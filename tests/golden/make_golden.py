"""Generate golden fixtures by running the REAL reference package.

Run in the development container (the only place /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports ``chunkattn`` from /root/reference/pkg/src (read-only; nothing is
copied), runs its public functions on seeded inputs and writes the results to
``tests/golden/*.npz`` / ``*.json``.  Inputs are regenerated at test time from
the recorded seeds with ``oracle.lf_oracle.synthetic_qkv`` (numpy's PCG64), so
only outputs are stored.

n = 1560-style ragged layouts are rejected by the reference selection path
(selection.py:88-92); for those the fixtures are produced by composing the
reference's own functions exactly as SURVEY.md Appendix A.2 prescribes
(per-frame mean_pool, reference CompressedViews/frame_scores/select_frames/
select_blocks, reference dense_attention over each query block's active keys).
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
sys.dont_write_bytecode = True
REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REF)
sys.path.insert(0, ROOT)

import chunkattn as ca  # noqa: E402  (the reference)
from chunkattn import numerics as ca_num  # noqa: E402
from chunkattn import selection as ca_sel  # noqa: E402

from oracle.lf_oracle import Tiling, synthetic_qkv  # noqa: E402


def pool_fixtures():
    rng = np.random.default_rng(2602)
    cases = {}
    shapes = [(4, 1, 3), (64, 8, 64), (100, 5, 32), (1560, 16, 64), (130, 3, 48), (7, 2, 7), (200, 4, 1)]
    for idx, (rows, d, g) in enumerate(shapes):
        x = (rng.standard_normal((rows, d)) * np.exp(rng.uniform(-6, 6, (rows, 1)))).astype(np.float32)
        cases[f"x{idx}"] = x
        cases[f"g{idx}"] = np.int64(g)
        cases[f"out{idx}"] = ca_num.mean_pool(x, g)
    cases["x_hand"] = np.array([[1.0], [2.0], [3.0], [4.0]], np.float32)
    cases["out_hand"] = ca_num.mean_pool(cases["x_hand"], 3)
    np.savez_compressed(os.path.join(HERE, "pool.npz"), **cases)


def topk_fixtures():
    rng = np.random.default_rng(7)
    out = []
    vecs = [[3.0, 1.0, 2.0], [5.0, 7.0, 7.0, 5.0], [4.0, 4.0, 4.0, 4.0], [0.0, -0.0, 0.0, -1.0]]
    for _ in range(20):
        n = int(rng.integers(1, 200))
        v = np.round(rng.standard_normal(n), int(rng.integers(0, 3)))  # force ties
        vecs.append(v.tolist())
    for v in vecs:
        for k in (0, 1, 2, 3, 6, 50):
            res = ca_num.topk_indices(np.asarray(v, np.float64), k)
            out.append({"scores": v, "k": k, "indices": res.indices.tolist()})
    with open(os.path.join(HERE, "topk.json"), "w") as fh:
        json.dump(out, fh)


def _layout(f, n, b_q, b_kv, d, N):
    return ca.ChunkLayout(f=f, n=n, b_q=b_q, b_kv=b_kv, d=d, N=N)


# (name, f, n, b_q, b_kv, d, N)
HSA_LAYOUTS = [
    ("A", 3, 128, 64, 64, 16, 7),
    ("B", 2, 256, 64, 64, 64, 3),     # BASELINE config 1 shape
    ("C", 1, 128, 32, 64, 32, 5),
    ("D", 3, 192, 64, 64, 128, 5),
]


def hsa_fixtures():
    rows = []
    arrays = {}
    case = 0
    for name, f, n, b_q, b_kv, d, N in HSA_LAYOUTS:
        lay = _layout(f, n, b_q, b_kv, d, N)
        for i in sorted({1, 2, N // 2 + 1, N}):
            for s_i in (0.0, 0.35, 0.5, 0.75):
                for topk in (2, 6):
                    for mode in ("global", "per-frame"):
                        if mode == "per-frame" and topk == 6 and s_i != 0.5:
                            continue
                        seed = 1000 + case
                        # a few plain-fp32 (non-bf16) inputs exercise the pooling order
                        q, k, v = synthetic_qkv(seed, lay.chunk_tokens, lay.context_tokens(i), d,
                                                bf16=(case % 7 != 3))
                        q, k, v = q[0], k[0], v[0]
                        cfg = ca.SelectionConfig(topk_frames=topk, block_budget_mode=mode)
                        out, stats, mask = ca.hsa_attention(q, k, v, i, s_i, cfg, lay)
                        views = ca.compress(q, k, i, lay)
                        arrays[f"bits{case}"] = np.packbits(mask.bits, axis=1)
                        if case % 5 == 0:
                            arrays[f"qb{case}"] = views.q_block
                            arrays[f"kb{case}"] = views.k_block
                            arrays[f"kf{case}"] = views.k_frame
                        if case % 6 == 0:
                            arrays[f"out{case}"] = out
                        rows.append(dict(case=case, layout=name, f=f, n=n, b_q=b_q, b_kv=b_kv, d=d,
                                         N=N, i=i, s_i=s_i, topk=topk, mode=mode, seed=seed,
                                         fp32_inputs=bool(case % 7 == 3),
                                         nq=mask.n_q, nk=mask.n_k,
                                         active=stats.active_tiles, total=stats.total_tiles,
                                         flops=stats.flop_estimate, clamped=stats.budget_clamped,
                                         has_out=bool(case % 6 == 0),
                                         has_views=bool(case % 5 == 0)))
                        case += 1
    np.savez_compressed(os.path.join(HERE, "hsa_aligned.npz"), **arrays)
    with open(os.path.join(HERE, "hsa_aligned.json"), "w") as fh:
        json.dump(rows, fh, indent=0)


# framewise layouts (n not divisible by the block): composed from reference functions
FW_LAYOUTS = [
    ("R1", 2, 100, 32, 32, 16, 4),
    ("R2", 3, 1560, 64, 64, 8, 3),    # the BASELINE 480p frame, tiny head dim
    ("R3", 1, 90, 16, 40, 16, 5),
]


def _fw_bounds(total, n, b):
    return Tiling(total, n, b).all_bounds()


def framewise_reference(q, k, v, i, s_i, f, n, b_q, b_kv, topk, mode, N):
    lay = _layout(f, n, b_q, b_kv, q.shape[1], N)
    bpf = -(-n // b_kv)
    qb = _fw_bounds(f * n, n, b_q)
    kb = _fw_bounds(i * f * n, n, b_kv)
    q_block = np.concatenate([ca_num.mean_pool(q[t * n:(t + 1) * n], b_q) for t in range(f)])
    k_block = np.concatenate([ca_num.mean_pool(k[t * n:(t + 1) * n], b_kv) for t in range(i * f)])
    k_frame = ca_num.mean_pool(k_block, bpf)[: (i - 1) * f]
    views = ca_sel.CompressedViews(q_block=q_block, k_block=k_block, k_frame=k_frame,
                                   blocks_per_frame=bpf)
    cfg = ca.SelectionConfig(topk_frames=topk, block_budget_mode=mode)
    current = f * bpf
    total = current if i == 1 else ca.chunk_block_budget(s_i, i, lay)
    past_budget = max(0, total - current)
    bits = np.zeros((qb.shape[0], kb.shape[0]), dtype=bool)
    bits[:, (i - 1) * f * bpf:] = True
    for r in range(qb.shape[0]):
        p = ca.frame_scores(views, r)
        fset = ca.select_frames(p, cfg, i, lay)
        sel = ca.select_blocks(views, r, fset, past_budget, cfg)
        for tau, j in sel.blocks:
            bits[r, tau * bpf + j] = True
    out = np.empty_like(q)
    for r in range(qb.shape[0]):
        keys = np.concatenate([np.arange(*kb[c]) for c in np.flatnonzero(bits[r])])
        s0, s1 = qb[r]
        out[s0:s1] = ca.dense_attention(q[s0:s1], k[keys], v[keys])
    return views, bits, out, total < current


def framewise_fixtures():
    rows = []
    arrays = {}
    case = 0
    for name, f, n, b_q, b_kv, d, N in FW_LAYOUTS:
        for i in sorted({1, 2, N}):
            for s_i, topk, mode in ((0.0, 99, "global"), (0.4, 2, "global"), (0.55, 3, "per-frame"),
                                    (0.3, 1, "per-frame"), (0.8, 6, "global")):
                seed = 5000 + case
                q, k, v = synthetic_qkv(seed, f * n, i * f * n, d)
                q, k, v = q[0], k[0], v[0]
                views, bits, out, clamped = framewise_reference(q, k, v, i, s_i, f, n, b_q, b_kv,
                                                                topk, mode, N)
                arrays[f"bits{case}"] = np.packbits(bits, axis=1)
                arrays[f"qb{case}"] = views.q_block
                arrays[f"kb{case}"] = views.k_block
                arrays[f"kf{case}"] = views.k_frame
                if n < 1000:
                    arrays[f"out{case}"] = out
                rows.append(dict(case=case, layout=name, f=f, n=n, b_q=b_q, b_kv=b_kv, d=d, N=N,
                                 i=i, s_i=s_i, topk=topk, mode=mode, seed=seed,
                                 nq=bits.shape[0], nk=bits.shape[1], clamped=bool(clamped),
                                 has_out=bool(n < 1000)))
                case += 1
    np.savez_compressed(os.path.join(HERE, "hsa_framewise.npz"), **arrays)
    with open(os.path.join(HERE, "hsa_framewise.json"), "w") as fh:
        json.dump(rows, fh, indent=0)


def attention_fixtures():
    """block_sparse_attention on random ragged shapes (contiguous tiling)."""
    rng = np.random.default_rng(20261017)
    rows = []
    arrays = {}
    for case in range(24):
        d = int(rng.choice([16, 64, 128]))
        nrows = int(rng.integers(1, 420))
        keys = int(rng.integers(1, 700))
        b_q = int(rng.choice([16, 32, 48, 64, 128]))
        b_kv = int(rng.choice([16, 32, 48, 64, 128, 205]))
        seed = 9000 + case
        q, k, v = synthetic_qkv(seed, nrows, keys, d)
        q, k, v = q[0], k[0], v[0]
        n_q, n_k = -(-nrows // b_q), -(-keys // b_kv)
        bits = rng.random((n_q, n_k)) < rng.uniform(0.1, 1.0)
        bits[~bits.any(axis=1), 0] = True
        lay = _layout(1, keys, b_q, b_kv, d, 1)
        out, stats = ca.block_sparse_attention(q, k, v, ca.BlockMask(bits), lay)
        arrays[f"bits{case}"] = np.packbits(bits, axis=1)
        arrays[f"out{case}"] = out
        rows.append(dict(case=case, d=d, rows=nrows, keys=keys, b_q=b_q, b_kv=b_kv, seed=seed,
                         nq=n_q, nk=n_k, active=stats.active_tiles, total=stats.total_tiles,
                         flops=stats.flop_estimate))
    np.savez_compressed(os.path.join(HERE, "attention.npz"), **arrays)
    with open(os.path.join(HERE, "attention.json"), "w") as fh:
        json.dump(rows, fh, indent=0)


def plan_fixtures():
    cases = [
        dict(st=0.9, sb=0.98, N=7, T=4, f=3, n=512, b=64, d=64),      # stock golden
        dict(st=0.9, sb=0.98, N=7, T=4, f=3, n=1560, b=64, d=128),    # config 2
        dict(st=0.9, sb=0.98, N=21, T=4, f=3, n=1560, b=64, d=128),   # config 3
        dict(st=0.5, sb=0.9, N=3, T=4, f=2, n=256, b=64, d=64),       # config 1
        dict(st=0.3, sb=0.5, N=3, T=4, f=2, n=256, b=64, d=64),
        dict(st=0.9, sb=0.98, N=3, T=4, f=2, n=256, b=64, d=64),
        dict(st=0.2, sb=0.3, N=8, T=4, f=2, n=64, b=32, d=16),
        dict(st=0.75, sb=0.95, N=8, T=4, f=2, n=128, b=64, d=16, redistribute=True),
        dict(st=0.75, sb=0.95, N=8, T=4, f=2, n=128, b=64, d=16),
        dict(st=0.5, sb=0.9, N=7, T=4, f=3, n=512, b=64, d=64, first_chunk_dense=False),
        dict(st=0.0, sb=0.5, N=1, T=4, f=1, n=64, b=64, d=8),
        dict(st=0.6, sb=0.8, N=64, T=3, f=3, n=1560, b=64, d=128, redistribute=True),
    ]
    rng = np.random.default_rng(99)
    for _ in range(40):
        N = int(rng.integers(1, 40))
        st = float(rng.uniform(0.0, 0.9))
        sb = float(min(1.0, st + rng.uniform(0.0, 0.3)))
        cases.append(dict(st=st, sb=sb, N=N, T=int(rng.integers(1, 9)), f=int(rng.integers(1, 4)),
                          n=int(rng.choice([64, 128, 1536, 1560])), b=64, d=int(rng.choice([64, 128])),
                          redistribute=bool(rng.integers(0, 2)),
                          first_chunk_dense=bool(rng.integers(0, 4) > 0)))
    out = []
    for c in cases:
        lay = _layout(c["f"], c["n"], c["b"], c["b"], c["d"], c["N"])
        p = ca.allocate(c["st"], c["sb"], c["N"], c["T"], lay,
                        first_chunk_dense=c.get("first_chunk_dense", True),
                        redistribute=c.get("redistribute", False))
        out.append(dict(case=c, alpha=list(p.alpha), beta=p.beta, s=list(p.s),
                        budgets=list(p.budgets), clamped=list(p.clamped),
                        achieved=p.achieved_flops_ratio))
    with open(os.path.join(HERE, "plans.json"), "w") as fh:
        json.dump(out, fh, indent=0)


def report_fixtures():
    """The reference CLI's report formats (cli.py:71-78, 125-178, 220-266):
    a bench CSV (deterministic columns compared), mask-dump PGMs and selection
    traces, all written by running the reference's own CLI entry points."""
    import tempfile
    from chunkattn import cli as ca_cli
    with tempfile.TemporaryDirectory() as td:
        out = os.path.join(td, "bench.csv")
        assert ca_cli.main(["bench", "--seq", "512", "--dim", "64", "--block", "64",
                            "--densities", "0.5,0.25", "--repeats", "3", "--seed", "5",
                            "--threads", "1", "--out", out]) == 0
        with open(out, encoding="utf-8", newline="") as fh:
            lines = fh.read().split("\r\n")
        # timing columns (wall_time_*, speedup) and max_abs_err vary run to run: blank them
        kept = [lines[0], lines[1]]
        for ln in lines[2:]:
            if ln:
                kept.append(",".join(ln.split(",")[:10]))
        with open(os.path.join(HERE, "report_bench.csv"), "w", encoding="utf-8") as fh:
            fh.write("\n".join(kept) + "\n")
        cases = [("global", 0.6, 7), ("per-frame", 0.7, 5)]
        for mode, sparsity, chunk in cases:
            pgm = os.path.join(HERE, f"report_mask_{mode}.pgm")
            tr = os.path.join(HERE, f"report_trace_{mode}.json")
            assert ca_cli.main(["mask-dump", "--frames", "3", "--tokens", "128", "--block", "64",
                                "--dim", "32", "--chunks", "7", "--chunk", str(chunk),
                                "--sparsity", str(sparsity), "--topk", "3", "--mode", mode,
                                "--seed", "11", "--out", pgm, "--trace", tr]) == 0


if __name__ == "__main__":
    pool_fixtures()
    topk_fixtures()
    plan_fixtures()
    attention_fixtures()
    hsa_fixtures()
    framewise_fixtures()
    report_fixtures()
    for fn in sorted(os.listdir(HERE)):
        print(fn, os.path.getsize(os.path.join(HERE, fn)))
