"""Attention backends behind the reference's rollout protocol (rollout.py:164-251).

Each backend exposes ``.name``, ``.layout``, ``.run(q, k, v, chunk_index)``,
``.stats_log`` and ``.mask_log`` (``HsaBackend`` also ``.plan``), so the
reference's ``denoise_step``/``rollout`` can drive them unchanged
(tests/test_gpu_backends.py runs ``chunkattn.rollout`` with them).  ``layout``
may be this package's ``ChunkLayout`` or the reference's: ``.layout`` keeps
the caller's object, so ``rollout()``'s ``backend.layout == layout`` check
(rollout.py:281-282) holds either way.  All
attention work runs on the GPU; inputs/outputs keep the caller's container
type (numpy in, numpy out).
"""

from __future__ import annotations

import numpy as np

from .attention import _Timer, block_sparse_attention, dense_attention
from .layout import AttnStats, BlockMask, ChunkLayout, as_layout, ceil_div, is_aligned
from .planner import SparsityPlan
from .selection import SelectionConfig, hsa_attention

BACKEND_KINDS = ("dense", "hsa", "fixed-mask")


class DenseBackend:
    """Full attention, stats synthesised at full density (rollout.py:164-188)."""

    name = "dense"

    def __init__(self, layout: ChunkLayout, threads: int = 1):
        self.layout = layout
        self.threads = threads
        self.stats_log: list[AttnStats] = []
        self.mask_log: list[BlockMask] = []

    def run(self, q, k, v, chunk_index: int):
        with _Timer() as tm:
            out = dense_attention(q, k, v)
        lay = self.layout
        n_q = ceil_div(q.shape[0], lay.b_q)
        n_k = ceil_div(k.shape[0], lay.b_kv)
        tiles = n_q * n_k
        self.stats_log.append(AttnStats(
            active_tiles=tiles, total_tiles=tiles,
            flop_estimate=tiles * lay.b_q * lay.b_kv * lay.d * 2,
            wall_time=tm.seconds(),
            effective_flops=4 * q.shape[0] * k.shape[0] * lay.d))
        self.mask_log.append(BlockMask.full(n_q, n_k))
        return out


class HsaBackend:
    """Two-stage selection driven by a sparsity plan (rollout.py:191-211)."""

    name = "hsa"

    def __init__(self, layout: ChunkLayout, plan: SparsityPlan, cfg: SelectionConfig | None = None,
                 threads: int = 1, *, framewise: bool | None = None):
        self.layout = layout
        self.plan = plan
        self.cfg = cfg or SelectionConfig()
        self.threads = threads
        self.framewise = (not is_aligned(layout)) if framewise is None else framewise
        self.stats_log: list[AttnStats] = []
        self.mask_log: list[BlockMask] = []

    def run(self, q, k, v, chunk_index: int):
        s_i = self.plan.s[chunk_index - 1]
        out, stats, mask = hsa_attention(q, k, v, chunk_index, s_i, self.cfg, self.layout,
                                         threads=self.threads, framewise=self.framewise)
        self.stats_log.append(stats)
        self.mask_log.append(mask)
        return out


class FixedMaskBackend:
    """Random per-row block budget, keyed by (seed, chunk) (rollout.py:214-251).

    The mask is drawn on the host exactly like the reference (it is data-free
    configuration, not compute); attention runs on the GPU.
    """

    name = "fixed-mask"

    def __init__(self, layout: ChunkLayout, budgets, seed: int, threads: int = 1):
        self.layout = layout
        self.budgets = tuple(int(b) for b in budgets)
        if any(b < 1 for b in self.budgets):
            raise ValueError(f"per-row budgets must be >= 1: {self.budgets}")
        self.seed = seed
        self.threads = threads
        self.stats_log: list[AttnStats] = []
        self.mask_log: list[BlockMask] = []

    def mask_for_chunk(self, chunk_index: int, n_q: int, n_k: int) -> BlockMask:
        budget = min(self.budgets[chunk_index - 1], n_k)
        rng = np.random.default_rng([self.seed, chunk_index])
        bits = np.zeros((n_q, n_k), dtype=bool)
        for r in range(n_q):
            bits[r, rng.choice(n_k, size=budget, replace=False)] = True
        return BlockMask(bits)

    def run(self, q, k, v, chunk_index: int):
        lay = self.layout
        n_q = ceil_div(q.shape[0], lay.b_q)
        n_k = ceil_div(k.shape[0], lay.b_kv)
        mask = self.mask_for_chunk(chunk_index, n_q, n_k)
        out, stats = block_sparse_attention(q, k, v, mask, lay, threads=self.threads)
        self.stats_log.append(stats)
        self.mask_log.append(mask)
        return out
