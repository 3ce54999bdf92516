"""Reference-compatible kernel API (attention.py:191-274 of chunkattn).

``block_sparse_attention`` and ``dense_attention`` keep the reference's names,
argument order, return values and exceptions; the work runs in the sm_100a
tcgen05 kernels (csrc/attn_sm100_v3.cuh / _v5.cuh) on bf16 copies of the operands with fp32
accumulation.  ``threads`` is accepted and ignored (the reference's
ThreadPoolExecutor has no GPU analogue; results never depended on it).
"""

from __future__ import annotations

import math

import numpy as np
import torch

from . import _convert as C
from . import device as D
from .errors import ZeroActiveRowError
from .layout import AttnStats, BlockMask, ChunkLayout, ceil_div


def _check_qkv(q, k, v):
    qd = C.as_matrix_dev(q, "q")
    kd = C.as_matrix_dev(k, "k")
    vd = C.as_matrix_dev(v, "v")
    if qd.shape[1] != kd.shape[1]:
        raise ValueError(f"q cols {qd.shape[1]} != k cols {kd.shape[1]}")
    if kd.shape[0] != vd.shape[0]:
        raise ValueError(f"k rows {kd.shape[0]} != v rows {vd.shape[0]}")
    return qd, kd, vd


class _Timer:
    def __init__(self):
        self.a = torch.cuda.Event(enable_timing=True)
        self.b = torch.cuda.Event(enable_timing=True)

    def __enter__(self):
        self.a.record()
        return self

    def __exit__(self, *exc):
        self.b.record()

    def seconds(self) -> float:
        self.b.synchronize()
        return self.a.elapsed_time(self.b) / 1e3


def mask_lists(bits: np.ndarray):
    """Per-row ascending active columns of a bool grid -> (blocks [1,nq,cap], count [1,nq])."""
    counts = bits.sum(axis=1).astype(np.int32)
    cap = max(1, int(counts.max()) if counts.size else 1)
    rows, cols = np.nonzero(bits)
    lst = np.full((bits.shape[0], cap), -1, dtype=np.int32)
    pos = np.arange(rows.size) - np.repeat(np.cumsum(counts) - counts, counts)
    lst[rows, pos] = cols
    return lst[None], counts[None]


def sparse_attention_device(qd, kd, vd, bits: np.ndarray, qt: D.TilingSpec, kt: D.TilingSpec,
                            d_true: int, out_dtype=torch.float32) -> torch.Tensor:
    """Run the tcgen05 kernel for one head given a host bool mask over (qt, kt) blocks."""
    dev = qd.device
    blocks, counts = mask_lists(bits)
    blocks_t = torch.from_numpy(blocks).to(dev)
    counts_t = torch.from_numpy(counts).to(dev)
    qperm = (D.pair_qblocks(blocks_t, counts_t, bits.shape[1]) if D.qtile_mode(qt) == 2
             else None)
    tiles = D.plan_tiles(blocks_t, counts_t, qt, kt, list_blocks=bits.shape[1], qperm=qperm)
    qb = C.to_bf16_heads(qd)
    kb = C.to_bf16_heads(kd)
    vb = C.to_bf16_heads(vd)
    out = D.attention(qb, kb, vb, qt, tiles, 0, 0, out_dtype=out_dtype,
                      scale=1.0 / math.sqrt(d_true), qperm=qperm)
    return out[0, :, :d_true]


def effective_flops(bits: np.ndarray, qt: D.TilingSpec, kt: D.TilingSpec, d: int) -> int:
    qb, kb = qt.bounds(), kt.bounds()
    rows = (qb[:, 1] - qb[:, 0]).astype(np.int64)
    cols = (kb[:, 1] - kb[:, 0]).astype(np.int64)
    return int(4 * d * (bits.astype(np.int64) * cols[None, :]).sum(axis=1).dot(rows))


def dense_attention(q, k, v, threads: int = 1):
    """Full softmax(q k^T / sqrt d) v (attention.py:212-226)."""
    qd, kd, vd = _check_qkv(q, k, v)
    d = qd.shape[1]
    qt = D.TilingSpec(qd.shape[0], qd.shape[0], 128)
    out = D.attention(C.to_bf16_heads(qd), C.to_bf16_heads(kd), C.to_bf16_heads(vd), qt, None, 0,
                      kd.shape[0], out_dtype=torch.float32, scale=1.0 / math.sqrt(d))
    return C.like_input(out[0, :, :d], q)


def block_sparse_attention(q, k, v, mask: BlockMask, layout: ChunkLayout, threads: int = 1):
    """Attention restricted to the active tiles of ``mask`` (attention.py:229-274)."""
    qd, kd, vd = _check_qkv(q, k, v)
    if qd.shape[1] != layout.d:
        raise ValueError(f"q cols {qd.shape[1]} != layout d {layout.d}")
    n_q = ceil_div(qd.shape[0], layout.b_q)
    n_k = ceil_div(kd.shape[0], layout.b_kv)
    if (mask.n_q, mask.n_k) != (n_q, n_k):
        raise ValueError(
            f"mask is {mask.n_q}x{mask.n_k}, expected {n_q}x{n_k} "
            f"for {qd.shape[0]} queries, {kd.shape[0]} keys")
    bits = mask.bits
    if not bits.any(axis=1).all():
        raise ZeroActiveRowError("query-block row has no active key blocks")
    qt = D.TilingSpec(qd.shape[0], qd.shape[0], layout.b_q)
    kt = D.TilingSpec(kd.shape[0], kd.shape[0], layout.b_kv)
    with _Timer() as tm:
        out = sparse_attention_device(qd, kd, vd, bits, qt, kt, layout.d)
    active = int(bits.sum())
    stats = AttnStats(
        active_tiles=active,
        total_tiles=n_q * n_k,
        flop_estimate=active * layout.b_q * layout.b_kv * layout.d * 2,
        wall_time=tm.seconds(),
        effective_flops=effective_flops(bits, qt, kt, layout.d),
    )
    return C.like_input(out, q), stats
