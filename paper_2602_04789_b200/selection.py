"""Two-stage (frame -> block) mask selection, reference-compatible API
(chunkattn selection.py:1-249).

Names, argument order, return types and exceptions follow the reference.
All arithmetic on the data runs on the GPU: pooling (csrc/pool.cuh), frame
and block scoring + top-k (csrc/select.cuh), tile planning (csrc/tiles.cuh)
and attention (csrc/attn_sm100_v3.cuh, csrc/attn_sm100_v5.cuh).  Host code only validates arguments and
formats results (sorting a handful of selected indices, building the bool
mask for callers that ask for it).

Extension: ``framewise=True`` enables the frame-local ragged tiling needed
when the block does not divide the tokens-per-frame (n = 1560, b = 64;
DESIGN.md "Framewise ragged extension").  Without it, misaligned layouts raise
the reference's ValueError (selection.py:88-92).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _convert as C
from . import device as D
from .attention import _Timer, effective_flops
from .layout import AttnStats, BlockMask, ChunkLayout, as_layout
from .planner import chunk_block_budget

_BUDGET_MODES = ("global", "per-frame")
_CHUNK_POLICIES = ("dense-within-chunk",)


@dataclass(frozen=True)
class SelectionConfig:
    """selection.py:39-51."""

    topk_frames: int = 6
    current_chunk_policy: str = "dense-within-chunk"
    block_budget_mode: str = "global"

    def __post_init__(self):
        if self.topk_frames < 0:
            raise ValueError(f"topk_frames must be >= 0, got {self.topk_frames}")
        if self.current_chunk_policy not in _CHUNK_POLICIES:
            raise ValueError(f"unknown current_chunk_policy {self.current_chunk_policy!r}")
        if self.block_budget_mode not in _BUDGET_MODES:
            raise ValueError(f"unknown block_budget_mode {self.block_budget_mode!r}")


@dataclass(frozen=True)
class CompressedViews:
    """Pooled summaries (selection.py:54-70); arrays are numpy or CUDA tensors."""

    q_block: object
    k_block: object
    k_frame: object
    blocks_per_frame: int

    @property
    def past_frames(self) -> int:
        return self.k_frame.shape[0]


@dataclass(frozen=True)
class QueryBlockSelection:
    """selection.py:73-85."""

    frames: tuple
    blocks: tuple
    budget_used: int
    block_scores: tuple = ()


def _require_frame_aligned(layout: ChunkLayout) -> None:
    if layout.n % layout.b_q or layout.n % layout.b_kv:
        raise ValueError(
            f"selection needs b_q and b_kv to divide n: "
            f"n={layout.n}, b_q={layout.b_q}, b_kv={layout.b_kv}")


def tilings(layout: ChunkLayout, chunk_index: int, framewise: bool):
    """Query/key block tilings of one hot-path call (identical when aligned)."""
    lq = layout.chunk_tokens
    lk = chunk_index * lq
    qt = D.TilingSpec(lq, layout.n if framewise else lq, layout.b_q)
    kt = D.TilingSpec(lk, layout.n if framewise else lk, layout.b_kv)
    return qt, kt


def _dev_tensor(a):
    if torch.is_tensor(a):
        return a.to(C.device())
    return torch.from_numpy(np.ascontiguousarray(a)).to(C.device())


def compress(q, k, chunk_index: int, layout: ChunkLayout, *, framewise: bool = False
             ) -> CompressedViews:
    """Mean-pool q and k into block summaries plus past frame summaries (selection.py:95-114)."""
    layout = as_layout(layout)
    if not framewise:
        _require_frame_aligned(layout)
    layout.check_chunk(chunk_index)
    if tuple(q.shape) != (layout.chunk_tokens, layout.d):
        raise ValueError(f"q shape {tuple(q.shape)}, expected ({layout.chunk_tokens}, {layout.d})")
    ctx = layout.context_tokens(chunk_index)
    if tuple(k.shape) != (ctx, layout.d):
        raise ValueError(f"k shape {tuple(k.shape)}, expected ({ctx}, {layout.d})")
    qd = _dev_tensor(q).float()
    kd = _dev_tensor(k).float()
    qt, kt = tilings(layout, chunk_index, framewise)
    bpf = layout.frame_kv_blocks
    past = (chunk_index - 1) * layout.f
    qb, kb, kf = D.compress(qd[None], kd[None], qt, kt, bpf, past)
    return CompressedViews(C.like_input(qb[0], q), C.like_input(kb[0], q), C.like_input(kf[0], q),
                           bpf)


def frame_scores(views: CompressedViews, r: int):
    """Raw fp64 retrieval logits of query block r vs every past frame (selection.py:117-122)."""
    nq = views.q_block.shape[0]
    if not 0 <= r < nq:
        raise ValueError(f"query block {r} outside 0..{nq - 1}")
    kf = _dev_tensor(views.k_frame).float()
    if kf.shape[0] == 0:
        return C.like_input(torch.zeros(0, dtype=torch.float64, device=C.device()), views.q_block)
    qv = _dev_tensor(views.q_block).float()[r]
    return C.like_input(D.rowdot(kf, qv), views.q_block)


def select_frames(p, cfg: SelectionConfig, chunk_index: int, layout: ChunkLayout) -> np.ndarray:
    """Top-k past frames by score plus every current frame, sorted (selection.py:125-134)."""
    past = (chunk_index - 1) * layout.f
    pd = _dev_tensor(p).double()
    if tuple(pd.shape) != (past,):
        raise ValueError(f"expected {past} past-frame scores, got shape {tuple(pd.shape)}")
    picked = D.topk(pd, cfg.topk_frames).cpu().numpy().astype(np.int64) if past else \
        np.zeros(0, np.int64)
    current = np.arange(past, past + layout.f)
    return np.sort(np.concatenate([picked, current]))


def _topk_host(scores_dev: torch.Tensor, k: int) -> np.ndarray:
    return D.topk(scores_dev, k).cpu().numpy().astype(np.int64)


def select_blocks(views: CompressedViews, r: int, frames, budget: int,
                  cfg: SelectionConfig) -> QueryBlockSelection:
    """Spend ``budget`` blocks inside the retrieved past frames (selection.py:137-175)."""
    if budget < 0:
        raise ValueError(f"budget must be >= 0, got {budget}")
    past = sorted(int(t) for t in np.asarray(frames).ravel() if t < views.past_frames)
    if not past or budget == 0:
        return QueryBlockSelection(frames=tuple(past), blocks=(), budget_used=0)
    bpf = views.blocks_per_frame
    cand = np.concatenate([np.arange(t * bpf, (t + 1) * bpf) for t in past])
    kb = _dev_tensor(views.k_block).float()
    qv = _dev_tensor(views.q_block).float()[r]
    scores = D.rowdot(kb[torch.from_numpy(cand).to(kb.device)], qv)
    if cfg.block_budget_mode == "global":
        order = np.sort(_topk_host(scores, budget))
    else:
        per = -(-budget // len(past))
        picks: list[int] = []
        for fi in range(len(past)):
            loc = _topk_host(scores[fi * bpf:(fi + 1) * bpf], per)
            picks.extend(int(fi * bpf + j) for j in loc)
        order = np.sort(np.asarray(picks[:budget], dtype=np.int64))
    sc = scores.cpu().numpy()
    chosen = cand[order]
    blocks = tuple((int(c) // bpf, int(c) % bpf) for c in chosen)
    return QueryBlockSelection(frames=tuple(past), blocks=blocks, budget_used=len(blocks),
                               block_scores=tuple(float(s) for s in sc[order]))


def build_mask(selections, chunk_index: int, layout: ChunkLayout, *, framewise: bool = False
               ) -> BlockMask:
    """Current chunk dense, past blocks as selected (selection.py:178-193)."""
    layout = as_layout(layout)
    if not framewise:
        _require_frame_aligned(layout)
    n_q = layout.framewise_q_blocks() if framewise else layout.q_blocks
    if len(selections) != n_q:
        raise ValueError(f"{len(selections)} selections for {n_q} query blocks")
    bpf = layout.frame_kv_blocks
    n_k = layout.total_blocks(chunk_index)
    past_cols = (chunk_index - 1) * layout.f * bpf
    bits = np.zeros((n_q, n_k), dtype=bool)
    bits[:, past_cols:] = True
    for r, sel in enumerate(selections):
        for tau, j in sel.blocks:
            bits[r, tau * bpf + j] = True
    return BlockMask(bits)


def mask_from_lists(blocks: np.ndarray, count: np.ndarray, n_k: int, past_cols: int) -> np.ndarray:
    """Bool grid [nqb, n_k] from per-row block lists + the dense current chunk."""
    nqb = count.shape[0]
    bits = np.zeros((nqb, n_k), dtype=bool)
    bits[:, past_cols:] = True
    rows = np.repeat(np.arange(nqb), count)
    cols = np.concatenate([blocks[r, :count[r]] for r in range(nqb)]) if nqb else np.zeros(0, int)
    bits[rows, cols.astype(np.int64)] = True
    return bits


def hsa_attention(q, k, v, chunk_index: int, s_i: float, cfg: SelectionConfig,
                  layout: ChunkLayout, threads: int = 1, *, framewise: bool = False):
    """Compress, retrieve frames, pick blocks, run the sparse kernel (selection.py:196-231).

    Returns (out, AttnStats, BlockMask) like the reference.  select_time and
    wall_time are GPU times of the selection stages and of the attention
    kernel.  fp32 inputs are pooled in fp32 (bit-exact selection) and cast to
    bf16 for the tensor-core attention.
    """
    layout = as_layout(layout)
    if not 0.0 <= s_i < 1.0:
        raise ValueError(f"s_i must lie in [0, 1), got {s_i}")
    if not framewise:
        _require_frame_aligned(layout)
    layout.check_chunk(chunk_index)
    qd = C.as_matrix_dev(q, "q")
    kd = C.as_matrix_dev(k, "k")
    vd = C.as_matrix_dev(v, "v")
    if tuple(qd.shape) != (layout.chunk_tokens, layout.d):
        raise ValueError(f"q shape {tuple(qd.shape)}, expected ({layout.chunk_tokens}, {layout.d})")
    ctx = layout.context_tokens(chunk_index)
    if tuple(kd.shape) != (ctx, layout.d) or tuple(vd.shape) != (ctx, layout.d):
        raise ValueError(f"k/v shape {tuple(kd.shape)}/{tuple(vd.shape)}, expected ({ctx}, {layout.d})")
    qt, kt = tilings(layout, chunk_index, framewise)
    bpf = layout.frame_kv_blocks
    P = (chunk_index - 1) * layout.f
    current = layout.f * bpf
    dev = qd.device
    s_dev = torch.tensor([float(s_i)], dtype=torch.float64, device=dev)

    with _Timer() as t_sel:
        qb, kb, kf = D.compress(qd[None], kd[None], qt, kt, bpf, P)
        sel, tiles, _ = D.select_plan(qb, kb, kf, bpf, chunk_index, layout.f, cfg.topk_frames,
                                      cfg.block_budget_mode == "per-frame", s_dev, qt, kt,
                                      P * bpf)
    qh, kh, vh = C.to_bf16_heads(qd), C.to_bf16_heads(kd), C.to_bf16_heads(vd)
    with _Timer() as t_att:
        out = D.attention(qh, kh, vh, qt, tiles, P * layout.n, ctx, out_dtype=torch.float32,
                          scale=1.0 / math.sqrt(layout.d), qperm=tiles.qperm)
    count = sel.count[0].cpu().numpy()
    blocks = sel.blocks[0].cpu().numpy()
    budget = sel.budget.cpu().numpy()
    nqb, nkb = qt.count, kt.count
    bits = mask_from_lists(blocks, count, nkb, P * bpf)
    mask = BlockMask(bits)
    active = int(count.sum()) + nqb * current
    total = current if chunk_index == 1 else chunk_block_budget(s_i, chunk_index, layout)
    stats = AttnStats(
        active_tiles=active,
        total_tiles=nqb * nkb,
        flop_estimate=active * layout.b_q * layout.b_kv * layout.d * 2,
        wall_time=t_att.seconds(),
        select_time=t_sel.seconds(),
        budget_clamped=bool(total < current),
        effective_flops=effective_flops(bits, qt, kt, layout.d),
    )
    assert bool(budget[2]) == stats.budget_clamped or chunk_index == 1
    out = out[0, :, :layout.d]
    return C.like_input(out, q), stats, mask


def selection_trace(selections, frame_score_rows=None) -> list:
    """JSON-ready per-query-block record (selection.py:234-249)."""
    rows = []
    for r, sel in enumerate(selections):
        row = {
            "query_block": r,
            "frames": list(sel.frames),
            "blocks": [list(b) for b in sel.blocks],
            "block_scores": list(sel.block_scores),
            "budget_used": sel.budget_used,
        }
        if frame_score_rows is not None:
            row["frame_scores"] = [float(x) for x in frame_score_rows[r]]
        rows.append(row)
    return rows
