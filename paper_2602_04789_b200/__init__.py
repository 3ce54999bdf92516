"""B200-native (sm_100a) Light Forcing sparse-attention hot path.

Drop-in for the hot path of the reference package ``chunkattn`` 0.1.0
(/root/reference/pkg/src/chunkattn/__init__.py:61-106): same names, argument
order, return values and exceptions for pooling, hierarchical selection,
Chunk-Aware Growth planning, block-sparse / dense attention and the rollout
backend protocol.  Compute runs in hand-written CUDA kernels reached through
the C ABI in include/lfattn.h (library: _lib/liblfattn.so); there is no CPU
fallback.  Batched multi-head calls: ``HsaPipeline``.
"""

from .attention import block_sparse_attention, dense_attention
from .backends import BACKEND_KINDS, DenseBackend, FixedMaskBackend, HsaBackend
from .errors import DegenerateScheduleError, EmptyActiveSetError, ZeroActiveRowError
from .layout import AttnStats, BlockMask, ChunkLayout, ceil_div
from .numerics import TopKResult, as_matrix, mean_pool, stable_softmax_row, topk_indices
from .pipeline import HsaPipeline
from .rollout import HsaRollout, largest_remainder_split, matched_budget_settings
from .planner import (
    ChunkLengths,
    SparsityPlan,
    allocate,
    alpha_schedule,
    budget_for_chunk,
    chunk_block_budget,
    plan_from_json,
    plan_to_json,
    round_half_up,
    s_max_for_chunk,
    solve_beta,
    tv_bound,
)
from .selection import (
    CompressedViews,
    QueryBlockSelection,
    SelectionConfig,
    build_mask,
    compress,
    frame_scores,
    hsa_attention,
    select_blocks,
    select_frames,
    selection_trace,
)

__version__ = "0.1.0"

__all__ = [
    "AttnStats", "BACKEND_KINDS", "BlockMask", "ChunkLayout", "ChunkLengths", "CompressedViews",
    "DegenerateScheduleError", "DenseBackend", "EmptyActiveSetError", "FixedMaskBackend",
    "HsaBackend", "HsaPipeline", "QueryBlockSelection", "SelectionConfig", "SparsityPlan",
    "TopKResult", "ZeroActiveRowError", "allocate", "alpha_schedule", "as_matrix",
    "block_sparse_attention", "budget_for_chunk", "build_mask", "ceil_div", "chunk_block_budget",
    "compress", "dense_attention", "frame_scores", "hsa_attention", "mean_pool", "plan_from_json",
    "plan_to_json", "round_half_up", "s_max_for_chunk", "select_blocks", "select_frames",
    "selection_trace", "solve_beta", "stable_softmax_row", "topk_indices", "tv_bound",
    "HsaRollout", "largest_remainder_split", "matched_budget_settings",
]
