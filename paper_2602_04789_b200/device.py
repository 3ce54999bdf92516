"""Typed torch wrappers over the C ABI: one function per entry point.

Everything here takes/returns CUDA tensors and enqueues work on the current
stream; nothing synchronises.  The reference-compatible API (selection.py,
attention.py, planner.py, numerics.py in this package) is built on these.
"""

from __future__ import annotations

import contextlib
import ctypes
import math
import os
from dataclasses import dataclass

import torch

from . import _lib as L

SEG_KEYS = 64
TILE_ROWS = 128  # query rows per tcgen05 tile (one TMEM lane each)


def plan_rows() -> int:
    """Rows per tile plan: 256 (a pair of 128-row query tiles) unless the legacy kernel is selected."""
    return int(L.lib().lf_plan_tile_rows())


_qmode_req = -1


def set_qtile_mode(mode: int) -> None:
    """Query-tile geometry for later plans and attention calls: 1 = block-aligned
    (two consecutive query blocks per tensor-core tile), 2 = two query blocks
    paired by selection overlap (pair_qblocks), 0 = 128-row tiles, -1 =
    automatic (LF_QTILE env when set, else chosen per step by the rollout /
    pipeline)."""
    global _qmode_req
    _qmode_req = -1 if mode < 0 else int(mode)
    L.lib().lf_set_qtile_mode(_qmode_req)


BLOCK_TILES_MIN_PAST = 16  # csrc/lfattn.cu kBlockTilesMinPast
PAIRED_MIN_PAST = 80       # csrc/lfattn.cu kPairedMinPast


def auto_qtile_mode(s_host, chunk: int, f: int, bpf: int, topk_frames: int) -> int:
    """Geometry for one step from the host s_i (mirrors auto_qmode in lfattn.cu):
    block-aligned tiles when the estimated past blocks per query block is >= 16
    and below all past blocks (a fully selected past gives every block one list),
    paired by selection overlap from 80 past blocks on."""
    P = (chunk - 1) * f
    if P <= 0 or s_host is None or not (0.0 <= float(s_host) < 1.0):
        return 0
    cur = f * bpf
    past = min(int((1.0 - float(s_host)) * chunk * cur + 0.5) - cur, min(topk_frames, P) * bpf)
    if not BLOCK_TILES_MIN_PAST <= past < P * bpf:
        return 0
    return 2 if past >= PAIRED_MIN_PAST else 1


@contextlib.contextmanager
def qtile_scope(mode: int):
    """Plans and attention calls inside use query-tile geometry `mode` (an
    explicit LF_QTILE environment setting still wins)."""
    if _qmode_req >= 0 or os.environ.get("LF_QTILE"):
        yield  # an explicit choice wins
        return
    L.lib().lf_set_qtile_mode(int(mode))
    try:
        yield
    finally:
        L.lib().lf_set_qtile_mode(-1)


def qtile_mode(qt) -> int:
    """The query-tile geometry the library uses for this query tiling."""
    return int(L.lib().lf_qtile_mode(qt.abi()))


def qtile_rows(qt, mode: int, t: int):
    """Rows [x0, x1) of query tile t (csrc/common.cuh qtile_rows; geometries 0, 1)."""
    if mode == 2:
        raise ValueError("paired query tiles have no row range: use the pairing (qperm)")
    if mode:
        nb = qt.count
        x0 = qt.block_start(2 * t)
        x1 = qt.block_start(2 * t + 2) if 2 * t + 2 < nb else qt.total
        return x0, x1
    return t * TILE_ROWS, min(t * TILE_ROWS + TILE_ROWS, qt.total)


def _dev():
    return torch.device("cuda", torch.cuda.current_device())


@dataclass(frozen=True)
class TilingSpec:
    """A token axis cut into blocks; period = n (framewise) or total (contiguous)."""

    total: int
    period: int
    block: int

    @property
    def per_period(self) -> int:
        return -(-self.period // self.block)

    @property
    def count(self) -> int:
        full, rem = divmod(self.total, self.period)
        return full * self.per_period + -(-rem // self.block)

    def block_of(self, row: int) -> int:
        t = row // self.period
        return t * self.per_period + (row - t * self.period) // self.block

    def bounds(self):
        """[count, 2] int64 tensor of (start, end) for every block (host)."""
        import numpy as np
        g = np.arange(self.count, dtype=np.int64)
        t, j = np.divmod(g, self.per_period)
        s = t * self.period + j * self.block
        e = np.minimum(np.minimum(s + self.block, t * self.period + self.period), self.total)
        return np.stack([s, e], axis=1)

    def block_start(self, g: int) -> int:
        t, j = divmod(g, self.per_period)
        return t * self.period + j * self.block

    def max_blocks_per_tile(self, rows: int = TILE_ROWS) -> int:
        worst = 0
        for q0 in range(0, self.total, rows):
            q1 = min(q0 + rows, self.total)
            worst = max(worst, self.block_of(q1 - 1) - self.block_of(q0) + 1)
        return worst

    def abi(self) -> L.LfTiling:
        return L.tiling(self.total, self.period, self.block)


def pool_blocks(x: torch.Tensor, spec: TilingSpec, max_blocks: int = -1) -> torch.Tensor:
    """Block means of x [H, L, d] (bf16 or fp32) -> fp32 [H, nblocks, d]."""
    lib = L.lib()
    x3 = x if x.dim() == 3 else x.unsqueeze(0)
    nb = spec.count if max_blocks < 0 else min(max_blocks, spec.count)
    out = torch.empty((x3.shape[0], nb, x3.shape[2]), device=x.device, dtype=torch.float32)
    m = L.mat(x3)
    L.check(lib.lf_pool_blocks(ctypes.byref(m), spec.abi(), int(max_blocks), out.data_ptr(),
                               nb * x3.shape[2], L.stream_ptr()))
    return out if x.dim() == 3 else out[0]


def compress(q: torch.Tensor, k: torch.Tensor, qt: TilingSpec, kt: TilingSpec, bpf: int,
             past_frames: int):
    """q_block, k_block, k_frame for [H, L, d] inputs (selection.py:95-114)."""
    lib = L.lib()
    H, d = q.shape[0], q.shape[2]
    q_block = torch.empty((H, qt.count, d), device=q.device, dtype=torch.float32)
    k_block = torch.empty((H, kt.count, d), device=q.device, dtype=torch.float32)
    k_frame = torch.empty((H, max(past_frames, 0), d), device=q.device, dtype=torch.float32)
    mq, mk = L.mat(q), L.mat(k)
    L.check(lib.lf_compress(ctypes.byref(mq), ctypes.byref(mk), qt.abi(), kt.abi(), int(bpf),
                            int(past_frames), q_block.data_ptr(), k_block.data_ptr(),
                            k_frame.data_ptr() if past_frames > 0 else None, L.stream_ptr()))
    return q_block, k_block, k_frame


@dataclass
class Selections:
    blocks: torch.Tensor     # [H, nqb, cap] int32 ascending absolute past block ids
    count: torch.Tensor      # [H, nqb] int32
    frames: torch.Tensor     # [H, nqb, frame_cap] int32 (-1 padded)
    budget: torch.Tensor     # [3] int32: total, past budget, clamped
    scores: torch.Tensor | None = None
    fscores: torch.Tensor | None = None


def select(q_block, k_block, k_frame, bpf: int, chunk: int, f: int, topk: int, per_frame: bool,
           s_i, want_scores: bool = False) -> Selections:
    """Frame top-k + block top-budget for every (head, query block).

    k_block / k_frame may be capacity-sized caches [H, cap, d] (only the
    first past blocks / frames are read); their head strides are passed on.
    """
    lib = L.lib()
    H, nqb, d = q_block.shape
    nkb = k_block.shape[1]
    P = (chunk - 1) * f
    kf = min(topk, P)
    cap = max(1, kf * bpf)
    frame_cap = max(1, kf)
    dev = q_block.device
    if not torch.is_tensor(s_i):
        s_i = torch.tensor([float(s_i)], dtype=torch.float64, device=dev)
    blocks = torch.empty((H, nqb, cap), dtype=torch.int32, device=dev)
    count = torch.empty((H, nqb), dtype=torch.int32, device=dev)
    frames = torch.empty((H, nqb, frame_cap), dtype=torch.int32, device=dev)
    budget = torch.empty(4, dtype=torch.int32, device=dev)  # all four written by the kernel
    scores = torch.empty((H, nqb, cap), dtype=torch.float64, device=dev) if want_scores else None
    fscores = torch.empty((H, nqb, max(P, 1)), dtype=torch.float64, device=dev) if want_scores else None
    for t in (q_block, k_block, k_frame):
        assert t.stride(2) == 1 and t.stride(1) == d, "summaries must have contiguous rows"
    L.check(lib.lf_select_strided(q_block.data_ptr(), k_block.data_ptr(), k_block.stride(0),
                                  k_frame.data_ptr() if P > 0 else None,
                                  k_frame.stride(0) if P > 0 else 0, H, nqb, nkb, d, int(bpf),
                                  int(chunk), int(f), int(topk), 1 if per_frame else 0,
                                  s_i.data_ptr(), cap, frame_cap, blocks.data_ptr(),
                                  count.data_ptr(), frames.data_ptr(), L.ptr(scores),
                                  L.ptr(fscores), budget.data_ptr(), L.stream_ptr()))
    return Selections(blocks, count, frames, budget, scores, fscores)


def select_fallbacks(reset: bool = False) -> tuple[int, int, int, int]:
    """(frame lists, block lists) the fp32 screen did not decide, then (frame,
    block) lists of those completed from exact scores of their ambiguous items
    only; summed over every selection launch since the last reset (device-wide
    counters; synchronous)."""
    out = (ctypes.c_uint64 * 4)()
    L.check(L.lib().lf_select_fallbacks(ctypes.cast(out, ctypes.c_void_p), 1 if reset else 0))
    return tuple(int(v) for v in out)


@dataclass
class CagPlan:
    alpha: torch.Tensor
    s: torch.Tensor
    budgets: torch.Tensor
    clamped: torch.Tensor
    scalars: torch.Tensor   # beta, achieved
    status: torch.Tensor


def cag_plan(s_target, s_base, N, T, f, n, b_kv, d, first_chunk_dense=True,
             redistribute=False) -> CagPlan:
    lib = L.lib()
    dev = _dev()
    p = CagPlan(torch.empty(N, dtype=torch.float64, device=dev),
                torch.empty(N, dtype=torch.float64, device=dev),
                torch.empty(N, dtype=torch.int32, device=dev),
                torch.empty(N, dtype=torch.int32, device=dev),
                torch.empty(2, dtype=torch.float64, device=dev),
                torch.zeros(1, dtype=torch.int32, device=dev))
    L.check(lib.lf_cag_plan(float(s_target), float(s_base), int(N), int(T), int(f), int(n),
                            int(b_kv), int(d), int(bool(first_chunk_dense)), int(bool(redistribute)),
                            p.alpha.data_ptr(), p.s.data_ptr(), p.budgets.data_ptr(),
                            p.clamped.data_ptr(), p.scalars.data_ptr(), p.status.data_ptr(),
                            L.stream_ptr()))
    return p


@dataclass
class TilePlan:
    segs: torch.Tensor       # [H, ntiles, seg_cap, 4] int32
    seg_count: torch.Tensor  # [H, ntiles] int32
    seg_cap: int
    qperm: torch.Tensor | None = None  # geometry 2: [H, 2 * n_qtiles] query-block pairing


def pair_qblocks(blocks, count, list_blocks: int) -> torch.Tensor:
    """Geometry-2 pairing of each head's query blocks by selection overlap
    (lf_pair_qblocks): int32 [H, 2 * ceil(nqb / 2)], -1 = empty half."""
    lib = L.lib()
    H, nqb, cap = blocks.shape
    qperm = torch.empty((H, 2 * ((nqb + 1) // 2)), dtype=torch.int32, device=blocks.device)
    L.check(lib.lf_pair_qblocks(blocks.data_ptr(), count.data_ptr(), H, nqb, cap,
                                int(list_blocks), qperm.data_ptr(), L.stream_ptr()))
    return qperm


def plan_tiles(blocks, count, qt: TilingSpec, kt: TilingSpec, list_blocks: int,
               seg_cap: int | None = None, qperm: torch.Tensor | None = None) -> TilePlan:
    lib = L.lib()
    H, nqb, cap = blocks.shape
    rows = plan_rows()
    ntiles = int(lib.lf_plan_tile_count(qt.abi()))
    mq = 4 if qtile_mode(qt) else qt.max_blocks_per_tile(rows)
    pieces = -(-kt.block // SEG_KEYS)
    if seg_cap is None:
        seg_cap = max(1, min(mq * cap * pieces, max(list_blocks, 0) * pieces)
                      + (3 if rows > TILE_ROWS else 0))
    dev = blocks.device
    segs = torch.empty((H, ntiles, seg_cap, 4), dtype=torch.int32, device=dev)
    seg_count = torch.empty((H, ntiles), dtype=torch.int32, device=dev)
    L.check(lib.lf_plan_tiles_paired(blocks.data_ptr(), count.data_ptr(), H, nqb, cap, qt.abi(),
                                     kt.abi(), int(list_blocks), int(seg_cap), segs.data_ptr(),
                                     seg_count.data_ptr(), L.ptr(qperm), L.stream_ptr()))
    return TilePlan(segs, seg_count, seg_cap)


def select_plan(q_block, k_block, k_frame, bpf: int, chunk: int, f: int, topk: int,
                per_frame: bool, s_i, qt: TilingSpec, kt: TilingSpec, list_blocks: int,
                want_margin: bool = False, want_frames: bool = True):
    """select() + plan_tiles() of one step (lf_select_plan).  Returns
    (Selections, TilePlan, margin) with margin = [H, nqb, 2] fp64 top-k margin
    certificate (frames, blocks) or None.  want_frames=False: Selections.frames
    is None and a step whose past budget is 0 skips the frame ranking (it
    cannot change the blocks)."""
    lib = L.lib()
    H, nqb, d = q_block.shape
    nkb = k_block.shape[1]
    P = (chunk - 1) * f
    kf = min(topk, P)
    cap = max(1, kf * bpf)
    frame_cap = max(1, kf)
    dev = q_block.device
    if not torch.is_tensor(s_i):
        s_i = torch.tensor([float(s_i)], dtype=torch.float64, device=dev)
    for t in (q_block, k_block, k_frame):
        assert t.stride(2) == 1 and t.stride(1) == d, "summaries must have contiguous rows"
    blocks = torch.empty((H, nqb, cap), dtype=torch.int32, device=dev)
    count = torch.empty((H, nqb), dtype=torch.int32, device=dev)
    frames = (torch.empty((H, nqb, frame_cap), dtype=torch.int32, device=dev)
              if want_frames else None)
    budget = torch.empty(4, dtype=torch.int32, device=dev)  # all four written by the kernel
    margin = torch.empty((H, nqb, 2), dtype=torch.float64, device=dev) if want_margin else None
    rows = plan_rows()
    ntiles = int(lib.lf_plan_tile_count(qt.abi()))
    mq = 4 if qtile_mode(qt) else qt.max_blocks_per_tile(rows)
    pieces = -(-kt.block // SEG_KEYS)
    seg_cap = max(1, min(mq * cap * pieces, max(list_blocks, 0) * pieces)
                  + (3 if rows > TILE_ROWS else 0))
    segs = torch.empty((H, ntiles, seg_cap, 4), dtype=torch.int32, device=dev)
    seg_count = torch.empty((H, ntiles), dtype=torch.int32, device=dev)
    qperm = (torch.empty((H, 2 * ((nqb + 1) // 2)), dtype=torch.int32, device=dev)
             if qtile_mode(qt) == 2 else None)
    L.check(lib.lf_select_plan(q_block.data_ptr(), k_block.data_ptr(), k_block.stride(0),
                               k_frame.data_ptr() if P > 0 else None,
                               k_frame.stride(0) if P > 0 else 0, H, nqb, nkb, d, int(bpf),
                               int(chunk), int(f), int(topk), 1 if per_frame else 0,
                               s_i.data_ptr(), cap, frame_cap, blocks.data_ptr(),
                               count.data_ptr(), L.ptr(frames), budget.data_ptr(),
                               L.ptr(margin), qt.abi(), kt.abi(), int(list_blocks), int(seg_cap),
                               segs.data_ptr(), seg_count.data_ptr(), L.ptr(qperm),
                               L.stream_ptr()))
    return (Selections(blocks, count, frames, budget),
            TilePlan(segs, seg_count, seg_cap, qperm), margin)


def past_tiles_hint(s_host, chunk: int, f: int, bpf: int, topk_frames: int,
                    qt: TilingSpec) -> int:
    """Estimated non-dense 128-key tiles per 256-row plan tile (the work hint of
    lf_attention_ex; mirrors past_tiles_estimate in lfattn.cu).  -1 if unknown."""
    P = (chunk - 1) * f
    if P <= 0:
        return 0
    if s_host is None or not (0.0 <= float(s_host) < 1.0):
        return -1
    cur = f * bpf
    past = int((1.0 - float(s_host)) * chunk * cur + 0.5) - cur
    if past <= 0:
        return 0
    past = min(past, min(topk_frames, P) * bpf)
    blocks = min(qt.max_blocks_per_tile(plan_rows()) * past, P * bpf)
    return (blocks + 1) // 2


def attention(q, k, v, qt: TilingSpec, tiles: TilePlan | None, dense_lo: int, dense_hi: int,
              out: torch.Tensor | None = None, out_dtype=torch.float32, scale: float | None = None,
              lse: torch.Tensor | None = None, err: torch.Tensor | None = None,
              kernel: int = L.LF_KERNEL_AUTO, past_tiles: int = -1,
              scratch: torch.Tensor | None = None,
              qperm: torch.Tensor | None = None) -> torch.Tensor:
    """Block-sparse flash attention over bf16 [H, L, d] (d in {64, 128}).

    kernel / past_tiles: lf_attention_ex's kernel choice and work hint.
    scratch: zero-filled uint8 buffer of lf_attention_scratch_bytes (the caller
    owns it, one launch in flight per buffer); None = the device's library scratch."""
    lib = L.lib()
    H, Lq, d = q.shape
    if out is None:
        out = torch.empty((H, Lq, d), dtype=out_dtype, device=q.device)
    odt = L.LF_F32 if out.dtype == torch.float32 else L.LF_BF16
    mq, mk, mv = L.mat(q), L.mat(k), L.mat(v)
    if scale is None:
        scale = 1.0 / math.sqrt(d)
    L.check(lib.lf_attention_paired(ctypes.byref(mq), ctypes.byref(mk), ctypes.byref(mv),
                                    qt.abi(), tiles.segs.data_ptr() if tiles else None,
                                    tiles.seg_count.data_ptr() if tiles else None,
                                    tiles.seg_cap if tiles else 0, int(dense_lo), int(dense_hi),
                                    float(scale), out.data_ptr(), odt, out.stride(1),
                                    out.stride(0), L.ptr(lse), L.ptr(err), int(kernel),
                                    int(past_tiles), L.ptr(scratch),
                                    scratch.numel() if scratch is not None else 0, L.ptr(qperm),
                                    L.stream_ptr()))
    return out


def rowdot(A: torch.Tensor, x: torch.Tensor) -> torch.Tensor:
    lib = L.lib()
    A = A.contiguous().float()
    x = x.contiguous().float()
    out = torch.empty(A.shape[0], dtype=torch.float64, device=A.device)
    L.check(lib.lf_rowdot(A.data_ptr(), A.shape[0], A.shape[1], x.data_ptr(), out.data_ptr(),
                          L.stream_ptr()))
    return out


def topk(scores: torch.Tensor, k: int) -> torch.Tensor:
    lib = L.lib()
    scores = scores.contiguous().double()
    n = scores.shape[0]
    kk = max(0, min(k, n))
    out = torch.empty(max(kk, 1), dtype=torch.int32, device=scores.device)
    L.check(lib.lf_topk(scores.data_ptr(), n, int(k), out.data_ptr(), L.stream_ptr()))
    return out[:kk]
