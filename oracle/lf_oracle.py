"""CPU oracle for the Light Forcing sparse-attention hot path.

TEST INFRASTRUCTURE ONLY.  Nothing under ``paper_2602_04789_b200/`` may import
this module; only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs use it, always as the checker or
the timed CPU baseline, never as the product path.

It restates, in NumPy, the reference package ``chunkattn`` 0.1.0
(``/root/reference/pkg/src/chunkattn``) for the functions on the hot path, with
the same precision rules (fp64 sequential pooling sums, fp64 selection dot
products through NumPy/OpenBLAS, fp32 QK^T -> fp64 softmax -> fp64 PV), and
adds the *framewise ragged extension* needed when the
block size does not divide the tokens-per-frame (n = 1560, b = 64):

  * every frame is tiled on its own: block j of frame t covers tokens
    [t*n + j*b, t*n + min((j+1)*b, n)), so a frame has ceil(n/b) blocks, the
    last one ragged (24 tokens at n = 1560);
  * query blocks are tiled the same way (f*ceil(n/b_q) per chunk);
  * k_frame = mean of the frame's block means (the reference composition
    selection.py:109-111 and PAPER.md Eq. 7), not the token mean.

For aligned layouts (n % b == 0) the extension is identical to the reference.

Parity pinning: ``tests/golden/make_golden.py`` imports the real reference
(available in the development container only) and records its outputs as
fixtures under ``tests/golden/``; ``tests/test_oracle_golden.py`` checks this
oracle against every fixture (bit-exact for pooling / indices / masks / plan
budgets, the reference's own tolerances for floats).
"""

from __future__ import annotations

import math
import os
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass

import numpy as np

KEY_SPAN = 512  # attention.py:29 (_KEY_SPAN), cap on a streamed key span


# ---------------------------------------------------------------------------
# geometry


def ceil_div(a: int, b: int) -> int:
    return -(-a // b)


@dataclass(frozen=True)
class Tiling:
    """Row tiling of a token axis into blocks.

    ``period`` is the length of one independently tiled run: ``n`` for the
    framewise extension, the whole axis length for the reference's contiguous
    tiling (attention.py:75-87).  Block ``g`` of run ``t`` starts at
    ``t*period + j*block`` and holds ``min(block, period - j*block)`` rows.
    """

    total: int
    period: int
    block: int

    @property
    def per_period(self) -> int:
        return ceil_div(self.period, self.block)

    @property
    def count(self) -> int:
        full, rem = divmod(self.total, self.period)
        return full * self.per_period + ceil_div(rem, self.block)

    def bounds(self, g: int) -> tuple[int, int]:
        t, j = divmod(g, self.per_period)
        s = t * self.period + j * self.block
        e = min(s + self.block, t * self.period + self.period, self.total)
        return s, e

    def all_bounds(self) -> np.ndarray:
        return np.array([self.bounds(g) for g in range(self.count)], dtype=np.int64).reshape(-1, 2)


def q_tiling(f, n, b_q, framewise):
    total = f * n
    return Tiling(total, n if framewise else total, b_q)


def k_tiling(i, f, n, b_kv, framewise):
    total = i * f * n
    return Tiling(total, n if framewise else total, b_kv)


# ---------------------------------------------------------------------------
# numerics (numerics.py)


def mean_pool_bounds(x: np.ndarray, bounds: np.ndarray) -> np.ndarray:
    """Group means with the reference's rounding (numerics.py:44-66).

    Sums run in float64 in row order (the reference's reshape/reduceat
    reductions accumulate sequentially along the pooled axis), are divided by
    the group size in float64 and rounded once to the input dtype.
    """
    x = np.asarray(x)
    lens = bounds[:, 1] - bounds[:, 0]
    out = np.empty((bounds.shape[0], x.shape[1]), dtype=np.float64)
    width = int(lens.max()) if lens.size else 0
    starts = bounds[:, 0]
    acc = x[starts].astype(np.float64)
    for j in range(1, width):
        live = lens > j
        acc[live] += x[starts[live] + j].astype(np.float64)
    out[:] = acc / lens[:, None].astype(np.float64)
    return out.astype(x.dtype, copy=False)


def mean_pool(x: np.ndarray, group: int) -> np.ndarray:
    """numerics.py:44-66 -- contiguous groups of ``group`` rows."""
    if group < 1:
        raise ValueError(f"pool size must be >= 1, got {group}")
    x = np.asarray(x)
    if x.ndim != 2 or x.shape[0] < 1:
        raise ValueError(f"expected non-empty 2-D input, got shape {x.shape}")
    return mean_pool_bounds(x, Tiling(x.shape[0], x.shape[0], group).all_bounds())


def topk_indices(scores: np.ndarray, k: int) -> np.ndarray:
    """numerics.py:91-104: k largest, ties to the lower index (stable sort of -s)."""
    if k < 0:
        raise ValueError(f"k must be >= 0, got {k}")
    scores = np.asarray(scores)
    return np.argsort(-scores, kind="stable")[: min(k, scores.shape[0])]


# ---------------------------------------------------------------------------
# selection (selection.py)


@dataclass(frozen=True)
class Views:
    """CompressedViews (selection.py:54-70)."""

    q_block: np.ndarray
    k_block: np.ndarray
    k_frame: np.ndarray
    blocks_per_frame: int


def compress(q, k, i, f, n, b_q, b_kv, framewise=False) -> Views:
    """selection.py:95-114 (+ framewise extension)."""
    if not framewise and (n % b_q or n % b_kv):
        raise ValueError("selection needs b_q and b_kv to divide n")  # selection.py:88-92
    qt = q_tiling(f, n, b_q, framewise)
    kt = k_tiling(i, f, n, b_kv, framewise)
    bpf = ceil_div(n, b_kv)
    q_block = mean_pool_bounds(q, qt.all_bounds())
    k_block = mean_pool_bounds(k, kt.all_bounds())
    # framewise summaries pool the block summaries frame by frame (:111)
    k_frame = mean_pool(k_block, bpf)[: (i - 1) * f]
    return Views(q_block, k_block, k_frame, bpf)


def frame_scores(views: Views, r: int) -> np.ndarray:
    """selection.py:117-122 -- raw fp64 dots, no 1/sqrt(d)."""
    return views.k_frame.astype(np.float64) @ views.q_block[r].astype(np.float64)


def select_frames(p, topk_frames, i, f) -> np.ndarray:
    """selection.py:125-134 -- top-k past frames plus every current frame, sorted."""
    past = (i - 1) * f
    picked = topk_indices(np.asarray(p, dtype=np.float64), topk_frames)
    return np.sort(np.concatenate([picked, np.arange(past, past + f)]))


def select_blocks(views: Views, r, frames, budget, mode="global"):
    """selection.py:137-175.  Returns (past_frames, sorted absolute block ids, scores)."""
    if budget < 0:
        raise ValueError(f"budget must be >= 0, got {budget}")
    n_past = views.k_frame.shape[0]
    past = sorted(int(t) for t in np.asarray(frames).ravel() if t < n_past)
    if not past or budget == 0:
        return tuple(past), np.zeros(0, np.int64), np.zeros(0)
    bpf = views.blocks_per_frame
    cand = np.concatenate([np.arange(t * bpf, (t + 1) * bpf) for t in past])
    scores = views.k_block.astype(np.float64)[cand] @ views.q_block[r].astype(np.float64)
    if mode == "global":
        order = np.sort(topk_indices(scores, budget))
    else:
        per = ceil_div(budget, len(past))
        picks = []
        for fi in range(len(past)):
            picks.extend(fi * bpf + topk_indices(scores[fi * bpf:(fi + 1) * bpf], per))
        order = np.sort(np.asarray(picks[:budget], dtype=np.int64))
    return tuple(past), cand[order].astype(np.int64), scores[order]


def round_half_up(x: float) -> int:
    """planner.py:28-29."""
    return int(math.floor(x + 0.5))


def chunk_budget(s_i, i, f, n, b_kv) -> tuple[int, int, bool]:
    """selection.py:212-218 + planner.py:119-123 -> (total, past_budget, clamped)."""
    current = f * ceil_div(n, b_kv)
    total = current if i == 1 else round_half_up((1.0 - s_i) * i * current)
    return total, max(0, total - current), total < current


@dataclass
class Selection:
    frames: list          # per q-block: tuple of retrieved past frames
    blocks: list          # per q-block: sorted absolute past block ids
    scores: list          # per q-block: fp64 scores aligned with blocks
    frame_scores: list    # per q-block: fp64 frame scores
    bits: np.ndarray      # [n_qb, n_kb] bool
    past_budget: int
    total_budget: int
    clamped: bool


def select(q, k, i, s_i, f, n, b_q, b_kv, topk_frames=6, mode="global",
           framewise=False) -> tuple[Views, Selection]:
    """The selection half of hsa_attention (selection.py:196-226)."""
    if not 0.0 <= s_i < 1.0:
        raise ValueError(f"s_i must lie in [0, 1), got {s_i}")
    views = compress(q, k, i, f, n, b_q, b_kv, framewise)
    total, past_budget, clamped = chunk_budget(s_i, i, f, n, b_kv)
    nqb = views.q_block.shape[0]
    nkb = views.k_block.shape[0]
    bits = np.zeros((nqb, nkb), dtype=bool)
    bits[:, (i - 1) * f * views.blocks_per_frame:] = True  # build_mask :188
    sel = Selection([], [], [], [], bits, past_budget, total, clamped)
    for r in range(nqb):
        p = frame_scores(views, r)
        fr = select_frames(p, topk_frames, i, f)
        past, blocks, sc = select_blocks(views, r, fr, past_budget, mode)
        bits[r, blocks] = True
        sel.frames.append(past)
        sel.blocks.append(blocks)
        sel.scores.append(sc)
        sel.frame_scores.append(p)
    return views, sel


# ---------------------------------------------------------------------------
# attention (attention.py)


def _runs(cols: np.ndarray) -> list[tuple[int, int]]:
    """Maximal runs of consecutive active blocks (attention.py:159-165)."""
    if cols.size == 0:
        raise ValueError("query-block row has no active key blocks")
    cut = np.flatnonzero(np.diff(cols) > 1) + 1
    return [(int(g[0]), int(g[-1]) + 1) for g in np.split(cols, cut)]


def _stream(q_rows, k, v64, spans, inv_scale):
    """attention.py:168-188: fp32 QK^T, fp64 online softmax and PV."""
    m = den = acc = None
    for s0, s1 in spans:
        for c in range(s0, s1, KEY_SPAN):
            c1 = min(c + KEY_SPAN, s1)
            s = (q_rows @ k[c:c1].T).astype(np.float64) * inv_scale
            smax = s.max(axis=1)
            if m is None:
                m = smax
                e = np.exp(s - m[:, None])
                den = e.sum(axis=1)
                acc = e @ v64[c:c1]
            else:
                mn = np.maximum(m, smax)
                carry = np.exp(m - mn)
                e = np.exp(s - mn[:, None])
                den = den * carry + e.sum(axis=1)
                acc = acc * carry[:, None] + e @ v64[c:c1]
                m = mn
    return acc / den[:, None]


def block_sparse_attention(q, k, v, bits, q_tiles: Tiling, k_tiles: Tiling, threads=None):
    """attention.py:229-274 generalised to any row/key tiling.

    Each query block attends to the union of its active key blocks; blocks
    that are adjacent in token space are coalesced into spans (attention.py
    :249-262), so the contiguous tiling reproduces the reference exactly.
    """
    q = np.asarray(q, dtype=np.float32)
    k = np.asarray(k, dtype=np.float32)
    v = np.asarray(v, dtype=np.float32)
    bits = np.asarray(bits, dtype=bool)
    qb = q_tiles.all_bounds()
    kb = k_tiles.all_bounds()
    assert bits.shape == (qb.shape[0], kb.shape[0]), (bits.shape, qb.shape, kb.shape)
    inv_scale = 1.0 / math.sqrt(q.shape[1])
    v64 = v.astype(np.float64)
    out = np.empty((q.shape[0], v.shape[1]), dtype=np.float32)
    spans_per_row = []
    for r in range(qb.shape[0]):
        cols = np.flatnonzero(bits[r])
        if cols.size == 0:
            raise ValueError("query-block row has no active key blocks")
        tok = []
        for c in cols:
            s, e = kb[c]
            if tok and tok[-1][1] == s:
                tok[-1] = (tok[-1][0], e)
            else:
                tok.append((int(s), int(e)))
        spans_per_row.append(tok)

    def run(r):
        s, e = qb[r]
        out[s:e] = _stream(q[s:e], k, v64, spans_per_row[r], inv_scale)

    threads = threads or os.cpu_count() or 1
    if threads <= 1:
        for r in range(qb.shape[0]):
            run(r)
    else:
        with ThreadPoolExecutor(max_workers=threads) as ex:
            list(ex.map(run, range(qb.shape[0])))
    active = int(bits.sum())
    return out, active


def dense_attention(q, k, v):
    """attention.py:212-226 (full softmax(q k^T / sqrt d) v)."""
    q = np.asarray(q, dtype=np.float32)
    k = np.asarray(k, dtype=np.float32)
    v = np.asarray(v, dtype=np.float32)
    out = np.empty((q.shape[0], v.shape[1]), dtype=np.float32)
    inv_scale = 1.0 / math.sqrt(q.shape[1])
    v64 = v.astype(np.float64)
    for r0 in range(0, q.shape[0], 128):
        r1 = min(r0 + 128, q.shape[0])
        out[r0:r1] = _stream(q[r0:r1], k, v64, [(0, k.shape[0])], inv_scale)
    return out


def hsa_attention(q, k, v, i, s_i, f, n, b_q, b_kv, topk_frames=6, mode="global",
                  framewise=False, threads=None):
    """selection.py:196-231 (+ framewise extension)."""
    views, sel = select(q, k, i, s_i, f, n, b_q, b_kv, topk_frames, mode, framewise)
    out, active = block_sparse_attention(
        q, k, v, sel.bits, q_tiling(f, n, b_q, framewise),
        k_tiling(i, f, n, b_kv, framewise), threads=threads)
    return out, sel, views


def effective_flops(bits, q_tiles: Tiling, k_tiles: Tiling, d: int) -> int:
    """Exact-extent FLOPs of the active tiles: 4 * rows * cols * d (QK^T + PV)."""
    qb = q_tiles.all_bounds()
    kb = k_tiles.all_bounds()
    rows = (qb[:, 1] - qb[:, 0]).astype(np.int64)
    cols = (kb[:, 1] - kb[:, 0]).astype(np.int64)
    return int(4 * d * (rows[:, None] * cols[None, :] * np.asarray(bits, bool)).sum())


def token_oracle(q, k, v, bits, q_tiles: Tiling, k_tiles: Tiling) -> np.ndarray:
    """Fully materialised fp64 masked attention (test_attention.py:25-38 style)."""
    q64, k64, v64 = (np.asarray(a, np.float64) for a in (q, k, v))
    s = q64 @ k64.T / math.sqrt(q.shape[1])
    qid = np.empty(q.shape[0], np.int64)
    for g, (a, b) in enumerate(q_tiles.all_bounds()):
        qid[a:b] = g
    kid = np.empty(k.shape[0], np.int64)
    for g, (a, b) in enumerate(k_tiles.all_bounds()):
        kid[a:b] = g
    tok = np.asarray(bits, bool)[qid][:, kid]
    s = np.where(tok, s, -np.inf)
    s -= s.max(axis=1, keepdims=True)
    w = np.exp(s)
    w /= w.sum(axis=1, keepdims=True)
    return (w @ v64).astype(np.float32)


# ---------------------------------------------------------------------------
# CAG planner (planner.py)


class DegenerateSchedule(ValueError):
    pass


def alpha_schedule(N: int, T: int) -> np.ndarray:
    """planner.py:56-66."""
    raw = 1.0 / np.sqrt(np.arange(1, N + 1, dtype=np.float64) * T)
    return raw / raw.max()


@dataclass(frozen=True)
class Plan:
    alpha: tuple
    beta: float
    s: tuple
    budgets: tuple
    clamped: tuple
    achieved: float


def allocate(s_target, s_base, N, T, f, n, b_kv, d, first_chunk_dense=True,
             redistribute=False) -> Plan:
    """planner.py:126-175 with _solve_clamped 178-208."""
    if not 0.0 <= s_target < 1.0 or not 0.0 <= s_base <= 1.0:
        raise ValueError("need 0 <= s_target < 1 and 0 <= s_base <= 1")
    if s_target > s_base:
        raise ValueError("s_target > s_base")
    alpha = alpha_schedule(N, T)
    lq = f * n
    w = np.asarray([lq * (i * lq) * d for i in range(1, N + 1)], dtype=np.float64)
    bpf = ceil_div(n, b_kv)
    cur = f * bpf
    s_hi = np.asarray([1.0 - cur / (i * cur) for i in range(1, N + 1)])
    planned = np.ones(N, dtype=bool)
    if first_chunk_dense:
        planned[0] = False
    s = np.zeros(N)
    clamped = np.zeros(N, dtype=bool)
    beta = 0.0
    if planned.any():
        target = (1.0 - s_target) * float(w[planned].sum())
        free = planned.copy()
        while True:
            den = float(np.dot(alpha[free], w[free]))
            if den <= 0.0:
                raise DegenerateSchedule("no solvable chunks left")
            fixed = planned & ~free
            resid = target - float(((1.0 - s[fixed]) * w[fixed]).sum())
            beta = (resid - (1.0 - s_base) * float(w[free].sum())) / den
            raw = s_base - alpha * beta
            s[free] = np.clip(raw[free], 0.0, s_hi[free])
            newly = free & (raw != s)
            clamped |= newly
            if not redistribute or not newly.any() or not (free & ~newly).any():
                break
            free = free & ~newly
    s[~planned] = 0.0
    clamped[~planned] = False
    budgets = tuple(round_half_up((1.0 - float(s[i - 1])) * i * cur) for i in range(1, N + 1))
    if planned.any():
        achieved = float(((1.0 - s[planned]) * w[planned]).sum()) / float(w[planned].sum())
    else:
        achieved = 1.0
    return Plan(tuple(float(a) for a in alpha), float(beta), tuple(float(x) for x in s),
                budgets, tuple(bool(c) for c in clamped), achieved)


# ---------------------------------------------------------------------------
# inputs shared by tests and the bench


def bf16_round(x: np.ndarray) -> np.ndarray:
    """Round fp32 -> bf16 (nearest-even) and back, exactly as torch does."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    u = x.view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) >> 16
    return (u.astype(np.uint32) << 16).view(np.float32)


def synthetic_qkv(seed, lq, lk, d, heads=1, bf16=True):
    """Seeded N(0,1) q/k/v as fp32 arrays [heads, L, d].

    With ``bf16`` (the default) every value is rounded to a bf16 value, so the
    GPU's bf16 copies and the oracle's fp32 copies hold identical numbers.
    """
    rng = np.random.default_rng(seed)
    rnd = bf16_round if bf16 else (lambda a: a)
    q = rnd(rng.standard_normal((heads, lq, d), dtype=np.float32))
    k = rnd(rng.standard_normal((heads, lk, d), dtype=np.float32))
    v = rnd(rng.standard_normal((heads, lk, d), dtype=np.float32))
    return q, k, v
