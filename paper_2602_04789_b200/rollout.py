"""Device-resident rollout driver with an incremental pooled-summary cache.

The reference's rollout (rollout.py:276-309) calls ``HsaBackend.run`` ->
``hsa_attention`` on every denoising step with the full concatenated K/V
(rollout.py:263-266), and ``compress`` re-pools the whole key context each
time (selection.py:109-111), although past chunks are fixed once committed
(rollout.py:306-308).  ``HsaRollout`` keeps the KV cache on the GPU and pools
each clean chunk's key blocks and frame summaries exactly once, when the
chunk is committed; a denoising step then pools only its query chunk:
selection reads past summaries from the cache.

Selections and outputs are bit-identical to ``HsaPipeline`` on the same
inputs: the selection only ever reads *past* block/frame summaries, and those
come from the same pooling kernels applied to the same rows (the current
chunk's key summaries are never candidates, selection.py:137-175).

Per step: pool Q (1 launch) -> select -> plan tiles -> attention (4 launches),
HBM traffic for pooling f*n*d*2 bytes per head instead of (i+1)*f*n*d*2.
"""

from __future__ import annotations

import math

import torch

from . import _lib as L
from . import device as D
from .layout import ChunkLayout, as_layout, is_aligned
from .planner import SparsityPlan
from .selection import SelectionConfig, tilings


class HsaRollout:
    def __init__(self, layout: ChunkLayout, heads: int, plan: SparsityPlan | None = None,
                 cfg: SelectionConfig | None = None, framewise: bool | None = None,
                 out_dtype=torch.bfloat16, device=None, keep_frames: bool = False):
        """keep_frames: also return each step's retrieved past frames
        (StepPlan.selection.frames, else None).  Nothing downstream of the
        selection reads them, and without them a step whose past budget is 0
        skips the frame ranking (it cannot change the mask)."""
        self.layout = layout = as_layout(layout)
        self.keep_frames = bool(keep_frames)
        self.heads = int(heads)
        self.plan = plan
        self.cfg = cfg or SelectionConfig()
        self.framewise = (not is_aligned(self.layout)) if framewise is None else bool(framewise)
        if not self.framewise and not is_aligned(self.layout):
            raise ValueError(
                f"selection needs b_q and b_kv to divide n: n={layout.n}, b_q={layout.b_q}, "
                f"b_kv={layout.b_kv}")
        self.out_dtype = out_dtype
        self.device = device or torch.device("cuda", torch.cuda.current_device())
        lay = layout
        H, d = self.heads, lay.d
        self.bpf = lay.frame_kv_blocks
        self.cap_tokens = lay.N * lay.f * lay.n
        # device KV cache and summary caches, sized for the whole rollout
        self.kv_k = torch.zeros((H, self.cap_tokens, d), dtype=torch.bfloat16, device=self.device)
        self.kv_v = torch.zeros((H, self.cap_tokens, d), dtype=torch.bfloat16, device=self.device)
        self.kb_cache = torch.zeros((H, lay.N * lay.f * self.bpf, d), dtype=torch.float32,
                                    device=self.device)
        self.kf_cache = torch.zeros((H, lay.N * lay.f, d), dtype=torch.float32, device=self.device)
        self.committed = 0  # chunks whose clean K/V are in the cache
        self.err = torch.zeros(1, dtype=torch.int32, device=self.device)
        # this rollout's attention split-KV scratch (zero-filled once, lfattn.h):
        # independent of every other rollout / pipeline, also on other devices
        nbytes = int(L.load_library().lf_attention_scratch_bytes(
            H, L.tiling(lay.chunk_tokens, lay.n, lay.b_q), d))
        with torch.cuda.device(self.device):
            self.scratch = torch.zeros(nbytes, dtype=torch.uint8, device=self.device)

    # ------------------------------------------------------------------ helpers
    def _slot(self, i: int) -> slice:
        cl = self.layout.chunk_tokens
        return slice((i - 1) * cl, i * cl)

    def _s_dev(self, i: int, s_i):
        if s_i is not None:
            if torch.is_tensor(s_i):
                return s_i
            return torch.tensor([float(s_i)], dtype=torch.float64, device=self.device)
        if self.plan is None:
            raise ValueError("no sparsity plan: pass s_i")
        return self.plan.s_device(i)

    # ------------------------------------------------------------------ API
    def kv_slot(self, chunk_index: int):
        """Device views (k, v) [H, f*n, d] of chunk i's cache slot, for producers
        that write their K/V projections in place (then pass None to step)."""
        sl = self._slot(int(chunk_index))
        return self.kv_k[:, sl], self.kv_v[:, sl]

    def commit(self, k_clean: torch.Tensor, v_clean: torch.Tensor, chunk_index: int,
               overwrite: bool = False) -> None:
        """Append chunk i's clean K/V (rollout.py:306-308) and pool its summaries once.

        ``overwrite`` re-writes an already committed chunk in place (used by
        the benchmark to replay one chunk of a steady-state rollout).
        """
        lay = self.layout
        i = int(chunk_index)
        if overwrite and 1 <= i <= self.committed:
            pass
        elif i != self.committed + 1:
            raise ValueError(f"chunks must be committed in order: expected {self.committed + 1}, got {i}")
        lay.check_chunk(i)
        sl = self._slot(i)
        if k_clean is not None:  # None: already written in place (kv_slot)
            self.kv_k[:, sl].copy_(k_clean)
        if v_clean is not None:
            self.kv_v[:, sl].copy_(v_clean)
        # k_block rows of this chunk's frames
        spec = D.TilingSpec(lay.chunk_tokens, lay.n if self.framewise else lay.chunk_tokens,
                            lay.b_kv)
        nb = lay.f * self.bpf
        kb = self.kb_cache[:, (i - 1) * nb:i * nb]
        kf = self.kf_cache[:, (i - 1) * lay.f:i * lay.f]
        # one launch (block means + frame summaries, lf_pool_chunk_k) when the
        # layout allows it, else two pooling passes; both bit-identical
        if not (self.framewise and self._pool_chunk(self.kv_k[:, sl], spec, kb, kf)):
            self._pool_into(self.kv_k[:, sl], spec, kb)
            # k_frame rows = mean of each frame's block means (selection.py:111)
            fspec = D.TilingSpec(nb, nb, self.bpf)
            self._pool_into(kb, fspec, kf)
        self.committed = max(self.committed, i)

    def selection_flops(self) -> int:
        """Exact-extent FLOPs (4*rows*cols*d over active tiles) of the last step."""
        import numpy as np
        sel, i = self.last_selection, self.last_chunk
        qt, kt = tilings(self.layout, i, self.framewise)
        b, c = sel.blocks.cpu().numpy(), sel.count.cpu().numpy()
        qb, kb = qt.bounds(), kt.bounds()
        rows = (qb[:, 1] - qb[:, 0]).astype(np.int64)
        cols = (kb[:, 1] - kb[:, 0]).astype(np.int64)
        cur = int(cols[(i - 1) * self.layout.f * self.bpf:].sum())
        total = 0
        for h in range(self.heads):
            for r in range(qt.count):
                total += int(rows[r]) * (cur + int(cols[b[h, r, :c[h, r]]].sum()))
        return int(4 * self.layout.d * total)

    def _pool_chunk(self, x, spec: D.TilingSpec, kb, kf) -> bool:
        import ctypes

        from . import _lib as L
        m = L.mat(x)
        rc = L.lib().lf_pool_chunk_k(ctypes.byref(m), spec.abi(), self.bpf, kb.data_ptr(),
                                     kb.stride(0), kf.data_ptr(), kf.stride(0), L.stream_ptr())
        if rc == L.LF_ERR_UNSUPPORTED:
            return False
        L.check(rc)
        return True

    def _pool_into(self, x: torch.Tensor, spec: D.TilingSpec, out: torch.Tensor) -> None:
        import ctypes

        from . import _lib as L
        lib = L.lib()
        m = L.mat(x)
        L.check(lib.lf_pool_blocks(ctypes.byref(m), spec.abi(), -1, out.data_ptr(), out.stride(0),
                                   L.stream_ptr()))

    def step(self, q: torch.Tensor, k_cur: torch.Tensor, v_cur: torch.Tensor, chunk_index: int,
             s_i=None, out: torch.Tensor | None = None, s_host=None) -> torch.Tensor:
        """One denoising step of chunk i (rollout.py:254-273 attention part).

        q, k_cur, v_cur: bf16 [H, f*n, d] for the noisy current chunk.
        Past chunks 1..i-1 must have been committed.
        """
        self.layout.check_chunk(int(chunk_index))
        if k_cur is not None or v_cur is not None:
            sl = self._slot(int(chunk_index))
            if k_cur is not None:  # None: the caller already wrote them in place (kv_slot)
                self.kv_k[:, sl].copy_(k_cur)
            if v_cur is not None:
                self.kv_v[:, sl].copy_(v_cur)
        return self.attend(self.prepare(q, chunk_index, s_i=s_i, s_host=s_host), out=out)

    def prepare(self, q: torch.Tensor, chunk_index: int, s_i=None, s_host=None) -> "StepPlan":
        """Selection half of a step: pool q, hierarchical selection against the
        cached summaries, tile plan.  Reads only q and the committed summaries
        (not the current chunk's K/V), so a caller may run it for step s+1 on a
        side stream while step s attends.  Enqueued on the current stream."""
        lay = self.layout
        i = int(chunk_index)
        lay.check_chunk(i)
        if self.committed != i - 1:
            raise ValueError(f"chunk {i} needs chunks 1..{i - 1} committed (have {self.committed})")
        qt, kt = tilings(lay, i, self.framewise)
        P = (i - 1) * lay.f
        q_block = D.pool_blocks(q, qt)
        s_dev = self._s_dev(i, s_i)
        if s_host is None and s_i is not None and not torch.is_tensor(s_i):
            s_host = float(s_i)
        if s_host is None and s_i is None and self.plan is not None:
            s_host = float(self.plan.s[i - 1])
        # query-tile geometry of this step (block-aligned when the past selection is large)
        with D.qtile_scope(D.auto_qtile_mode(s_host, i, lay.f, self.bpf, self.cfg.topk_frames)):
            sel, tiles, _ = D.select_plan(q_block, self.kb_cache, self.kf_cache, self.bpf, i,
                                          lay.f, self.cfg.topk_frames,
                                          self.cfg.block_budget_mode == "per-frame", s_dev, qt,
                                          kt, P * self.bpf, want_frames=self.keep_frames)
            qmode = D.qtile_mode(qt)
        hint = D.past_tiles_hint(s_host, i, lay.f, self.bpf, self.cfg.topk_frames, qt)
        self.last_selection = sel
        self.last_chunk = i
        return StepPlan(q, i, qt, q_block, sel, tiles, hint, qmode)

    def attend(self, plan: "StepPlan", out: torch.Tensor | None = None) -> torch.Tensor:
        """Attention half of a step: block-sparse attention of plan.q over the
        cache (past chunks + the current chunk's K/V in its slot).

        The plan may come from ``prepare`` on another stream: its device
        tensors are marked used by the current stream, so the caching allocator
        cannot hand their memory to new work before this launch has run."""
        lay = self.layout
        i = plan.chunk
        P = (i - 1) * lay.f
        lk = lay.context_tokens(i)
        cur = torch.cuda.current_stream()
        for t in plan.device_tensors():
            t.record_stream(cur)
        with D.qtile_scope(plan.qmode):
            return D.attention(plan.q, self.kv_k[:, :lk], self.kv_v[:, :lk], plan.qt, plan.tiles,
                               P * lay.n, lk, out=out, out_dtype=self.out_dtype,
                               scale=1.0 / math.sqrt(lay.d), err=self.err, past_tiles=plan.hint,
                               scratch=self.scratch, qperm=plan.tiles.qperm)


class StepPlan:
    """Device results of HsaRollout.prepare (kept alive until attend has run)."""

    def __init__(self, q, chunk, qt, q_block, selection, tiles, hint, qmode=0):
        self.q = q
        self.chunk = chunk
        self.qt = qt
        self.q_block = q_block
        self.selection = selection
        self.tiles = tiles
        self.hint = hint
        self.qmode = qmode  # query-tile geometry the plan was made for (device.qtile_rows)

    def device_tensors(self):
        """The CUDA tensors attend() reads (for record_stream)."""
        sel = self.selection
        out = [self.q, self.q_block, self.tiles.segs, self.tiles.seg_count, self.tiles.qperm,
               sel.blocks, sel.count, sel.frames, sel.budget]
        return [t for t in out if t is not None and t.is_cuda]


# --------------------------------------------------------------------------- ablation settings
# Host-side helpers of the reference's Fig. 2 ablation (rollout.py:333-374):
# two budget settings matched in nominal FLOPs, run through FixedMaskBackend.

def largest_remainder_split(total: int, weights) -> list:
    """Split integer ``total`` in proportion to ``weights`` (largest remainder,
    ties to the lowest index).  Restates rollout.py:333-347."""
    import numpy as np
    w = np.asarray(weights, dtype=np.float64)
    if total < 0 or w.size == 0 or (w < 0).any() or w.sum() <= 0:
        raise ValueError("need total >= 0 and positive weight mass")
    exact = total * w / w.sum()
    parts = np.floor(exact).astype(np.int64)
    left = total - int(parts.sum())
    rem = exact - parts
    # stable order: larger remainder first, then lower index
    order = sorted(range(w.size), key=lambda j: (-rem[j], j))
    for j in order[:left]:
        parts[j] += 1
    return [int(x) for x in parts]


def matched_budget_settings(layout, N: int, first_chunk_sparsity: float):
    """Per-chunk row budgets (key blocks) of the two ablation settings, equal in
    total: A sparsifies chunk 1 only, B keeps chunk 1 dense and removes the same
    number of blocks from chunks 2..N in proportion to their context.
    Restates rollout.py:350-374 (same errors)."""
    from .planner import round_half_up
    if not 0.0 < first_chunk_sparsity < 1.0:
        raise ValueError(f"first_chunk_sparsity must lie in (0, 1), got {first_chunk_sparsity}")
    if N < 2 or N > layout.N:
        raise ValueError(f"need 2 <= N <= {layout.N}, got {N}")
    full = [layout.k_blocks(i) for i in range(1, N + 1)]
    keep = max(1, round_half_up((1.0 - first_chunk_sparsity) * full[0]))
    a = [keep] + full[1:]
    cut = largest_remainder_split(full[0] - keep, full[1:])
    b = [full[0]] + [max(1, fb - c) for fb, c in zip(full[1:], cut)]
    if sum(a) != sum(b):
        raise ValueError("could not match totals; increase chunk sizes")
    return a, b
