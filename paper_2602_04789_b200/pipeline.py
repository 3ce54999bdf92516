"""Batched, device-resident hot path: all heads of one layer per call.

``HsaPipeline`` wraps ``lf_hsa_forward`` (compress -> select -> plan tiles ->
tcgen05 sparse attention, five launches, no host sync) for bf16 [H, L, d]
CUDA tensors, with a preallocated workspace and optional CUDA-graph capture
of the whole call.  This is the path the bench measures and the GPU rollout
backends use; ``selection.hsa_attention`` is the single-head drop-in.
"""

from __future__ import annotations

import ctypes
import math

import numpy as np
import torch

from . import _lib as L
from .layout import BlockMask, ChunkLayout, as_layout, is_aligned
from .selection import SelectionConfig, mask_from_lists, tilings


class HsaPipeline:
    def __init__(self, layout: ChunkLayout, heads: int, chunk_index: int,
                 cfg: SelectionConfig | None = None, framewise: bool | None = None,
                 out_dtype=torch.bfloat16, device=None, keep_frames: bool = True):
        """keep_frames=False: selections() returns no frame lists (None), and a
        call whose past budget is 0 skips the frame ranking (it cannot change
        the mask) -- what the bench's stateless leg runs."""
        self.layout = layout = as_layout(layout)
        self.keep_frames = bool(keep_frames)
        self.heads = int(heads)
        self.chunk = int(chunk_index)
        self.cfg = cfg or SelectionConfig()
        self.framewise = (not is_aligned(self.layout)) if framewise is None else bool(framewise)
        if not self.framewise and not is_aligned(self.layout):
            raise ValueError(
                f"selection needs b_q and b_kv to divide n: n={layout.n}, b_q={layout.b_q}, "
                f"b_kv={layout.b_kv}")
        layout.check_chunk(self.chunk)
        self.out_dtype = out_dtype
        self.device = device or torch.device("cuda", torch.cuda.current_device())
        self.qt, self.kt = tilings(layout, self.chunk, self.framewise)
        self.lq = layout.chunk_tokens
        self.lk = layout.context_tokens(self.chunk)
        self._args = None
        self._ws = None
        self._graph = None
        self._bound = None
        self.err = torch.zeros(1, dtype=torch.int32, device=self.device)
        self.attn_kernel = L.LF_KERNEL_AUTO
        self._s_host = None

    # ------------------------------------------------------------------ binding
    def _make_args(self, q, k, v, s_dev, out):
        a = L.LfHsaArgs()
        a.q, a.k, a.v = L.mat(q), L.mat(k), L.mat(v)
        lay = self.layout
        a.f, a.n, a.b_q, a.b_kv = lay.f, lay.n, lay.b_q, lay.b_kv
        a.framewise = 1 if self.framewise else 0
        a.chunk_index = self.chunk
        a.topk_frames = self.cfg.topk_frames
        a.per_frame_mode = 1 if self.cfg.block_budget_mode == "per-frame" else 0
        a.s_i_dev = s_dev.data_ptr()
        a.out = out.data_ptr()
        a.out_dtype = L.LF_F32 if out.dtype == torch.float32 else L.LF_BF16
        a.out_row_stride = out.stride(1)
        a.out_head_stride = out.stride(0)
        a.lse = None
        a.err_flag = self.err.data_ptr()
        a.attn_kernel = self.attn_kernel
        a.s_i_host = float("nan") if self._s_host is None else float(self._s_host)
        a.skip_frames = 0 if self.keep_frames else 1
        return a

    def bind(self, q, k, v, s_i, out=None, s_host=None):
        """Fix the buffers a (captured) call reads and writes.

        s_host: host value of s_i when s_i is a device tensor (the kernel choice
        uses it; None = unknown)."""
        lib = L.lib()
        H, d = self.heads, self.layout.d
        for name, t, rows in (("q", q, self.lq), ("k", k, self.lk), ("v", v, self.lk)):
            if t.dtype != torch.bfloat16 or t.dim() != 3 or t.shape[0] != H or t.shape[2] != d:
                raise ValueError(f"{name}: expected bf16 [{H}, L, {d}], got {t.dtype} {tuple(t.shape)}")
            if t.shape[1] < rows:
                raise ValueError(f"{name}: {t.shape[1]} rows < {rows}")
        self._s_host = s_host
        if not torch.is_tensor(s_i):
            self._s_host = float(s_i)
            s_i = torch.tensor([float(s_i)], dtype=torch.float64, device=self.device)
        if out is None:
            out = torch.empty((H, self.lq, d), dtype=self.out_dtype, device=self.device)
        a = self._make_args(q, k, v, s_i, out)
        nbytes = lib.lf_hsa_workspace_bytes(ctypes.byref(a))
        if nbytes == 0:
            L.check(L.LF_ERR_INVALID)
        if self._ws is None or self._ws.numel() < nbytes:
            # zero-filled once: the attention scratch in it must start at zero (lfattn.h)
            self._ws = torch.zeros(nbytes, dtype=torch.uint8, device=self.device)
        self._args = a
        self._bound = (q, k, v, s_i, out)
        self._graph = None
        return out

    def launch(self):
        """Enqueue one full hot-path call on the current stream."""
        lib = L.lib()
        L.check(lib.lf_hsa_forward(ctypes.byref(self._args), self._ws.data_ptr(),
                                   self._ws.numel(), L.stream_ptr()))

    def __call__(self, q, k, v, s_i, out=None, s_host=None):
        out = self.bind(q, k, v, s_i, out, s_host=s_host)
        self.launch()
        return out

    # ------------------------------------------------------------------ graphs
    def capture(self, warmup: int = 1):
        """Capture launch() into a CUDA graph (buffers fixed by bind())."""
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            for _ in range(warmup):
                self.launch()
        torch.cuda.current_stream().wait_stream(s)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self.launch()
        self._graph = g
        return g

    def replay(self):
        if self._graph is None:
            self.capture()
        self._graph.replay()

    # ------------------------------------------------------------------ results
    def _views(self):
        lib = L.lib()
        ptrs = [ctypes.c_void_p() for _ in range(7)]
        cap = ctypes.c_int32()
        fcap = ctypes.c_int32()
        L.check(lib.lf_hsa_views(ctypes.byref(self._args), self._ws.data_ptr(),
                                 *[ctypes.byref(p) for p in ptrs], ctypes.byref(cap),
                                 ctypes.byref(fcap)))
        return ptrs, cap.value, fcap.value

    def _read(self, ptr, count, dtype):
        """View of a workspace region (no copy; offsets are 256-byte aligned)."""
        off = ptr - self._ws.data_ptr()
        esz = torch.empty(0, dtype=dtype).element_size()
        return self._ws[off:off + count * esz].view(dtype)

    def selections(self):
        """Per-head selected past blocks: (blocks [H, nqb, cap], count [H, nqb], frames, budget)."""
        ptrs, cap, fcap = self._views()
        H, nqb = self.heads, self.qt.count
        blocks = self._read(ptrs[3].value, H * nqb * cap, torch.int32).view(H, nqb, cap)
        count = self._read(ptrs[4].value, H * nqb, torch.int32).view(H, nqb)
        frames = (self._read(ptrs[5].value, H * nqb * fcap, torch.int32).view(H, nqb, fcap)
                  if self.keep_frames else None)
        budget = self._read(ptrs[6].value, 4, torch.int32)
        return blocks, count, frames, budget

    def views(self):
        """Pooled summaries q_block [H,nqb,d], k_block [H,nkb,d], k_frame [H,P,d] (fp32)."""
        ptrs, _, _ = self._views()
        H, d = self.heads, self.layout.d
        P = (self.chunk - 1) * self.layout.f
        qb = self._read(ptrs[0].value, H * self.qt.count * d, torch.float32).view(H, -1, d)
        kb = self._read(ptrs[1].value, H * self.kt.count * d, torch.float32).view(H, -1, d)
        kf = self._read(ptrs[2].value, H * P * d, torch.float32).view(H, P, d) if P else None
        return qb, kb, kf

    def masks(self):
        """Lazy BlockMask per head."""
        blocks, count, _, _ = self.selections()
        b, c = blocks.cpu().numpy(), count.cpu().numpy()
        bpf = self.layout.frame_kv_blocks
        past_cols = (self.chunk - 1) * self.layout.f * bpf
        nkb = self.kt.count
        return [BlockMask.lazy(lambda h=h: mask_from_lists(b[h], c[h], nkb, past_cols),
                               self.qt.count, nkb) for h in range(self.heads)]

    def effective_flops(self) -> int:
        """Exact-extent FLOPs (4*rows*cols*d over active tiles) of the last call."""
        blocks, count, _, _ = self.selections()
        b, c = blocks.cpu().numpy(), count.cpu().numpy()
        qb, kb = self.qt.bounds(), self.kt.bounds()
        rows = (qb[:, 1] - qb[:, 0]).astype(np.int64)
        cols = (kb[:, 1] - kb[:, 0]).astype(np.int64)
        past_cols = (self.chunk - 1) * self.layout.f * self.layout.frame_kv_blocks
        cur = int(cols[past_cols:].sum())
        total = 0
        for h in range(self.heads):
            for r in range(self.qt.count):
                total += int(rows[r]) * (cur + int(cols[b[h, r, :c[h, r]]].sum()))
        return int(4 * self.layout.d * total)

    def errors(self) -> int:
        return int(self.err.item())


def scale_for(d: int) -> float:
    return 1.0 / math.sqrt(d)
