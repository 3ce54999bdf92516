"""Numeric primitives with the reference's names (chunkattn numerics.py:1-104).

``mean_pool`` and ``topk_indices`` run on the GPU (csrc/pool.cuh,
csrc/select.cuh) and are bit-identical to the reference; ``as_matrix`` is the
reference's host-side validation.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _convert as C
from . import device as D
from .errors import EmptyActiveSetError


@dataclass(frozen=True)
class TopKResult:
    """numerics.py:19-30."""

    indices: np.ndarray
    scores: np.ndarray

    def __len__(self) -> int:
        return len(self.indices)


def as_matrix(a, name: str = "matrix") -> np.ndarray:
    """Validate a 2-D finite float array and return it as float32 (numerics.py:33-41)."""
    arr = np.asarray(a.detach().cpu() if torch.is_tensor(a) else a)
    if arr.ndim != 2 or arr.size == 0:
        raise ValueError(f"{name} must be non-empty 2-D, got shape {arr.shape}")
    arr = arr.astype(np.float32, copy=False)
    if not np.all(np.isfinite(arr)):
        raise ValueError(f"{name} contains non-finite values")
    return arr


def mean_pool(x, group: int):
    """Average consecutive groups of ``group`` rows on the GPU (numerics.py:44-66)."""
    if group < 1:
        raise ValueError(f"pool size must be >= 1, got {group}")
    shape = tuple(x.shape)
    if len(shape) != 2 or shape[0] < 1:
        raise ValueError(f"expected non-empty 2-D input, got shape {shape}")
    xd = x.to(C.device()) if torch.is_tensor(x) else \
        torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).to(C.device())
    if xd.dtype not in (torch.float32, torch.bfloat16):
        xd = xd.float()
    out = D.pool_blocks(xd.contiguous(), D.TilingSpec(shape[0], shape[0], group))
    return C.like_input(out, x)


def topk_indices(scores, k: int) -> TopKResult:
    """k largest scores, ties to the lower index, on the GPU (numerics.py:91-104)."""
    if k < 0:
        raise ValueError(f"k must be >= 0, got {k}")
    s = scores if torch.is_tensor(scores) else np.asarray(scores)
    if s.ndim != 1:
        raise ValueError(f"expected 1-D scores, got shape {tuple(s.shape)}")
    n = s.shape[0]
    if n == 0 or k == 0:
        idx = np.zeros(0, dtype=np.int64)
        sc = np.asarray(s.cpu() if torch.is_tensor(s) else s)[idx]
        return TopKResult(indices=idx, scores=sc)
    sd = s.to(C.device()).double() if torch.is_tensor(s) else \
        torch.from_numpy(np.ascontiguousarray(s, dtype=np.float64)).to(C.device())
    idx = D.topk(sd, k).cpu().numpy().astype(np.int64)
    host = s.detach().cpu().numpy() if torch.is_tensor(s) else s
    return TopKResult(indices=idx, scores=host[idx])


def stable_softmax_row(logits, active=None) -> np.ndarray:
    """Softmax over an active index set, fp64 statistics (numerics.py:69-88).

    Diagnostic helper (not on the hot path); evaluated with torch on the device.
    """
    lg = torch.as_tensor(np.asarray(logits, dtype=np.float64), device=C.device())
    if lg.dim() != 1:
        raise ValueError(f"expected 1-D logits, got shape {tuple(lg.shape)}")
    act = torch.arange(lg.shape[0], device=lg.device) if active is None else \
        torch.as_tensor(np.asarray(active, dtype=np.int64), device=lg.device)
    if act.numel() == 0:
        raise EmptyActiveSetError("softmax row has no active entries")
    picked = lg[act]
    e = torch.exp(picked - picked.max())
    out = torch.zeros_like(lg)
    out[act] = e / e.sum()
    return out.cpu().numpy()
