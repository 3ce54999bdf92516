"""Host<->device plumbing shared by the reference-compatible API."""

from __future__ import annotations

import numpy as np
import torch


def is_torch(a) -> bool:
    return torch.is_tensor(a)


def device() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2602_04789_b200 needs a CUDA (sm_100a) device; none is visible")
    return torch.device("cuda", torch.cuda.current_device())


def as_matrix_dev(a, name: str = "matrix") -> torch.Tensor:
    """numerics.py:33-41 (as_matrix) for host or device input -> fp32 CUDA [rows, d].

    Validation (2-D, non-empty, finite) mirrors the reference; float64 input is
    rounded to float32 exactly like the reference's astype(float32).
    """
    if is_torch(a):
        t = a
        if t.dim() != 2 or t.numel() == 0:
            raise ValueError(f"{name} must be non-empty 2-D, got shape {tuple(t.shape)}")
        t = t.to(device=device(), dtype=torch.float32)
        if not bool(torch.isfinite(t).all()):
            raise ValueError(f"{name} contains non-finite values")
        return t.contiguous()
    arr = np.asarray(a)
    if arr.ndim != 2 or arr.size == 0:
        raise ValueError(f"{name} must be non-empty 2-D, got shape {arr.shape}")
    arr = np.ascontiguousarray(arr, dtype=np.float32)
    if not np.all(np.isfinite(arr)):
        raise ValueError(f"{name} contains non-finite values")
    return torch.from_numpy(arr).to(device(), non_blocking=False)


def padded_width(d: int) -> int:
    if d <= 64:
        return 64
    if d <= 128:
        return 128
    raise NotImplementedError(f"head dim {d} > 128 is not implemented by the sm_100a kernel")


def to_bf16_heads(x: torch.Tensor) -> torch.Tensor:
    """[L, d] or [H, L, d] -> bf16 [H, L, dp] with zero padding to the kernel width."""
    if x.dim() == 2:
        x = x.unsqueeze(0)
    d = x.shape[-1]
    dp = padded_width(d)
    if x.dtype == torch.bfloat16 and dp == d and x.stride(-1) == 1:
        return x
    out = torch.zeros((x.shape[0], x.shape[1], dp), dtype=torch.bfloat16, device=x.device)
    out[..., :d] = x
    return out


def like_input(t: torch.Tensor, ref):
    """Return a numpy array when the caller passed numpy, else the tensor."""
    if is_torch(ref):
        return t
    return t.detach().cpu().numpy()
