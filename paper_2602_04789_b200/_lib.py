"""ctypes binding of the C ABI (include/lfattn.h) and torch<->ABI plumbing.

The shared library is built in-tree (``_lib/liblfattn.so``) by
``__graft_entry__.build()`` / ``python -m paper_2602_04789_b200.build``.
There is no fallback: if the library or a CUDA device is missing, every
compute entry point raises ``RuntimeError``.
"""

from __future__ import annotations

import contextlib
import ctypes
import os

import torch

from .errors import DegenerateScheduleError, ZeroActiveRowError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_lib", "liblfattn.so")

LF_OK, LF_ERR_INVALID, LF_ERR_CUDA, LF_ERR_UNSUPPORTED = 0, 1, 2, 3
LF_ERR_ZERO_ACTIVE_ROW, LF_ERR_DEGENERATE, LF_ERR_NO_DRIVER = 4, 5, 6
LF_F32, LF_BF16 = 0, 1
LF_KERNEL_AUTO, LF_KERNEL_TILE = 0, 3

# every symbol include/lfattn.h declares (checked by tests/test_abi.py)
EXPORTS = (
    "lf_version", "lf_strerror", "lf_last_error", "lf_pool_blocks", "lf_compress", "lf_select",
    "lf_select_strided", "lf_select_plan", "lf_pair_qblocks", "lf_plan_tiles_paired",
    "lf_attention_paired",
    "lf_cag_plan", "lf_plan_tile_rows", "lf_pool_chunk_k", "lf_set_qtile_mode",
    "lf_qtile_mode", "lf_plan_tile_count", "lf_plan_tiles", "lf_attention", "lf_attention_ex",
    "lf_attention_kernel_choice", "lf_hsa_workspace_bytes", "lf_hsa_views",
    "lf_hsa_forward", "lf_select_fallbacks", "lf_rowdot", "lf_topk", "lf_attention_ws", "lf_attention_scratch_bytes",
    "lf_set_option", "lf_get_option",
)

# library options (include/lfattn.h LF_OPT_*)
OPTIONS = {
    "pool_cfg": 0, "pool_no_tma": 1, "attn_split": 2, "attn_sched": 3, "plan_warp": 4,
    "select_exact": 5, "attn_debug": 6, "attn_poly": 7, "attn_kernel": 8, "qtile": 9,
    "trace_cta": 10, "pdl": 11,
}


class LfTiling(ctypes.Structure):
    _fields_ = [("total", ctypes.c_int32), ("period", ctypes.c_int32), ("block", ctypes.c_int32)]


class LfMat(ctypes.Structure):
    _fields_ = [("ptr", ctypes.c_void_p), ("dtype", ctypes.c_int32), ("heads", ctypes.c_int32),
                ("rows", ctypes.c_int32), ("d", ctypes.c_int32), ("row_stride", ctypes.c_int64),
                ("head_stride", ctypes.c_int64)]


class LfHsaArgs(ctypes.Structure):
    _fields_ = [("q", LfMat), ("k", LfMat), ("v", LfMat),
                ("f", ctypes.c_int32), ("n", ctypes.c_int32), ("b_q", ctypes.c_int32),
                ("b_kv", ctypes.c_int32), ("framewise", ctypes.c_int32),
                ("chunk_index", ctypes.c_int32), ("topk_frames", ctypes.c_int32),
                ("per_frame_mode", ctypes.c_int32), ("s_i_dev", ctypes.c_void_p),
                ("out", ctypes.c_void_p), ("out_dtype", ctypes.c_int32),
                ("out_row_stride", ctypes.c_int64), ("out_head_stride", ctypes.c_int64),
                ("lse", ctypes.c_void_p), ("err_flag", ctypes.c_void_p),
                ("attn_kernel", ctypes.c_int32), ("s_i_host", ctypes.c_double),
                ("skip_frames", ctypes.c_int32)]


_P = ctypes.c_void_p
_I = ctypes.c_int32
_SIGS = {
    "lf_version": ([], ctypes.c_int),
    "lf_strerror": ([ctypes.c_int], ctypes.c_char_p),
    "lf_last_error": ([], ctypes.c_char_p),
    "lf_pool_blocks": ([ctypes.POINTER(LfMat), LfTiling, _I, _P, ctypes.c_int64, _P], ctypes.c_int),
    "lf_compress": ([ctypes.POINTER(LfMat), ctypes.POINTER(LfMat), LfTiling, LfTiling, _I, _I, _P,
                     _P, _P, _P], ctypes.c_int),
    "lf_select": ([_P, _P, _P, _I, _I, _I, _I, _I, _I, _I, _I, _I, _P, _I, _I, _P, _P, _P, _P, _P,
                   _P, _P], ctypes.c_int),
    "lf_select_strided": ([_P, _P, ctypes.c_int64, _P, ctypes.c_int64, _I, _I, _I, _I, _I, _I, _I,
                           _I, _I, _P, _I, _I, _P, _P, _P, _P, _P, _P, _P], ctypes.c_int),
    "lf_select_plan": ([_P, _P, ctypes.c_int64, _P, ctypes.c_int64, _I, _I, _I, _I, _I, _I, _I,
                        _I, _I, _P, _I, _I, _P, _P, _P, _P, _P, LfTiling, LfTiling, _I, _I, _P,
                        _P, _P, _P], ctypes.c_int),
    "lf_pair_qblocks": ([_P, _P, _I, _I, _I, _I, _P, _P], ctypes.c_int),
    "lf_plan_tiles_paired": ([_P, _P, _I, _I, _I, LfTiling, LfTiling, _I, _I, _P, _P, _P, _P],
                             ctypes.c_int),
    "lf_attention_paired": ([ctypes.POINTER(LfMat), ctypes.POINTER(LfMat),
                             ctypes.POINTER(LfMat), LfTiling, _P, _P, _I, _I, _I, ctypes.c_float,
                             _P, _I, ctypes.c_int64, ctypes.c_int64, _P, _P, _I, _I, _P,
                             ctypes.c_size_t, _P, _P], ctypes.c_int),
    "lf_cag_plan": ([ctypes.c_double, ctypes.c_double, _I, _I, _I, _I, _I, _I, _I, _I, _P, _P, _P,
                     _P, _P, _P, _P], ctypes.c_int),
    "lf_plan_tile_rows": ([], ctypes.c_int),
    "lf_set_qtile_mode": ([_I], None),
    "lf_pool_chunk_k": ([ctypes.POINTER(LfMat), LfTiling, _I, _P, ctypes.c_int64, _P, ctypes.c_int64,
                         _P], ctypes.c_int),
    "lf_qtile_mode": ([LfTiling], ctypes.c_int),
    "lf_plan_tile_count": ([LfTiling], ctypes.c_int),
    "lf_plan_tiles": ([_P, _P, _I, _I, _I, LfTiling, LfTiling, _I, _I, _P, _P, _P], ctypes.c_int),
    "lf_attention": ([ctypes.POINTER(LfMat), ctypes.POINTER(LfMat), ctypes.POINTER(LfMat), LfTiling,
                      _P, _P, _I, _I, _I, ctypes.c_float, _P, _I, ctypes.c_int64, ctypes.c_int64,
                      _P, _P, _P], ctypes.c_int),
    "lf_attention_ex": ([ctypes.POINTER(LfMat), ctypes.POINTER(LfMat), ctypes.POINTER(LfMat),
                         LfTiling, _P, _P, _I, _I, _I, ctypes.c_float, _P, _I, ctypes.c_int64,
                         ctypes.c_int64, _P, _P, _I, _I, _P], ctypes.c_int),
    "lf_attention_ws": ([ctypes.POINTER(LfMat), ctypes.POINTER(LfMat), ctypes.POINTER(LfMat),
                         LfTiling, _P, _P, _I, _I, _I, ctypes.c_float, _P, _I, ctypes.c_int64,
                         ctypes.c_int64, _P, _P, _I, _I, _P, ctypes.c_size_t, _P], ctypes.c_int),
    "lf_attention_scratch_bytes": ([_I, LfTiling, _I], ctypes.c_size_t),
    "lf_set_option": ([_I, _I], ctypes.c_int),
    "lf_get_option": ([_I], ctypes.c_int),
    "lf_attention_kernel_choice": ([_I, _I, _I, _I], ctypes.c_int),
    "lf_hsa_workspace_bytes": ([ctypes.POINTER(LfHsaArgs)], ctypes.c_size_t),
    "lf_hsa_views": ([ctypes.POINTER(LfHsaArgs), _P] + [ctypes.POINTER(_P)] * 7 +
                     [ctypes.POINTER(_I), ctypes.POINTER(_I)], ctypes.c_int),
    "lf_hsa_forward": ([ctypes.POINTER(LfHsaArgs), _P, ctypes.c_size_t, _P], ctypes.c_int),
    "lf_select_fallbacks": ([_P, _I], ctypes.c_int),
    "lf_rowdot": ([_P, _I, _I, _P, _P, _P], ctypes.c_int),
    "lf_topk": ([_P, _I, _I, _P, _P], ctypes.c_int),
}

_lib = None


def load_library(path: str = LIB_PATH):
    """dlopen the library (no GPU needed) and declare every signature."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(
            f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = ctypes.CDLL(path)
    for name, (args, res) in _SIGS.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    _lib = lib
    return lib


def lib():
    """The library, for compute: also requires a CUDA device (no CPU fallback)."""
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2602_04789_b200 needs a CUDA (sm_100a) device; none is visible")
    return load_library()


def set_option(name: str, value: int) -> int:
    """Set a library option (LF_OPT_*); returns the previous value."""
    lb = load_library()
    o = OPTIONS[name]
    prev = int(lb.lf_get_option(o))
    check(lb.lf_set_option(o, int(value)))
    return prev


@contextlib.contextmanager
def option(name: str, value: int):
    """Library option `name` = value inside the block (tests and experiments;
    the library reads its environment knobs once, so setenv does not work)."""
    prev = set_option(name, value)
    try:
        yield
    finally:
        set_option(name, prev)


def check(status: int) -> None:
    if status == LF_OK:
        return
    msg = (_lib.lf_last_error() or b"").decode() or _lib.lf_strerror(status).decode()
    if status == LF_ERR_ZERO_ACTIVE_ROW:
        raise ZeroActiveRowError(msg)
    if status == LF_ERR_DEGENERATE:
        raise DegenerateScheduleError(msg)
    if status in (LF_ERR_INVALID,):
        raise ValueError(msg)
    if status == LF_ERR_UNSUPPORTED:
        raise NotImplementedError(msg)
    raise RuntimeError(f"lfattn: {msg}")


def stream_ptr(stream=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def mat(t: torch.Tensor) -> LfMat:
    """LfMat over a CUDA tensor of shape [H, L, d] (any strides, unit last stride)."""
    if t.dim() == 2:
        t = t.unsqueeze(0)
    if t.dim() != 3 or t.stride(2) != 1:
        raise ValueError(f"expected [H, L, d] with contiguous rows, got {tuple(t.shape)} {t.stride()}")
    if t.dtype == torch.bfloat16:
        dt = LF_BF16
    elif t.dtype == torch.float32:
        dt = LF_F32
    else:
        raise ValueError(f"unsupported dtype {t.dtype}")
    h, L, d = t.shape
    return LfMat(t.data_ptr(), dt, h, L, d, t.stride(1), t.stride(0) if h > 1 else L * t.stride(1))


def tiling(total: int, period: int, block: int) -> LfTiling:
    return LfTiling(int(total), int(period), int(block))
