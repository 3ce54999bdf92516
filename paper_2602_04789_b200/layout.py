"""Host-side geometry and result types (reference: attention.py:45-156).

Pure integer/bookkeeping code with the reference's names, fields and error
behaviour; no arithmetic on the data lives here.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Callable

import numpy as np

from .errors import ZeroActiveRowError  # noqa: F401  (re-export, attention.py:99)


def ceil_div(a: int, b: int) -> int:
    return -(-a // b)


LAYOUT_FIELDS = ("f", "n", "b_q", "b_kv", "d", "N")


def _layout_key(obj):
    """(f, n, b_q, b_kv, d, N) of any layout-like object, else None."""
    try:
        return tuple(int(getattr(obj, name)) for name in LAYOUT_FIELDS)
    except (AttributeError, TypeError, ValueError):
        return None


@dataclass(frozen=True, eq=False)
class ChunkLayout:
    """Tiling geometry for a chunked rollout (attention.py:45-96).

    f frames per chunk, n tokens per frame, b_q x b_kv tiles, head dim d,
    N chunks.  Derived counts use ceilings (contiguous tiling); the framewise
    ragged extension uses ``framewise_*`` helpers instead.

    Equality is by the six fields against ANY layout-like object, so the
    reference's own ``chunkattn.ChunkLayout`` and this one compare equal when
    they describe the same geometry: ``chunkattn.rollout`` checks
    ``backend.layout == layout`` (rollout.py:281-282).
    """

    f: int
    n: int
    b_q: int
    b_kv: int
    d: int
    N: int

    def __post_init__(self):
        for name in LAYOUT_FIELDS:
            if getattr(self, name) < 1:
                raise ValueError(f"layout field {name} must be >= 1, got {getattr(self, name)}")

    def __eq__(self, other):
        key = _layout_key(other)
        if key is None:
            return NotImplemented
        return key == _layout_key(self)

    def __ne__(self, other):
        eq = self.__eq__(other)
        return eq if eq is NotImplemented else not eq

    def __hash__(self):
        return hash(_layout_key(self))

    @property
    def chunk_tokens(self) -> int:
        return self.f * self.n

    @property
    def q_blocks(self) -> int:
        return ceil_div(self.f * self.n, self.b_q)

    @property
    def frame_kv_blocks(self) -> int:
        return ceil_div(self.n, self.b_kv)

    def context_tokens(self, i: int) -> int:
        self.check_chunk(i)
        return i * self.f * self.n

    def k_blocks(self, i: int) -> int:
        return ceil_div(self.context_tokens(i), self.b_kv)

    def total_blocks(self, i: int) -> int:
        self.check_chunk(i)
        return i * self.f * self.frame_kv_blocks

    def check_chunk(self, i: int) -> None:
        if not 1 <= i <= self.N:
            raise ValueError(f"chunk index {i} outside 1..{self.N}")

    # --- framewise ragged extension: frame-local block tiling
    @property
    def aligned(self) -> bool:
        return is_aligned(self)

    @property
    def frame_q_blocks(self) -> int:
        return ceil_div(self.n, self.b_q)

    def framewise_q_blocks(self) -> int:
        return self.f * self.frame_q_blocks

    def framewise_k_blocks(self, i: int) -> int:
        return self.total_blocks(i)


def is_aligned(layout) -> bool:
    """Frame-aligned tiling (the reference's selection precondition, selection.py:88-92);
    works on any layout-like object, the reference's ChunkLayout included."""
    return layout.n % layout.b_q == 0 and layout.n % layout.b_kv == 0


def as_layout(layout) -> ChunkLayout:
    """This package's ChunkLayout for any layout-like object (e.g. chunkattn.ChunkLayout)."""
    if isinstance(layout, ChunkLayout):
        return layout
    key = _layout_key(layout)
    if key is None:
        raise TypeError(f"not a chunk layout: {layout!r}")
    return ChunkLayout(*key)


class BlockMask:
    """Boolean tile grid: bits[r, c] marks (query block r, key block c) active
    (attention.py:103-138).  Masks produced on the GPU are materialised on the
    host lazily, the first time ``bits`` is read."""

    def __init__(self, bits):
        bits = np.asarray(bits)
        if bits.ndim != 2:
            raise ValueError(f"mask must be 2-D, got shape {bits.shape}")
        self._bits = bits.astype(bool, copy=False)
        self._loader = None
        self._shape = self._bits.shape

    @classmethod
    def lazy(cls, loader: Callable[[], np.ndarray], n_q: int, n_k: int) -> "BlockMask":
        obj = cls.__new__(cls)
        obj._bits = None
        obj._loader = loader
        obj._shape = (int(n_q), int(n_k))
        return obj

    @property
    def bits(self) -> np.ndarray:
        if self._bits is None:
            self._bits = np.asarray(self._loader(), dtype=bool)
            self._loader = None
        return self._bits

    @bits.setter
    def bits(self, value):
        self._bits = np.asarray(value).astype(bool, copy=False)
        self._shape = self._bits.shape

    @property
    def n_q(self) -> int:
        return self._shape[0]

    @property
    def n_k(self) -> int:
        return self._shape[1]

    @classmethod
    def full(cls, n_q: int, n_k: int) -> "BlockMask":
        return cls(np.ones((n_q, n_k), dtype=bool))

    def popcount(self) -> int:
        return int(self.bits.sum())

    def row_popcounts(self) -> np.ndarray:
        return self.bits.sum(axis=1)

    def to_pgm(self, path) -> None:
        """Binary PGM (P5), one pixel per tile, 255 = active (attention.py:133-138)."""
        header = f"P5\n{self.n_k} {self.n_q}\n255\n".encode("ascii")
        with open(path, "wb") as fh:
            fh.write(header)
            fh.write((self.bits.astype(np.uint8) * 255).tobytes())

    def __repr__(self):
        return f"BlockMask(n_q={self.n_q}, n_k={self.n_k})"


@dataclass
class AttnStats:
    """Cost accounting for one kernel call (attention.py:141-156).

    flop_estimate is the reference's nominal count active*b_q*b_kv*d*2;
    ``effective_flops`` (extra field) counts exact ragged extents, QK^T + PV.
    wall_time / select_time are GPU times from CUDA events (seconds).
    """

    active_tiles: int
    total_tiles: int
    flop_estimate: int
    wall_time: float
    select_time: float = 0.0
    budget_clamped: bool = False
    effective_flops: int = 0
