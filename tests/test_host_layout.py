"""Layout handshake with the reference's own types (host only, no GPU).

``chunkattn.rollout`` rejects a backend whose ``.layout`` does not compare
equal to the rollout's layout (rollout.py:281-282); the backends, pipeline and
rollout driver must also accept the reference's ``ChunkLayout`` (it has no
``aligned`` property).
"""

from __future__ import annotations

import pytest

import paper_2602_04789_b200 as lf
from paper_2602_04789_b200.layout import as_layout, is_aligned


def _ref():
    from oracle.make_ref import import_reference
    try:
        return import_reference()
    except ImportError:
        pytest.skip("reference not staged in oracle/_ref")


def test_layout_equality_both_directions():
    R = _ref()
    for f, n, b, d, N in ((3, 1536, 64, 128, 7), (3, 1560, 64, 128, 21), (2, 256, 64, 64, 3)):
        ref = R.ChunkLayout(f=f, n=n, b_q=b, b_kv=b, d=d, N=N)
        ours = lf.ChunkLayout(f=f, n=n, b_q=b, b_kv=b, d=d, N=N)
        assert ours == ref and ref == ours
        assert not (ours != ref) and not (ref != ours)
        assert hash(ours) == hash(lf.ChunkLayout(f, n, b, b, d, N))
        other = R.ChunkLayout(f=f, n=n, b_q=b, b_kv=b, d=d, N=N + 1)
        assert ours != other and other != ours
        assert as_layout(ref) == ours and isinstance(as_layout(ref), lf.ChunkLayout)
        assert is_aligned(ref) == is_aligned(ours) == (n % b == 0)
    assert lf.ChunkLayout(3, 1536, 64, 64, 128, 7) != (3, 1536, 64, 64, 128, 7)
    with pytest.raises(TypeError):
        as_layout(object())


def test_backends_keep_the_callers_layout_object():
    R = _ref()
    ref = R.ChunkLayout(f=3, n=1560, b_q=64, b_kv=64, d=128, N=7)
    plan = R.allocate(0.9, 0.98, 7, 4, ref)  # the reference's plan object is accepted as is
    hsa = lf.HsaBackend(ref, plan, R.SelectionConfig())
    assert hsa.layout is ref and hsa.framewise  # 1560 % 64 != 0 -> framewise tiling
    for be in (lf.DenseBackend(ref), lf.FixedMaskBackend(ref, [5] * 7, seed=0), hsa):
        assert be.layout == ref
        assert getattr(be, "layout", None) == R.ChunkLayout(3, 1560, 64, 64, 128, 7)
