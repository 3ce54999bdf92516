"""CPU-side checks of the C ABI library and the host logic (no GPU needed)."""

import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "lfattn.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(lf_[a-z_]+)\s*\(", text)))


def test_library_loads_and_exports_header_symbols():
    from paper_2602_04789_b200 import _lib
    lib = _lib.load_library()
    syms = declared_symbols()
    assert len(syms) >= 12
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_lib.EXPORTS)
    assert lib.lf_version() == 101
    assert lib.lf_strerror(4) == b"query-block row has no active key blocks"


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2602_04789_b200 as lf
    with pytest.raises(RuntimeError):
        lf.mean_pool(np.ones((4, 2), np.float32), 2)


def test_abi_rejects_bad_arguments_without_touching_device():
    from paper_2602_04789_b200 import _lib
    lib = _lib.load_library()
    # invalid plan arguments are rejected before any launch
    rc = lib.lf_cag_plan(0.95, 0.9, 7, 4, 3, 512, 64, 64, 1, 0, *([None] * 6), None)
    assert rc == _lib.LF_ERR_INVALID
    assert b"s_target" in lib.lf_last_error()
    rc = lib.lf_topk(None, 3, -1, None, None)
    assert rc == _lib.LF_ERR_INVALID


def test_tiling_matches_oracle():
    from oracle.lf_oracle import Tiling
    from paper_2602_04789_b200.device import TilingSpec
    for total, period, block in [(4680, 1560, 64), (4680, 4680, 64), (300, 100, 32), (90, 90, 40),
                                 (32760, 1560, 64), (129, 129, 16)]:
        a = TilingSpec(total, period, block)
        b = Tiling(total, period, block)
        assert a.count == b.count
        np.testing.assert_array_equal(a.bounds(), b.all_bounds())
        for row in range(0, total, 7):
            g = a.block_of(row)
            s, e = b.bounds(g)
            assert s <= row < e


def test_framewise_tile_spans_at_most_four_blocks():
    from paper_2602_04789_b200.device import TilingSpec
    assert TilingSpec(4680, 1560, 64).max_blocks_per_tile() == 4
    assert TilingSpec(4680, 4680, 64).max_blocks_per_tile() == 2


def test_mask_lists_round_trip():
    from paper_2602_04789_b200.attention import mask_lists
    from paper_2602_04789_b200.selection import mask_from_lists
    rng = np.random.default_rng(0)
    bits = rng.random((7, 13)) < 0.4
    bits[:, 10:] = True
    blocks, count = mask_lists(bits[:, :10])
    back = mask_from_lists(blocks[0], count[0], 13, 10)
    np.testing.assert_array_equal(back, bits)


def test_layout_and_mask_host_logic():
    import paper_2602_04789_b200 as lf
    lay = lf.ChunkLayout(f=3, n=128, b_q=64, b_kv=64, d=32, N=7)
    assert (lay.chunk_tokens, lay.q_blocks, lay.frame_kv_blocks) == (384, 6, 2)
    assert lay.context_tokens(2) == 768 and lay.k_blocks(2) == 12 and lay.total_blocks(2) == 12
    with pytest.raises(ValueError):
        lf.ChunkLayout(f=0, n=128, b_q=64, b_kv=64, d=32, N=7)
    with pytest.raises(ValueError):
        lay.check_chunk(8)
    m = lf.BlockMask.full(3, 4)
    assert m.popcount() == 12
    lazy = lf.BlockMask.lazy(lambda: np.eye(2, dtype=bool), 2, 2)
    assert (lazy.n_q, lazy.n_k) == (2, 2) and lazy.popcount() == 2


def test_selection_config_validation():
    import paper_2602_04789_b200 as lf
    assert lf.SelectionConfig(topk_frames=0).topk_frames == 0
    with pytest.raises(ValueError):
        lf.SelectionConfig(topk_frames=-1)
    with pytest.raises(ValueError):
        lf.SelectionConfig(block_budget_mode="greedy")
    with pytest.raises(ValueError):
        lf.SelectionConfig(current_chunk_policy="sparse")


def test_hsa_argument_errors_precede_device_work():
    import paper_2602_04789_b200 as lf
    lay = lf.ChunkLayout(f=1, n=64, b_q=64, b_kv=64, d=4, N=2)
    q = np.zeros((64, 4), np.float32)
    with pytest.raises(ValueError):
        lf.hsa_attention(q, q, q, 2, 1.0, lf.SelectionConfig(), lay)
    lay2 = lf.ChunkLayout(f=1, n=100, b_q=64, b_kv=64, d=4, N=2)
    with pytest.raises(ValueError):
        lf.hsa_attention(q, q, q, 1, 0.5, lf.SelectionConfig(), lay2)


def test_planner_host_helpers():
    import paper_2602_04789_b200 as lf
    assert [lf.round_half_up(x) for x in (0.5, 1.5, 2.4, -0.5, 50.4)] == [1, 2, 2, 0, 50]
    lay = lf.ChunkLayout(f=3, n=1536, b_q=64, b_kv=64, d=64, N=7)
    assert lay.total_blocks(7) == 504 and lf.chunk_block_budget(0.9, 7, lay) == 50
    stock = lf.ChunkLayout(f=3, n=512, b_q=64, b_kv=64, d=64, N=7)
    assert lf.s_max_for_chunk(2, stock) == 0.5
    with pytest.raises(ValueError):
        lf.allocate(0.95, 0.9, 7, 4, stock)
    with pytest.raises(ValueError):
        lf.allocate(0.5, 0.9, 6, 4, stock)
    t = lf.tv_bound(1, np.e ** 2, 0.0, 1.0)
    np.testing.assert_allclose(t, 8.0 / np.e, rtol=1e-12)


def test_plan_json_round_trip():
    import paper_2602_04789_b200 as lf
    lay = lf.ChunkLayout(f=3, n=512, b_q=64, b_kv=64, d=64, N=7)
    plan = lf.SparsityPlan(0.9, 0.98, 4, (1.0,) * 7, 0.17, (0.0,) * 7, (24,) * 7, (False,) * 7,
                           True, 0.2)
    text = lf.plan_to_json(plan, lay)
    back, lay2 = lf.plan_from_json(text)
    assert lay2 == lay and back == plan and lf.plan_to_json(back, lay2) == text


def test_reference_staged_for_gpu_box():
    """oracle/make_ref.py copies the pure-Python reference into oracle/_ref (unmodified)."""
    import filecmp
    from oracle import make_ref
    if not os.path.isdir(make_ref.SRC):
        pytest.skip("no /root/reference here (GPU box): the staged copy travels instead")
    d = make_ref.stage()
    assert d and make_ref.ref_path() == d
    names = sorted(x for x in os.listdir(make_ref.SRC) if x.endswith(".py"))
    match, mismatch, errors = filecmp.cmpfiles(make_ref.SRC, make_ref.DST, names, shallow=False)
    assert not mismatch and not errors and len(match) == len(names) == 8


def test_options_roundtrip_without_gpu():
    """lf_set_option / lf_get_option: the environment is read once, then the
    cached value is what launch paths use; unknown options are rejected."""
    from paper_2602_04789_b200 import _lib
    lib = _lib.load_library()
    for name, o in _lib.OPTIONS.items():
        prev = lib.lf_get_option(o)
        assert lib.lf_set_option(o, 3) == _lib.LF_OK and lib.lf_get_option(o) == 3
        with _lib.option(name, 1):
            assert lib.lf_get_option(o) == 1
        assert lib.lf_get_option(o) == 3
        lib.lf_set_option(o, prev)
    assert lib.lf_set_option(99, 0) == _lib.LF_ERR_INVALID
    assert lib.lf_get_option(99) == -2


def test_pool_chunk_k_rejects_bad_output_strides():
    """lf_pool_chunk_k validates its caller-provided output strides before any launch."""
    import ctypes
    from paper_2602_04789_b200 import _lib
    lib = _lib.load_library()
    H, f, n, d, b = 2, 3, 1560, 128, 64
    bpf = -(-n // b)
    k = _lib.LfMat(0x10000, _lib.LF_BF16, H, f * n, d, d, f * n * d)
    t = _lib.tiling(f * n, n, b)
    good_kb, good_kf = f * bpf * d, f * d
    for kb_s, kf_s, kb_p in ((good_kb - 2, good_kf, 0x20000), (good_kb, good_kf - 2, 0x20000),
                             (good_kb + 1, good_kf, 0x20000), (good_kb, good_kf, 0x20004)):
        rc = lib.lf_pool_chunk_k(ctypes.byref(k), t, bpf, kb_p, kb_s, 0x40000, kf_s, None)
        assert rc == _lib.LF_ERR_INVALID, (kb_s, kf_s, kb_p)
        assert b"head strides" in lib.lf_last_error()
