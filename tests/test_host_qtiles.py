"""Host logic of the query-tile geometry (no GPU): the automatic choice per
step and the block-aligned row ranges."""

from paper_2602_04789_b200 import device as D


def test_auto_choice_at_the_bench_configs():
    bpf = 25  # n = 1560, b = 64
    # c2 / c5_s85: (almost) no past blocks -> 128-row tiles
    assert D.auto_qtile_mode(6 / 7, 7, 3, bpf, 6) == 0
    assert D.auto_qtile_mode(0.85, 7, 3, bpf, 6) == 0
    # c3 (chunk 14, 25 past blocks per query block) -> block-aligned
    assert D.auto_qtile_mode(0.904632706980882, 14, 3, bpf, 6) == 1
    # c5_s70 (83 past blocks), c5_s50 (whole retrieved frames, 150) -> paired by overlap
    assert D.auto_qtile_mode(0.7, 7, 3, bpf, 6) == 2
    assert D.auto_qtile_mode(0.5, 7, 3, bpf, 6) == 2
    # c5_dense: every past block selected (topk covers all 18 frames) -> 128-row tiles
    assert D.auto_qtile_mode(0.0, 7, 3, bpf, 18) == 0
    # chunk 1 and unknown s_i
    assert D.auto_qtile_mode(0.0, 1, 3, bpf, 6) == 0
    assert D.auto_qtile_mode(None, 7, 3, bpf, 6) == 0


def test_block_aligned_rows_cover_the_chunk():
    for total, period, block in [(4680, 1560, 64), (512, 256, 64), (100, 100, 64), (4608, 1536, 64)]:
        qt = D.TilingSpec(total, period, block)
        nq = -(-qt.count // 2)
        rows = [D.qtile_rows(qt, 1, t) for t in range(nq)]
        assert rows[0][0] == 0 and rows[-1][1] == total
        assert all(a[1] == b[0] for a, b in zip(rows, rows[1:]))
        assert all(0 < x1 - x0 <= 128 for x0, x1 in rows)
        # tile boundaries are block boundaries
        starts = {int(s) for s, _ in qt.bounds()}
        assert all(x0 in starts for x0, _ in rows)


def test_c_abi_geometry_queries_on_host():
    # host-only entry points (no device work): forced mode, tile counts, eligibility
    from paper_2602_04789_b200 import _lib as L
    lib = L.load_library()  # no device needed for these
    qt = D.TilingSpec(3 * 1560, 1560, 64)
    try:
        lib.lf_set_qtile_mode(1)
        assert lib.lf_qtile_mode(qt.abi()) == 1
        assert lib.lf_plan_tile_count(qt.abi()) == -(-qt.count // 4)  # 75 blocks -> 19
        assert lib.lf_qtile_mode(D.TilingSpec(1024, 1024, 128).abi()) == 0
        lib.lf_set_qtile_mode(2)  # paired: same tile counts as block-aligned
        assert lib.lf_qtile_mode(qt.abi()) == 2
        assert lib.lf_plan_tile_count(qt.abi()) == -(-qt.count // 4)
        lib.lf_set_qtile_mode(0)
        assert lib.lf_qtile_mode(qt.abi()) == 0
        assert lib.lf_plan_tile_count(qt.abi()) == -(-qt.total // 256)
    finally:
        lib.lf_set_qtile_mode(-1)
