"""lf_select_plan (selection + tile plan of one step) and the top-k margin
certificate.

* frames and blocks equal to the oracle's restatement of selection.py:117-175
  on the same fp32 summaries, over both query-tile geometries, ragged and
  aligned tilings, d 64/128, global and per-frame budget modes, chunks up to
  22 and forced exact ties (duplicated summary rows); the tile plan equal to
  lf_plan_tiles of those lists;
* the margin certificate: per query block, min(selected score) -
  max(rejected score) of the frame and the block decision, in the
  compensated fp64 scores -- equal to the gap of the oracle's numpy scores to
  within their rounding, 0 where a forced tie sits on the boundary, and at the
  BASELINE shapes larger than the fp64 error of any summation order of the
  reference's dot products (d * 2^-53 * sum|k q|, doubled), so the reference
  (numpy/BLAS) must select the same sets.
"""

from __future__ import annotations

import zlib

import numpy as np
import pytest
import torch

from oracle import lf_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def D():
    from paper_2602_04789_b200 import device as D
    return D


def _summaries(seed, H, nqb, nkb, P, d, ties):
    rng = np.random.default_rng(seed)
    qb = rng.standard_normal((H, nqb, d)).astype(np.float32) * 0.125
    kb = rng.standard_normal((H, nkb, d)).astype(np.float32) * 0.125
    kf = rng.standard_normal((H, max(P, 1), d)).astype(np.float32) * 0.05
    if ties == "near":
        # rows one fp32 ulp apart: fp64 scores differ by ~1e-9, far inside the
        # fp32 screening bound, so the screen cannot decide and the exact
        # fallback must
        nudge = lambda x: np.nextafter(x, np.float32(np.inf), dtype=np.float32)
        kb[:, 1::5] = nudge(kb[:, 0::5][:, : kb[:, 1::5].shape[1]])
        kb[:, 2::5] = kb[:, 0::5][:, : kb[:, 2::5].shape[1]]
        if P > 3:
            kf[:, 1] = nudge(kf[:, 0])
            kf[:, 2] = kf[:, 0]
        return qb, kb, kf
    if ties:
        # duplicated rows: exactly equal scores, broken by the lower index
        kb[:, 1::5] = kb[:, 0::5][:, : kb[:, 1::5].shape[1]]
        if nkb >= 60:
            kb[:, 30:60] = kb[:, 0:30]
        if P > 2:
            kf[:, 1] = kf[:, 0]
            kf[:, P - 1] = kf[:, 0]
    return qb, kb, kf


def _gap(scores, chosen):
    sel = scores[chosen]
    rej = scores[~chosen]
    if sel.size == 0 or rej.size == 0:
        return np.inf
    return sel.min() - rej.max()


CASES = [
    # H, f, n, d, chunk, s_i, topk, framewise, qmode, ties, mode
    (3, 3, 1560, 128, 7, 0.5, 6, True, 0, False, "global"),
    (3, 3, 1560, 128, 7, 0.5, 6, True, 1, False, "global"),
    (2, 3, 1560, 128, 14, 0.8, 6, True, 1, True, "global"),
    (2, 3, 1560, 128, 21, 0.85, 6, True, 0, False, "global"),
    (2, 3, 1536, 128, 9, 0.6, 4, False, 0, True, "global"),
    (2, 3, 1536, 128, 3, 0.3, 2, False, 1, False, "global"),
    (2, 2, 256, 64, 3, 0.3, 2, False, 0, True, "global"),
    (2, 2, 256, 64, 3, 0.5, 2, False, 1, False, "per-frame"),
    (2, 3, 1560, 128, 9, 0.7, 6, True, 0, False, "per-frame"),
    (1, 3, 1560, 128, 7, 0.0, 18, True, 0, False, "global"),   # dense sweep point: keeps all
    (2, 3, 1560, 128, 7, 6 / 7, 6, True, 0, False, "global"),  # past budget 0 (config 2 plan)
    (1, 3, 1560, 128, 22, 0.9, 20, True, 1, False, "global"),  # 63 past frames, 500 candidates
]


@pytest.mark.parametrize("case", CASES)
def test_select_plan_vs_oracle_and_margins(D, case):
    H, f, n, d, chunk, s_i, topk, fw, qmode, ties, mode = case
    bpf = -(-n // 64)
    qt = D.TilingSpec(f * n, n if fw else f * n, 64)
    kt = D.TilingSpec(chunk * f * n, n if fw else chunk * f * n, 64)
    P = (chunk - 1) * f
    qb, kb, kf = _summaries(zlib.crc32(repr(case).encode()) & 0xffff, H, qt.count, kt.count, P, d, ties)
    dev = torch.device("cuda")
    tq, tk, tf = (torch.from_numpy(a).to(dev) for a in (qb, kb, kf))
    with D.qtile_scope(qmode):
        sel, tiles, mg = D.select_plan(tq, tk, tf, bpf, chunk, f, topk, mode == "per-frame", s_i,
                                       qt, kt, P * bpf, want_margin=True)
        ref_tiles = D.plan_tiles(sel.blocks, sel.count, qt, kt, P * bpf)
    torch.cuda.synchronize()
    assert torch.equal(tiles.seg_count, ref_tiles.seg_count)
    sc = tiles.seg_count.cpu().numpy()
    a_, b_ = tiles.segs.cpu().numpy(), ref_tiles.segs.cpu().numpy()
    for h in range(H):
        for t in range(sc.shape[1]):
            np.testing.assert_array_equal(a_[h, t, :sc[h, t]], b_[h, t, :sc[h, t]])
    cnt = sel.count.cpu().numpy()
    blocks = sel.blocks.cpu().numpy()
    frames = sel.frames.cpu().numpy()
    past_budget = int(sel.budget.cpu().numpy()[1])
    mg = mg.cpu().numpy()
    assert (mg >= 0).all() and not np.isnan(mg).any()
    if not ties:
        assert (mg > 0).all()
    for h in range(H):
        views = O.Views(qb[h], kb[h], kf[h][:P], bpf)
        for r in range(qt.count):
            p = O.frame_scores(views, r) if P else np.zeros(0)
            fr = O.select_frames(p, topk, chunk, f) if P else np.arange(0)
            past = [int(t) for t in fr if t < P]
            assert [int(t) for t in frames[h, r] if t >= 0] == past, (h, r)
            _, ids, _ = O.select_blocks(views, r, fr, past_budget, mode)
            assert blocks[h, r, :cnt[h, r]].tolist() == [int(x) for x in ids], (h, r)
            # the certificate is the gap of the fp64 scores (within their rounding)
            if 0 < min(topk, P) < P:
                chosen = np.zeros(P, bool)
                chosen[past] = True
                gap = _gap(p, chosen)
                assert abs(mg[h, r, 0] - gap) <= 1e-12 * max(1.0, np.abs(p).max()), (h, r)
            if mode == "global" and past and 0 < past_budget < len(past) * bpf:
                cand = np.concatenate([np.arange(t * bpf, (t + 1) * bpf) for t in past])
                o = kb[h][cand].astype(np.float64) @ qb[h][r].astype(np.float64)
                gap = _gap(o, np.isin(cand, ids))
                assert abs(mg[h, r, 1] - gap) <= 1e-12 * max(1.0, np.abs(o).max()), (h, r)


SCREEN_CASES = [
    # the screened hot path (no scores / margins requested) against the oracle;
    # near-ties and exact ties across the cut go through the exact fallback
    (3, 3, 1560, 128, 7, 0.7, 6, True, 0, False, "global"),
    (2, 3, 1560, 128, 7, 0.7, 6, True, 0, "near", "global"),
    (2, 3, 1560, 128, 14, 0.8, 6, True, 1, True, "global"),
    (2, 3, 1560, 128, 14, 0.8, 6, True, 1, "near", "global"),
    (2, 3, 1536, 128, 9, 0.6, 4, False, 0, "near", "per-frame"),
    (2, 3, 1560, 128, 9, 0.7, 6, True, 0, True, "per-frame"),
    (2, 2, 256, 64, 3, 0.3, 2, False, 0, "near", "global"),
    (1, 3, 1560, 128, 22, 0.9, 20, True, 1, "near", "global"),
]


@pytest.mark.parametrize("case", SCREEN_CASES)
@pytest.mark.parametrize("exact", [0, 1])
def test_screened_selection_vs_oracle(D, case, exact, lfopt):
    """Frames and blocks of the screened selection (fp32 scores + bounds,
    exact re-rank where the bounds do not decide) and of the all-exact option
    equal the oracle's, including rows one ulp apart and exact duplicates."""
    lfopt("select_exact", exact)
    H, f, n, d, chunk, s_i, topk, fw, qmode, ties, mode = case
    bpf = -(-n // 64)
    qt = D.TilingSpec(f * n, n if fw else f * n, 64)
    kt = D.TilingSpec(chunk * f * n, n if fw else chunk * f * n, 64)
    P = (chunk - 1) * f
    qb, kb, kf = _summaries(zlib.crc32(repr(case).encode()) & 0xffff, H, qt.count, kt.count, P, d, ties)
    dev = torch.device("cuda")
    tq, tk, tf = (torch.from_numpy(a).to(dev) for a in (qb, kb, kf))
    D.select_fallbacks(reset=True)
    with D.qtile_scope(qmode):
        sel, tiles, _ = D.select_plan(tq, tk, tf, bpf, chunk, f, topk, mode == "per-frame", s_i,
                                      qt, kt, P * bpf)
    torch.cuda.synchronize()
    fb = D.select_fallbacks(reset=True)
    if ties == "near" and not exact:
        # rows one ulp apart straddle some cut: the screen must have handed lists
        # to the exact path (whole or ambiguous items only)
        assert fb[0] + fb[1] > 0, fb
    if exact:
        assert fb == (0, 0, 0, 0), fb  # no screening at all
    cnt = sel.count.cpu().numpy()
    blocks = sel.blocks.cpu().numpy()
    frames = sel.frames.cpu().numpy()
    past_budget = int(sel.budget.cpu().numpy()[1])
    for h in range(H):
        views = O.Views(qb[h], kb[h], kf[h][:P], bpf)
        for r in range(qt.count):
            p = O.frame_scores(views, r) if P else np.zeros(0)
            fr = O.select_frames(p, topk, chunk, f) if P else np.arange(0)
            past = [int(t) for t in fr if t < P]
            assert [int(t) for t in frames[h, r] if t >= 0] == past, (h, r)
            _, ids, _ = O.select_blocks(views, r, fr, past_budget, mode)
            assert blocks[h, r, :cnt[h, r]].tolist() == [int(x) for x in ids], (h, r)


@pytest.mark.parametrize("kind", ["huge", "tiny", "mixed"])
@pytest.mark.parametrize("exact", [0, 1])
def test_screened_selection_extreme_magnitudes(D, kind, exact, lfopt):
    """Magnitudes where fp32 screening cannot work -- squares overflowing to
    inf (huge), products underflowing to zero (tiny), rows 40 orders of
    magnitude apart (mixed): the bounds or the finiteness check hand the
    lists to the exact path, and the selections equal the oracle's."""
    lfopt("select_exact", exact)
    H, f, n, d, chunk, s_i, topk = 2, 3, 1560, 128, 7, 0.7, 6
    bpf = -(-n // 64)
    qt = D.TilingSpec(f * n, n, 64)
    kt = D.TilingSpec(chunk * f * n, n, 64)
    P = (chunk - 1) * f
    qb, kb, kf = _summaries(zlib.crc32(kind.encode()) & 0xffff, H, qt.count, kt.count, P, d, False)
    if kind == "huge":
        kb *= np.float32(1e19)
        kf *= np.float32(1e19)
    elif kind == "tiny":
        kb *= np.float32(1e-25)
        kf *= np.float32(1e-25)
        qb *= np.float32(1e-25)
    else:
        rng = np.random.default_rng(7)
        kb *= (10.0 ** rng.integers(-20, 20, size=(H, kt.count, 1))).astype(np.float32)
        kf *= (10.0 ** rng.integers(-20, 20, size=(H, max(P, 1), 1))).astype(np.float32)
    dev = torch.device("cuda")
    tq, tk, tf = (torch.from_numpy(a).to(dev) for a in (qb, kb, kf))
    sel, _, _ = D.select_plan(tq, tk, tf, bpf, chunk, f, topk, False, s_i, qt, kt, P * bpf)
    torch.cuda.synchronize()
    cnt = sel.count.cpu().numpy()
    blocks = sel.blocks.cpu().numpy()
    frames = sel.frames.cpu().numpy()
    past_budget = int(sel.budget.cpu().numpy()[1])
    for h in range(H):
        views = O.Views(qb[h], kb[h], kf[h][:P], bpf)
        for r in range(qt.count):
            p = O.frame_scores(views, r)
            fr = O.select_frames(p, topk, chunk, f)
            past = [int(t) for t in fr if t < P]
            assert [int(t) for t in frames[h, r] if t >= 0] == past, (h, r)
            _, ids, _ = O.select_blocks(views, r, fr, past_budget, "global")
            assert blocks[h, r, :cnt[h, r]].tolist() == [int(x) for x in ids], (h, r)


def _fp64_bound(views, r, rows):
    """Worst |x - x'| between two fp64 summation orders of <row, q_r>:
    2 * d * 2^-53 * sum|k q| (Higham's gamma_d, twice)."""
    q = np.abs(views.q_block[r].astype(np.float64))
    a = np.abs(rows.astype(np.float64)) @ q
    return 2 * rows.shape[1] * 2.0 ** -53 * a.max()


@pytest.mark.parametrize("chunk,s_i", [(7, 0.5), (14, None), (21, None)])
def test_margin_certificate_baseline_shapes(D, chunk, s_i):
    """BASELINE configs 2/3 shapes, summaries pooled from seeded bf16 N(0,1)
    q/k: every decision's margin exceeds the fp64 reordering bound."""
    import paper_2602_04789_b200 as lf
    H, f, n, d = 4, 3, 1560, 128
    if s_i is None:
        plan = lf.allocate(0.9, 0.98, 21, 4, lf.ChunkLayout(f=f, n=n, b_q=64, b_kv=64, d=d, N=21))
        s_i = plan.s[chunk - 1]
    q, k, _ = O.synthetic_qkv(4000 + chunk, f * n, chunk * f * n, d, heads=H)
    dev = torch.device("cuda")
    qd, kd = (torch.from_numpy(a).to(dev, torch.bfloat16) for a in (q, k))
    qt = D.TilingSpec(f * n, n, 64)
    kt = D.TilingSpec(chunk * f * n, n, 64)
    bpf, P = 25, (chunk - 1) * f
    qb, kb, kf = D.compress(qd, kd, qt, kt, bpf, P)
    sel, _, mg = D.select_plan(qb, kb, kf, bpf, chunk, f, 6, False, s_i, qt, kt, P * bpf,
                               want_margin=True)
    mg = mg.cpu().numpy()
    fr = sel.frames.cpu().numpy()
    qbh, kbh, kfh = qb.cpu().numpy(), kb.cpu().numpy(), kf.cpu().numpy()
    worst = np.inf
    for h in range(H):
        views = O.Views(qbh[h], kbh[h], kfh[h], bpf)
        for r in range(qt.count):
            bf = _fp64_bound(views, r, kfh[h])
            assert mg[h, r, 0] > bf, (h, r, mg[h, r, 0], bf)
            worst = min(worst, mg[h, r, 0] / bf)
            if np.isfinite(mg[h, r, 1]):
                cand = np.concatenate([np.arange(t * bpf, (t + 1) * bpf) for t in fr[h, r] if t >= 0])
                bb = _fp64_bound(views, r, kbh[h][cand])
                assert mg[h, r, 1] > bb, (h, r, mg[h, r, 1], bb)
                worst = min(worst, mg[h, r, 1] / bb)
    print(f"chunk {chunk}: min margin / fp64 reordering bound = {worst:.3e}; "
          f"min frame margin {mg[..., 0].min():.3e}, min block margin {mg[..., 1].min():.3e}")


@pytest.mark.parametrize("chunk,s_i,qmode", [(7, 6 / 7, 0), (7, 6 / 7, 2), (7, 0.5, 0),
                                             (14, 0.8, 1), (1, 0.0, 0)])
def test_select_plan_without_frames(D, chunk, s_i, qmode):
    """want_frames=False (out_frames NULL): the same blocks, counts, budget and
    tile plan as with the frame list; at a past budget of 0 (the c2 plan) the
    frame ranking is skipped, and a forced geometry 2 still pairs (empty
    bitsets)."""
    H, f, n, d, topk = 2, 3, 1560, 128, 6
    bpf = -(-n // 64)
    qt = D.TilingSpec(f * n, n, 64)
    kt = D.TilingSpec(chunk * f * n, n, 64)
    P = (chunk - 1) * f
    qb, kb, kf = _summaries(31 + chunk, H, qt.count, kt.count, P, d, False)
    dev = torch.device("cuda")
    tq, tk, tf = (torch.from_numpy(a).to(dev) for a in (qb, kb, kf))
    with D.qtile_scope(qmode):
        a, ta, _ = D.select_plan(tq, tk, tf, bpf, chunk, f, topk, False, s_i, qt, kt, P * bpf)
        b, tb, _ = D.select_plan(tq, tk, tf, bpf, chunk, f, topk, False, s_i, qt, kt, P * bpf,
                                 want_frames=False)
    torch.cuda.synchronize()
    assert b.frames is None
    assert torch.equal(a.count, b.count) and torch.equal(a.budget[:3], b.budget[:3])
    cnt = a.count.cpu()
    for h in range(H):
        for r in range(qt.count):
            c = int(cnt[h, r])
            assert torch.equal(a.blocks[h, r, :c], b.blocks[h, r, :c])
    assert torch.equal(ta.seg_count, tb.seg_count)
    sc = ta.seg_count.cpu()
    for h in range(H):
        for t in range(sc.shape[1]):
            assert torch.equal(ta.segs[h, t, :sc[h, t]], tb.segs[h, t, :sc[h, t]])
    if ta.qperm is not None:
        assert torch.equal(ta.qperm, tb.qperm)
    if chunk == 7 and s_i == 6 / 7:
        assert int(a.budget[1]) == 0 and int(cnt.sum()) == 0
