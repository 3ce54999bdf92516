"""Pin the CPU oracle against the reference's recorded outputs (tests/golden/).

Bit-exact for pooling, top-k indices, masks and plan budgets; the reference's
own float tolerances elsewhere (1e-12 relative for plans, test_planner.py:
136-144; 1e-5 absolute for attention outputs, test_acceptance.py:47-75).
"""

import numpy as np
import pytest

from oracle import lf_oracle as O
from tests.golden_io import case_inputs, hsa_cases, load_json, load_npz, unpack_bits


def test_pool_bit_exact():
    g = load_npz("pool.npz")
    idx = 0
    while f"x{idx}" in g:
        out = O.mean_pool(g[f"x{idx}"], int(g[f"g{idx}"]))
        np.testing.assert_array_equal(out.view(np.uint32), g[f"out{idx}"].view(np.uint32))
        idx += 1
    assert idx >= 5
    np.testing.assert_array_equal(O.mean_pool(g["x_hand"], 3), g["out_hand"])


def test_topk_indices():
    for c in load_json("topk.json"):
        got = O.topk_indices(np.asarray(c["scores"], np.float64), c["k"])
        assert got.tolist() == c["indices"], c


@pytest.mark.parametrize("kind", ["aligned", "framewise"])
def test_selection_masks_bit_exact(kind):
    n_cases = 0
    for m, arr in hsa_cases(kind):
        if m["n"] > 1000 and kind == "framewise" and m["i"] > 2:
            continue  # keep the CPU suite fast; the GPU suite covers these
        q, k, v = case_inputs(m)
        views, sel = O.select(q, k, m["i"], m["s_i"], m["f"], m["n"], m["b_q"], m["b_kv"],
                              m["topk"], m["mode"], framewise=(kind == "framewise"))
        bits = unpack_bits(arr[f"bits{m['case']}"], m["nk"])
        np.testing.assert_array_equal(sel.bits, bits, err_msg=str(m))
        assert sel.clamped == m["clamped"]
        if m.get("has_views", kind == "framewise"):
            c = m["case"]
            for mine, key in ((views.q_block, "qb"), (views.k_block, "kb"), (views.k_frame, "kf")):
                np.testing.assert_array_equal(mine, arr[f"{key}{c}"], err_msg=f"{key} {m}")
        n_cases += 1
    assert n_cases > 10


@pytest.mark.parametrize("kind", ["aligned", "framewise"])
def test_hsa_outputs_match_reference(kind):
    checked = 0
    for m, arr in hsa_cases(kind):
        if not m.get("has_out") or m["n"] > 1000:
            continue
        q, k, v = case_inputs(m)
        out, sel, _ = O.hsa_attention(q, k, v, m["i"], m["s_i"], m["f"], m["n"], m["b_q"],
                                      m["b_kv"], m["topk"], m["mode"],
                                      framewise=(kind == "framewise"), threads=1)
        np.testing.assert_allclose(out, arr[f"out{m['case']}"], atol=1e-5, rtol=0)
        checked += 1
    assert checked >= 5


def test_block_sparse_attention_matches_reference():
    meta = load_json("attention.json")
    arr = load_npz("attention.npz")
    for m in meta:
        q, k, v = O.synthetic_qkv(m["seed"], m["rows"], m["keys"], m["d"])
        bits = unpack_bits(arr[f"bits{m['case']}"], m["nk"])
        qt = O.Tiling(m["rows"], m["rows"], m["b_q"])
        kt = O.Tiling(m["keys"], m["keys"], m["b_kv"])
        out, active = O.block_sparse_attention(q[0], k[0], v[0], bits, qt, kt, threads=1)
        assert active == m["active"]
        np.testing.assert_allclose(out, arr[f"out{m['case']}"], atol=1e-5, rtol=0)
        tok = O.token_oracle(q[0], k[0], v[0], bits, qt, kt)
        np.testing.assert_allclose(out, tok, atol=1e-5, rtol=0)


def test_plans_match_reference():
    for rec in load_json("plans.json"):
        c = rec["case"]
        p = O.allocate(c["st"], c["sb"], c["N"], c["T"], c["f"], c["n"], c["b"], c["d"],
                       first_chunk_dense=c.get("first_chunk_dense", True),
                       redistribute=c.get("redistribute", False))
        assert list(p.budgets) == rec["budgets"], c
        assert list(p.clamped) == rec["clamped"], c
        np.testing.assert_allclose(p.s, rec["s"], rtol=1e-12, atol=0)
        np.testing.assert_allclose(p.beta, rec["beta"], rtol=1e-12, atol=1e-300)
        np.testing.assert_allclose(p.alpha, rec["alpha"], rtol=1e-15)
        np.testing.assert_allclose(p.achieved, rec["achieved"], rtol=1e-12)


def test_stock_golden_values():
    # test_planner.py:31-35 / test_acceptance.py:155-158
    p = O.allocate(0.9, 0.98, 7, 4, 3, 512, 64, 64)
    np.testing.assert_allclose(p.s, (0.0, 0.5, 2 / 3, 0.75, 0.8, 5 / 6, 6 / 7), rtol=1e-12)
    np.testing.assert_allclose(p.beta, 0.17311058252534645, rtol=1e-12)
    np.testing.assert_allclose(p.achieved, 2 / 9, rtol=1e-12)
    assert p.budgets == (24,) * 7


def test_budget_rounding_golden():
    # test_planner.py:92-101: 504 candidates, keep 10% -> 50.4 -> 50
    total, past, clamped = O.chunk_budget(0.9, 7, 3, 1536, 64)
    assert total == 50 and past == 0 and clamped


def test_framewise_equals_reference_when_aligned():
    q, k, v = O.synthetic_qkv(3, 3 * 128, 4 * 3 * 128, 16)
    a = O.select(q[0], k[0], 4, 0.5, 3, 128, 64, 64, 2, "global", framewise=False)[1]
    b = O.select(q[0], k[0], 4, 0.5, 3, 128, 64, 64, 2, "global", framewise=True)[1]
    np.testing.assert_array_equal(a.bits, b.bits)


def test_ragged_rejected_without_extension():
    q, k, v = O.synthetic_qkv(3, 3 * 100, 2 * 3 * 100, 8)
    with pytest.raises(ValueError):
        O.select(q[0], k[0], 2, 0.5, 3, 100, 64, 64)
