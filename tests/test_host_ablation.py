"""Host helpers of the reference's ablation (rollout.py:333-374), checked with
the values of the reference's own tests (test_rollout.py:316-347)."""

import pytest

import paper_2602_04789_b200 as lf

LAYOUT = lf.ChunkLayout(f=3, n=128, b_q=64, b_kv=64, d=32, N=7)


def test_largest_remainder_split_exact():
    assert lf.largest_remainder_split(5, [1, 1, 1]) == [2, 2, 1]
    assert lf.largest_remainder_split(0, [3, 7]) == [0, 0]
    assert sum(lf.largest_remainder_split(17, [2, 5, 9])) == 17


def test_largest_remainder_split_validation():
    with pytest.raises(ValueError):
        lf.largest_remainder_split(-1, [1.0])
    with pytest.raises(ValueError):
        lf.largest_remainder_split(3, [0.0, 0.0])


def test_matched_budget_settings_example():
    sa, sb = lf.matched_budget_settings(LAYOUT, 7, 0.8)
    assert sa == [1, 12, 18, 24, 30, 36, 42]
    assert sb == [6, 12, 17, 23, 29, 35, 41]


def test_matched_budget_settings_totals_always_equal():
    for s in (0.25, 0.5, 0.9):
        sa, sb = lf.matched_budget_settings(LAYOUT, 5, s)
        assert sum(sa) == sum(sb)
        assert sa[0] < sb[0]


def test_matched_budget_settings_validation():
    with pytest.raises(ValueError):
        lf.matched_budget_settings(LAYOUT, 7, 0.0)
    with pytest.raises(ValueError):
        lf.matched_budget_settings(LAYOUT, 1, 0.5)
