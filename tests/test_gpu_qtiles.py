"""Block-aligned query tiles (lf_set_qtile_mode(1): two query blocks per
tensor-core tile, plan tile = four query blocks) against the oracle, and
against the 128-row geometry on the same inputs. The geometry only regroups
rows, so masks stay bit-exact and outputs stay inside the same tolerance."""

import numpy as np
import pytest
import torch

from oracle import lf_oracle as O
from tests.test_gpu_parity import assert_close_attn, _pipeline_case
from tests.test_gpu_kernels import _run, TILE
from tests import test_gpu_rollout

pytestmark = pytest.mark.gpu


@pytest.fixture
def lf():
    import paper_2602_04789_b200 as lf
    from paper_2602_04789_b200 import device
    device.set_qtile_mode(1)
    yield lf
    device.set_qtile_mode(-1)


def test_mode_and_tile_count(lf):
    from paper_2602_04789_b200 import device
    qt = device.TilingSpec(3 * 1560, 1560, 64)
    assert device.qtile_mode(qt) == 1
    from paper_2602_04789_b200 import _lib
    assert _lib.lib().lf_plan_tile_count(qt.abi()) == -(-qt.count // 4)
    # every tile holds two blocks, rows cover the chunk exactly once
    rows = [device.qtile_rows(qt, 1, t) for t in range(-(-qt.count // 2))]
    assert rows[0][0] == 0 and rows[-1][1] == qt.total
    assert all(a[1] == b[0] for a, b in zip(rows, rows[1:]))
    assert max(x1 - x0 for x0, x1 in rows) <= 128
    # 128-row blocks are not eligible
    assert device.qtile_mode(device.TilingSpec(1024, 1024, 128)) == 0


@pytest.mark.parametrize("H,i,s_i,topk", [(12, 7, 0.5, 6), (3, 14, 0.8, 6), (1, 5, 0.0, 12),
                                          (2, 3, 0.3, 2)])
def test_block_tiles_vs_oracle(lf, H, i, s_i, topk):
    n, f, d = 1560, 3, 128
    pipe, out, (q, k, v) = _run(lf, TILE, H, n, f, i, d, s_i, topk, seed=700 + H * 10 + i)
    out = out.cpu().numpy()
    masks = pipe.masks()
    for h in sorted({0, H - 1}):
        _, sel = O.select(q[h], k[h], i, s_i, f, n, 64, 64, topk, "global", framewise=True)
        np.testing.assert_array_equal(masks[h].bits, sel.bits)
        ref, _ = O.block_sparse_attention(q[h], k[h], v[h], sel.bits, O.q_tiling(f, n, 64, True),
                                          O.k_tiling(i, f, n, 64, True))
        assert_close_attn(out[h], ref, f"block tiles head {h}")


@pytest.mark.parametrize("n,f,i,d,s_i,topk", [(256, 2, 3, 64, 0.3, 2), (1536, 3, 5, 128, 0.6, 3),
                                               (100, 1, 4, 64, 0.2, 2), (1560, 1, 3, 64, 0.5, 2)])
def test_block_tiles_small_shapes(lf, n, f, i, d, s_i, topk):
    H = 2
    pipe, out, (q, k, v) = _run(lf, TILE, H, n, f, i, d, s_i, topk, seed=n + i + 1)
    out = out.cpu().numpy()
    masks = pipe.masks()
    for h in range(H):
        _, sel = O.select(q[h], k[h], i, s_i, f, n, 64, 64, topk, "global", framewise=True)
        np.testing.assert_array_equal(masks[h].bits, sel.bits)
        ref, _ = O.block_sparse_attention(q[h], k[h], v[h], sel.bits, O.q_tiling(f, n, 64, True),
                                          O.k_tiling(i, f, n, 64, True))
        assert_close_attn(out[h], ref, f"block tiles n {n} head {h}")


def test_block_tiles_close_to_row_tiles(lf):
    from paper_2602_04789_b200 import device
    H, n, f, i, d = 4, 1560, 3, 7, 128
    _, out1, _ = _run(lf, TILE, H, n, f, i, d, 0.7, 6, seed=31)
    device.set_qtile_mode(0)
    _, out0, _ = _run(lf, TILE, H, n, f, i, d, 0.7, 6, seed=31)
    a, b = out1.cpu().numpy(), out0.cpu().numpy()
    # same masks and math, different tile grouping: fp32 outputs agree to rounding
    assert np.abs(a - b).max() <= 2e-3 * max(1.0, np.abs(b).max())


@pytest.mark.parametrize("split", ["1", "3"])
def test_block_tiles_split_kv(lf, split, lfopt):
    lfopt("attn_split", int(split))
    _pipeline_case(lf, 3, 1560, 3, 4, 128, 0.5, 6, "global", seed=5, check_heads=(1,))


def test_block_tiles_config2_shape(lf):
    _pipeline_case(lf, 12, 1560, 3, 7, 128, 0.5, 6, "global", seed=78, check_heads=(0, 11))


def test_block_tiles_rollout(lf):
    test_gpu_rollout.test_rollout_cache_matches_pipeline_and_oracle(1560, 3, 128, 5, 6, (0.3, 0.6))


# ---------------------------------------------------------------- dynamic schedule
# The tile kernel fetches units from a global counter (reset by the last CTA)
# for block-aligned plans; the result must not depend on which CTA ran a unit.

@pytest.mark.parametrize("split", [None, "3"])
def test_dynamic_schedule_vs_oracle(lf, split, lfopt):
    lfopt("attn_sched", 1)
    if split:
        lfopt("attn_split", int(split))
    _pipeline_case(lf, 3, 1560, 3, 5, 128, 0.6, 6, "global", seed=55, check_heads=(0, 2))


def test_dynamic_schedule_graph_replay(lf, lfopt):
    lfopt("attn_sched", 1)
    lay = lf.ChunkLayout(f=3, n=1560, b_q=64, b_kv=64, d=128, N=7)
    H, i = 5, 6
    q, k, v = O.synthetic_qkv(6, 3 * 1560, i * 3 * 1560, 128, heads=H)
    dev = torch.device("cuda")
    qd, kd, vd = (torch.from_numpy(a).to(dev, torch.bfloat16) for a in (q, k, v))
    pipe = lf.HsaPipeline(lay, H, i, lf.SelectionConfig(), framewise=True)
    out = pipe.bind(qd, kd, vd, 0.5)
    pipe.launch()
    first = out.clone()
    pipe.capture()
    for _ in range(4):  # the unit counter must be back at zero after every launch
        pipe.replay()
        torch.cuda.synchronize()
        assert torch.equal(first, out)
    lfopt("attn_sched", 0)
    pipe.launch()
    torch.cuda.synchronize()
    assert torch.equal(first, out)  # static round-robin: same result
