"""GPU parity: the sm_100a kernels vs the reference's recorded outputs and the oracle.

Bit-exact: pooled summaries, selected frames/blocks (masks), CAG budgets.
Tolerance (attention outputs, bf16 tensor-core path vs fp32/fp64 CPU):
    rel-L2 <= 1e-2  and  max-abs <= 1e-2 * max(1, max|ref|)
"""

import math

import numpy as np
import pytest
import torch

from oracle import lf_oracle as O
from tests.golden_io import case_inputs, hsa_cases, load_json, load_npz, unpack_bits

pytestmark = pytest.mark.gpu

REL_L2 = 1e-2
MAX_ABS = 1e-2


def assert_close_attn(out, ref, what=""):
    out = np.asarray(out, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    assert out.shape == ref.shape, (out.shape, ref.shape)
    assert np.isfinite(out).all(), what
    rel = np.linalg.norm(out - ref) / max(np.linalg.norm(ref), 1e-30)
    mab = np.abs(out - ref).max()
    assert rel <= REL_L2, f"{what} rel-L2 {rel:.3e}"
    assert mab <= MAX_ABS * max(1.0, np.abs(ref).max()), f"{what} max-abs {mab:.3e}"
    return rel, mab


@pytest.fixture(scope="module")
def lf():
    import paper_2602_04789_b200 as lf
    return lf


def test_library_is_loaded(lf):
    from paper_2602_04789_b200 import _lib
    lib = _lib.lib()
    assert lib.lf_version() == 101


def test_mean_pool_bit_exact(lf):
    g = load_npz("pool.npz")
    idx = 0
    while f"x{idx}" in g:
        out = lf.mean_pool(g[f"x{idx}"], int(g[f"g{idx}"]))
        np.testing.assert_array_equal(out.view(np.uint32), g[f"out{idx}"].view(np.uint32))
        idx += 1
    np.testing.assert_array_equal(lf.mean_pool(g["x_hand"], 3), g["out_hand"])


def test_topk_indices(lf):
    for c in load_json("topk.json"):
        got = lf.topk_indices(np.asarray(c["scores"], np.float64), c["k"]).indices
        assert got.tolist() == c["indices"], c


@pytest.mark.parametrize("pool_cfg", ["2x4", "4x4", "4x8", "8x8"])
@pytest.mark.parametrize("kind", ["aligned", "framewise"])
def test_compress_bit_exact(lf, kind, pool_cfg, lfopt):
    # every (consumer groups x ring stages) variant of the TMA pooling kernel
    lfopt("pool_cfg", {"2x4": 0, "4x4": 1, "4x8": 2, "8x8": 3}[pool_cfg])
    for m, arr in hsa_cases(kind):
        c = m["case"]
        if f"qb{c}" not in arr:
            continue
        lay = lf.ChunkLayout(f=m["f"], n=m["n"], b_q=m["b_q"], b_kv=m["b_kv"], d=m["d"], N=m["N"])
        q, k, _ = case_inputs(m)
        v = lf.compress(q, k, m["i"], lay, framewise=(kind == "framewise"))
        np.testing.assert_array_equal(v.q_block, arr[f"qb{c}"])
        np.testing.assert_array_equal(v.k_block, arr[f"kb{c}"])
        np.testing.assert_array_equal(v.k_frame, arr[f"kf{c}"])


@pytest.mark.parametrize("kind", ["aligned", "framewise"])
def test_hsa_masks_and_outputs(lf, kind):
    worst = 0.0
    for m, arr in hsa_cases(kind):
        lay = lf.ChunkLayout(f=m["f"], n=m["n"], b_q=m["b_q"], b_kv=m["b_kv"], d=m["d"], N=m["N"])
        cfg = lf.SelectionConfig(topk_frames=m["topk"], block_budget_mode=m["mode"])
        q, k, v = case_inputs(m)
        out, stats, mask = lf.hsa_attention(q, k, v, m["i"], m["s_i"], cfg, lay,
                                            framewise=(kind == "framewise"))
        bits = unpack_bits(arr[f"bits{m['case']}"], m["nk"])
        np.testing.assert_array_equal(mask.bits, bits, err_msg=str(m))
        assert stats.budget_clamped == m["clamped"]
        assert stats.active_tiles == int(bits.sum())
        if kind == "aligned":
            assert stats.total_tiles == m["total"] and stats.flop_estimate == m["flops"]
        if m.get("has_out"):
            rel, _ = assert_close_attn(out, arr[f"out{m['case']}"], str(m))
            worst = max(worst, rel)
    print(f"{kind}: worst rel-L2 {worst:.3e}")


def test_block_sparse_attention_golden(lf):
    meta = load_json("attention.json")
    arr = load_npz("attention.npz")
    for m in meta:
        q, k, v = O.synthetic_qkv(m["seed"], m["rows"], m["keys"], m["d"])
        bits = unpack_bits(arr[f"bits{m['case']}"], m["nk"])
        lay = lf.ChunkLayout(f=1, n=m["keys"], b_q=m["b_q"], b_kv=m["b_kv"], d=m["d"], N=1)
        out, stats = lf.block_sparse_attention(q[0], k[0], v[0], lf.BlockMask(bits), lay)
        assert stats.active_tiles == m["active"] and stats.total_tiles == m["total"]
        assert stats.flop_estimate == m["flops"]
        assert_close_attn(out, arr[f"out{m['case']}"], str(m))


def test_dense_attention(lf):
    q, k, v = O.synthetic_qkv(11, 300, 1000, 128)
    out = lf.dense_attention(q[0], k[0], v[0])
    assert_close_attn(out, O.dense_attention(q[0], k[0], v[0]))
    q, k, v = O.synthetic_qkv(12, 5, 1, 4)  # single key: output is that value row
    out = lf.dense_attention(q[0], k[0], v[0])
    np.testing.assert_allclose(out, np.repeat(v[0], 5, axis=0), atol=1e-2)


def test_zero_active_row_raises(lf):
    q, k, v = O.synthetic_qkv(13, 128, 128, 8)
    bits = np.ones((2, 2), bool)
    bits[1] = False
    lay = lf.ChunkLayout(f=1, n=128, b_q=64, b_kv=64, d=8, N=1)
    with pytest.raises(lf.ZeroActiveRowError):
        lf.block_sparse_attention(q[0], k[0], v[0], lf.BlockMask(bits), lay)


def test_excluded_tiles_have_no_influence(lf):
    # test_attention.py:163-176: perturbing masked keys leaves the output bit-identical
    q, k, v = O.synthetic_qkv(14, 128, 128, 64)
    bits = np.array([[True, False], [True, False]])
    lay = lf.ChunkLayout(f=1, n=128, b_q=64, b_kv=64, d=64, N=1)
    a, _ = lf.block_sparse_attention(q[0], k[0], v[0], lf.BlockMask(bits), lay)
    k2, v2 = k[0].copy(), v[0].copy()
    k2[64:] += 100.0
    v2[64:] -= 50.0
    b, _ = lf.block_sparse_attention(q[0], k2, v2, lf.BlockMask(bits), lay)
    np.testing.assert_array_equal(a, b)


def test_plans_on_device(lf):
    for rec in load_json("plans.json"):
        c = rec["case"]
        lay = lf.ChunkLayout(f=c["f"], n=c["n"], b_q=c["b"], b_kv=c["b"], d=c["d"], N=c["N"])
        p = lf.allocate(c["st"], c["sb"], c["N"], c["T"], lay,
                        first_chunk_dense=c.get("first_chunk_dense", True),
                        redistribute=c.get("redistribute", False))
        assert list(p.budgets) == rec["budgets"], c
        assert list(p.clamped) == rec["clamped"], c
        np.testing.assert_array_equal(np.asarray(p.alpha), np.asarray(rec["alpha"]))
        np.testing.assert_allclose(p.s, rec["s"], rtol=1e-12, atol=0)
        np.testing.assert_allclose(p.beta, rec["beta"], rtol=1e-12, atol=1e-300)
        np.testing.assert_allclose(p.achieved_flops_ratio, rec["achieved"], rtol=1e-12)


def _pipeline_case(lf, H, n, f, i, d, s_i, topk, mode, seed, check_heads, mask_heads=()):
    """HsaPipeline (lf_hsa_forward) on seeded inputs: masks of check_heads and
    mask_heads bit-exact against the oracle, outputs of check_heads in tolerance."""
    lay = lf.ChunkLayout(f=f, n=n, b_q=64, b_kv=64, d=d, N=max(i, 7))
    cfg = lf.SelectionConfig(topk_frames=topk, block_budget_mode=mode)
    q, k, v = O.synthetic_qkv(seed, f * n, i * f * n, d, heads=H)
    dev = torch.device("cuda")
    qd = torch.from_numpy(q).to(dev, torch.bfloat16)
    kd = torch.from_numpy(k).to(dev, torch.bfloat16)
    vd = torch.from_numpy(v).to(dev, torch.bfloat16)
    pipe = lf.HsaPipeline(lay, H, i, cfg, framewise=True, out_dtype=torch.float32)
    out = pipe(qd, kd, vd, s_i).cpu().numpy()
    torch.cuda.synchronize()
    assert pipe.errors() == 0
    masks = pipe.masks()
    fw = True
    for h in sorted(set(mask_heads) - set(check_heads)):
        _, sel = O.select(q[h], k[h], i, s_i, f, n, 64, 64, topk, mode, framewise=fw)
        np.testing.assert_array_equal(masks[h].bits, sel.bits, err_msg=f"head {h}")
    for h in check_heads:
        views, sel = O.select(q[h], k[h], i, s_i, f, n, 64, 64, topk, mode, framewise=fw)
        np.testing.assert_array_equal(masks[h].bits, sel.bits, err_msg=f"head {h}")
        ref, _ = O.block_sparse_attention(q[h], k[h], v[h], sel.bits, O.q_tiling(f, n, 64, fw),
                                          O.k_tiling(i, f, n, 64, fw))
        assert_close_attn(out[h], ref, f"head {h}")
    return pipe


@pytest.mark.parametrize("s_i,topk,mode", [(6 / 7, 6, "global"), (0.5, 6, "global"),
                                            (0.7, 6, "per-frame"), (0.0, 18, "global")])
def test_pipeline_config2_shape(lf, s_i, topk, mode):
    # BASELINE config 2: 12 heads x d128, n=1560 (framewise b=64), f=3, chunk 7
    _pipeline_case(lf, 12, 1560, 3, 7, 128, s_i, topk, mode, seed=77, check_heads=(0, 5, 11))


def test_pipeline_long_rollout_chunk14(lf):
    # BASELINE config 3 point: chunk 14 (39 past frames), past budget from the N=21 plan
    lay = lf.ChunkLayout(f=3, n=1560, b_q=64, b_kv=64, d=128, N=21)
    plan = lf.allocate(0.9, 0.98, 21, 4, lay)
    s14 = plan.s[13]
    _pipeline_case(lf, 4, 1560, 3, 14, 128, s14, 6, "global", seed=1414, check_heads=(0, 3))


def test_pipeline_long_rollout_chunk21(lf):
    # BASELINE config 3 at chunk 21 of the N=21 CAG plan: 60 past frames, past
    # budget 53; all 12 heads' masks bit-exact, outputs of two heads in tolerance
    lay = lf.ChunkLayout(f=3, n=1560, b_q=64, b_kv=64, d=128, N=21)
    plan = lf.allocate(0.9, 0.98, 21, 4, lay)
    assert plan.budgets[20] - 75 == 53
    pipe = _pipeline_case(lf, 12, 1560, 3, 21, 128, plan.s[20], 6, "global", seed=2121,
                          check_heads=(0, 11), mask_heads=range(12))
    assert int(pipe.selections()[3][1]) == 53


@pytest.mark.parametrize("s_i", [6 / 7, 0.5])
def test_pipeline_config4_heads40(lf, s_i):
    # BASELINE config 4: Wan-14B attention shape, 40 heads x d128 at chunk 7
    # (6/7 = the CAG plan's s_7: current chunk only; 0.5 selects past blocks)
    _pipeline_case(lf, 40, 1560, 3, 7, 128, s_i, 6, "global", seed=4040,
                   check_heads=(0, 17, 39), mask_heads=range(40))


def test_pipeline_config1_shape(lf):
    # BASELINE config 1: 2 heads, d 64, f=2, n=256, chunk 3
    for s_i in (0.0, 0.3, 0.5):
        _pipeline_case(lf, 2, 256, 2, 3, 64, s_i, 2, "global", seed=3, check_heads=(0, 1))


def test_pipeline_graph_replay_deterministic(lf):
    lay = lf.ChunkLayout(f=3, n=1560, b_q=64, b_kv=64, d=128, N=7)
    H, i = 4, 5
    q, k, v = O.synthetic_qkv(5, 3 * 1560, i * 3 * 1560, 128, heads=H)
    dev = torch.device("cuda")
    qd, kd, vd = (torch.from_numpy(a).to(dev, torch.bfloat16) for a in (q, k, v))
    pipe = lf.HsaPipeline(lay, H, i, lf.SelectionConfig(), framewise=True)
    out = pipe.bind(qd, kd, vd, 0.5)
    pipe.launch()
    first = out.clone()
    pipe.capture()
    for _ in range(3):
        pipe.replay()
    torch.cuda.synchronize()
    assert torch.equal(first, out)


@pytest.mark.parametrize("H,f,n,b,i,d", [(3, 3, 1560, 64, 4, 128), (2, 2, 256, 64, 3, 64),
                                         (2, 1, 100, 32, 5, 16), (1, 3, 1536, 64, 2, 128)])
def test_compress_bf16_frame_path_bit_exact(lf, H, f, n, b, i, d):
    # the fused bf16 frame-pooling kernel (hot path) vs the oracle's fp64 sequential pooling
    from paper_2602_04789_b200 import device as D
    q, k, _ = O.synthetic_qkv(99 + d, f * n, i * f * n, d, heads=H)
    k[:, 5, :] *= 3e4  # widen the exponent range of one block
    k = O.bf16_round(k)
    dev = torch.device("cuda")
    qd = torch.from_numpy(q).to(dev, torch.bfloat16)
    kd = torch.from_numpy(k).to(dev, torch.bfloat16)
    qt = D.TilingSpec(f * n, n, b)
    kt = D.TilingSpec(i * f * n, n, b)
    P = (i - 1) * f
    qb, kb, kf = D.compress(qd, kd, qt, kt, kt.per_period, P)
    for h in range(H):
        views = O.compress(q[h], k[h], i, f, n, b, b, framewise=True)
        np.testing.assert_array_equal(qb[h].cpu().numpy().view(np.uint32), views.q_block.view(np.uint32))
        np.testing.assert_array_equal(kb[h].cpu().numpy().view(np.uint32), views.k_block.view(np.uint32))
        np.testing.assert_array_equal(kf[h].cpu().numpy().view(np.uint32), views.k_frame.view(np.uint32))


@pytest.mark.parametrize("split", ["1", "2", "3", "4"])
def test_split_kv_merge(lf, split, lfopt):
    # the split-KV load balancing (parts merged by the last finisher) must not change results
    lfopt("attn_split", int(split))
    q, k, v = O.synthetic_qkv(21, 700, 3000, 128)
    out = lf.dense_attention(q[0], k[0], v[0])
    assert_close_attn(out, O.dense_attention(q[0], k[0], v[0]), f"split {split}")
    _pipeline_case(lf, 3, 1560, 3, 4, 128, 0.5, 6, "global", seed=4, check_heads=(1,))


@pytest.mark.parametrize("H,f,n,d", [(3, 3, 1560, 128), (2, 2, 256, 64)])
def test_pool_chunk_k_matches_compress(lf, H, f, n, d):
    # lf_pool_chunk_k (one launch, strided outputs into a cache) == lf_compress bit for bit
    import ctypes
    from paper_2602_04789_b200 import _lib as L, device as D
    dev = torch.device("cuda")
    L_ = f * n
    _, k, _ = O.synthetic_qkv(H * 7 + n, L_, L_, d, heads=H)
    kd = torch.from_numpy(k).to(dev, torch.bfloat16)
    kt = D.TilingSpec(L_, n, 64)
    bpf = -(-n // 64)
    _, kb_ref, kf_ref = D.compress(kd, kd, kt, kt, bpf, f)
    # outputs land in the middle of larger caches (head strides != dense)
    kb_cache = torch.full((H, 3 * f * bpf, d), 7.0, device=dev)
    kf_cache = torch.full((H, 3 * f, d), 7.0, device=dev)
    kb, kf = kb_cache[:, f * bpf:2 * f * bpf], kf_cache[:, f:2 * f]
    m = L.mat(kd)
    L.check(L.lib().lf_pool_chunk_k(ctypes.byref(m), kt.abi(), bpf, kb.data_ptr(), kb.stride(0),
                                    kf.data_ptr(), kf.stride(0), L.stream_ptr()))
    torch.cuda.synchronize()
    assert torch.equal(kb, kb_ref) and torch.equal(kf, kf_ref)
    assert torch.all(kb_cache[:, :f * bpf] == 7.0) and torch.all(kf_cache[:, 2 * f:] == 7.0)
    # a layout the one-launch path does not take reports UNSUPPORTED (callers pool twice)
    k32 = torch.from_numpy(k).to(dev)
    m32 = L.mat(k32)
    rc = L.lib().lf_pool_chunk_k(ctypes.byref(m32), kt.abi(), bpf, kb.data_ptr(), kb.stride(0),
                                 kf.data_ptr(), kf.stride(0), L.stream_ptr())
    assert rc == L.LF_ERR_UNSUPPORTED
