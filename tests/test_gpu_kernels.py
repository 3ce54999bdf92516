"""The attention kernel forced (LF_KERNEL_TILE: one query tile per CTA, two
softmax sets, split-KV tail) against the oracle on the same inputs (masks
bit-exact, outputs within the tolerance of test_gpu_parity.py), its bf16
epilogue and graph-replay determinism, and the kernel-choice ABI."""

import numpy as np
import pytest
import torch

from oracle import lf_oracle as O
from tests.test_gpu_parity import assert_close_attn

pytestmark = pytest.mark.gpu

TILE = 3


@pytest.fixture(scope="module")
def lf():
    import paper_2602_04789_b200 as lf
    return lf


def _run(lf, kernel, H, n, f, i, d, s_i, topk, seed, out_dtype=torch.float32, heads=None):
    lay = lf.ChunkLayout(f=f, n=n, b_q=64, b_kv=64, d=d, N=max(i, 7))
    cfg = lf.SelectionConfig(topk_frames=topk)
    q, k, v = O.synthetic_qkv(seed, f * n, i * f * n, d, heads=H)
    dev = torch.device("cuda")
    qd, kd, vd = (torch.from_numpy(a).to(dev, torch.bfloat16) for a in (q, k, v))
    pipe = lf.HsaPipeline(lay, H, i, cfg, framewise=True, out_dtype=out_dtype)
    pipe.attn_kernel = kernel
    out = pipe(qd, kd, vd, s_i)
    torch.cuda.synchronize()
    assert pipe.errors() == 0
    return pipe, out, (q, k, v)


@pytest.mark.parametrize("kernel", [TILE])
@pytest.mark.parametrize("H,i,s_i,topk", [(12, 7, 0.5, 6), (3, 14, 0.8, 6), (1, 5, 0.0, 12),
                                          (2, 3, 0.3, 2)])
def test_kernel_vs_oracle(lf, kernel, H, i, s_i, topk):
    # H = 1..3: every pair item is a tail item, split over many CTAs (>= 3 parts)
    n, f, d = 1560, 3, 128
    pipe, out, (q, k, v) = _run(lf, kernel, H, n, f, i, d, s_i, topk, seed=900 + H * 10 + i)
    out = out.cpu().numpy()
    masks = pipe.masks()
    for h in sorted({0, H - 1}):
        _, sel = O.select(q[h], k[h], i, s_i, f, n, 64, 64, topk, "global", framewise=True)
        np.testing.assert_array_equal(masks[h].bits, sel.bits)
        ref, _ = O.block_sparse_attention(q[h], k[h], v[h], sel.bits, O.q_tiling(f, n, 64, True),
                                          O.k_tiling(i, f, n, 64, True))
        assert_close_attn(out[h], ref, f"kernel {kernel} head {h}")


@pytest.mark.parametrize("kernel", [TILE])
@pytest.mark.parametrize("n,f,i,d,s_i,topk", [(256, 2, 3, 64, 0.3, 2), (1536, 3, 5, 128, 0.6, 3),
                                               (100, 1, 4, 64, 0.2, 2)])
def test_kernel_small_shapes(lf, kernel, n, f, i, d, s_i, topk):
    # config-1 shape (d = 64), the aligned 1536 layout, and a tiny ragged frame
    H = 2
    pipe, out, (q, k, v) = _run(lf, kernel, H, n, f, i, d, s_i, topk, seed=n + i)
    out = out.cpu().numpy()
    masks = pipe.masks()
    for h in range(H):
        _, sel = O.select(q[h], k[h], i, s_i, f, n, 64, 64, topk, "global", framewise=True)
        np.testing.assert_array_equal(masks[h].bits, sel.bits)
        ref, _ = O.block_sparse_attention(q[h], k[h], v[h], sel.bits, O.q_tiling(f, n, 64, True),
                                          O.k_tiling(i, f, n, 64, True))
        assert_close_attn(out[h], ref, f"kernel {kernel} n {n} head {h}")


@pytest.mark.parametrize("H", [12, 2])
def test_bf16_epilogue_matches_fp32(lf, H):
    # bf16 output (and, for H = 2, the split-KV merge path) equals the fp32
    # output rounded to bf16
    _, o32, _ = _run(lf, TILE, H, 1560, 3, 7, 128, 0.5, 6, seed=31)
    _, o16, _ = _run(lf, TILE, H, 1560, 3, 7, 128, 0.5, 6, seed=31, out_dtype=torch.bfloat16)
    assert torch.equal(o32.to(torch.bfloat16), o16)


def test_split_graph_replay_deterministic(lf):
    # split-KV tail merges: whichever part finishes last merges, the result is bitwise stable
    pipe, out, _ = _run(lf, TILE, 4, 1560, 3, 5, 128, 0.5, 6, seed=5, out_dtype=torch.bfloat16)
    first = out.clone()
    pipe.capture()
    for _ in range(4):
        pipe.replay()
    torch.cuda.synchronize()
    assert torch.equal(first, out)


def test_kernel_choice_is_reported(lf):
    from paper_2602_04789_b200 import _lib
    lib = _lib.lib()
    # the two-softmax-set tile kernel is the automatic choice at every shape
    for args in ((12, 4680, 4680, 0), (40, 4680, 4680, 0), (12, 4680, 4680, 226)):
        assert lib.lf_attention_kernel_choice(*args) == TILE
    # round 1's pair kernel (5) is gone: an explicit request for it is rejected
    with pytest.raises(Exception, match="attention kernel 5"):
        _run(lf, 5, 2, 256, 2, 3, 64, 0.3, 2, seed=3)


@pytest.mark.parametrize("i,s_i,topk", [(7, 0.5, 6), (14, 0.8, 6), (5, 0.0, 12)])
def test_plan_kernels_agree(lf, i, s_i, topk):
    # the 4-warp planner and the one-warp planner emit the same segment lists
    # (pads may carry a different, always valid, start row)
    from paper_2602_04789_b200 import _lib as L
    from paper_2602_04789_b200 import device as D
    from paper_2602_04789_b200.selection import tilings
    pipe, _, _ = _run(lf, TILE, 3, 1560, 3, i, 128, s_i, topk, seed=70 + i)
    lay = lf.ChunkLayout(f=3, n=1560, b_q=64, b_kv=64, d=128, N=max(i, 7))
    qt, kt = tilings(lay, i, True)
    P = (i - 1) * 3
    blocks, count, _, _ = pipe.selections()
    plans = []
    for warp in (0, 1):
        with L.option("plan_warp", warp):
            t = D.plan_tiles(blocks, count, qt, kt, P * lay.frame_kv_blocks)
            torch.cuda.synchronize()
            plans.append((t.segs.cpu().numpy(), t.seg_count.cpu().numpy()))
    (s0, c0), (s1, c1) = plans
    np.testing.assert_array_equal(c0, c1)
    for idx in np.ndindex(c0.shape):
        n = int(c0[idx])
        a, b = s0[idx][:n].copy(), s1[idx][:n].copy()
        pad = a[:, 1] == 0
        np.testing.assert_array_equal(pad, b[:, 1] == 0)
        a[pad, 0] = 0
        b[pad, 0] = 0
        np.testing.assert_array_equal(a, b)


def test_concurrent_calls_own_their_scratch(lf):
    """Two hot-path calls in flight at once on two streams, each with its own
    workspace (split-KV scratch included), give the results of running them
    one after the other (lfattn.h: one call in flight per workspace, no
    library-global scratch on the lf_hsa_forward path)."""
    H, n, f, i, d = 2, 1560, 3, 5, 128  # 2 heads: every item is a split tail item
    lay = lf.ChunkLayout(f=f, n=n, b_q=64, b_kv=64, d=d, N=7)
    cfg = lf.SelectionConfig(topk_frames=6)
    dev = torch.device("cuda")
    cases = []
    for seed, s_i in ((301, 0.5), (302, 0.7)):
        q, k, v = O.synthetic_qkv(seed, f * n, i * f * n, d, heads=H)
        t = [torch.from_numpy(a).to(dev, torch.bfloat16) for a in (q, k, v)]
        cases.append((t, s_i))
    seq = []
    for t, s_i in cases:
        pipe = lf.HsaPipeline(lay, H, i, cfg, framewise=True, out_dtype=torch.float32)
        seq.append(pipe(*t, s_i).clone())
    torch.cuda.synchronize()
    pipes = [lf.HsaPipeline(lay, H, i, cfg, framewise=True, out_dtype=torch.float32)
             for _ in cases]
    outs = [p.bind(*t, s_i) for p, (t, s_i) in zip(pipes, cases)]
    streams = [torch.cuda.Stream() for _ in cases]
    torch.cuda.synchronize()
    for _ in range(3):
        for p, s in zip(pipes, streams):
            with torch.cuda.stream(s):
                p.launch()
    torch.cuda.synchronize()
    for p, o, ref in zip(pipes, outs, seq):
        assert p.errors() == 0
        assert torch.equal(o, ref)


def test_rollouts_have_independent_attention_scratch(lf):
    from paper_2602_04789_b200 import _lib as L
    lay = lf.ChunkLayout(f=3, n=1560, b_q=64, b_kv=64, d=128, N=7)
    a, b = (lf.HsaRollout(lay, 2) for _ in range(2))
    assert a.scratch.data_ptr() != b.scratch.data_ptr()
    assert a.scratch.numel() == L.lib().lf_attention_scratch_bytes(2, L.tiling(4680, 1560, 64), 128)
    assert int(a.scratch.sum()) == 0


@pytest.mark.parametrize("i,s_i", [(7, 6 / 7), (7, 0.5)])
def test_pipeline_without_frames_is_bit_identical(lf, i, s_i):
    """HsaPipeline(keep_frames=False) (lf_hsa_args.skip_frames): the same output
    bits, blocks and counts as with the frame lists; at a past budget of 0 (the
    c2 plan) the frame ranking is skipped."""
    H, f, n, d = 2, 3, 1560, 128
    lay = lf.ChunkLayout(f=f, n=n, b_q=64, b_kv=64, d=d, N=7)
    cfg = lf.SelectionConfig(topk_frames=6)
    g = torch.Generator(device="cuda").manual_seed(100 + i)
    q = torch.randn((H, f * n, d), device="cuda", generator=g).to(torch.bfloat16)
    k = torch.randn((H, i * f * n, d), device="cuda", generator=g).to(torch.bfloat16)
    v = torch.randn((H, i * f * n, d), device="cuda", generator=g).to(torch.bfloat16)
    s_dev = torch.tensor([s_i], dtype=torch.float64, device="cuda")
    outs, sels = [], []
    for keep in (True, False):
        pipe = lf.HsaPipeline(lay, H, i, cfg, framewise=True, keep_frames=keep)
        outs.append(pipe(q, k, v, s_dev, s_host=s_i).clone())
        sels.append(pipe.selections())
    torch.cuda.synchronize()
    assert torch.equal(outs[0].view(torch.int16), outs[1].view(torch.int16))
    (b0, c0, f0, g0), (b1, c1, f1, g1) = sels
    assert f0 is not None and f1 is None
    assert torch.equal(c0, c1) and torch.equal(g0[:3], g1[:3])
    for h in range(H):
        for r in range(c0.shape[1]):
            m = int(c0[h, r])
            assert torch.equal(b0[h, r, :m], b1[h, r, :m])
    if s_i == 6 / 7:
        assert int(g0[1]) == 0
