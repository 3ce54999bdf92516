"""Query-tile geometry 2: query blocks paired into tensor-core tiles by the
overlap of their selections (lf_pair_qblocks).  Regrouping only -- every row
still attends to exactly its own selection (attention.py:229-274):

* the pairing is a permutation of each head's query blocks (every block in
  exactly one tile half), deterministic, and pairs blocks with identical
  selections when they exist;
* the full pipeline (lf_hsa_forward) and the rollout driver under geometry 2
  give bit-exact masks and outputs within the bf16 tolerance of the oracle;
* it issues no more key tiles than adjacent pairing on these inputs.
"""

import numpy as np
import pytest
import torch

from oracle import lf_oracle as O
from tests.test_gpu_parity import assert_close_attn

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lf():
    import paper_2602_04789_b200 as lf
    return lf


def test_pairing_is_a_deterministic_permutation(lf):
    from paper_2602_04789_b200 import device as D
    rng = np.random.default_rng(5)
    H, nqb, cap, L = 3, 75, 150, 975
    blocks = np.full((H, nqb, cap), -1, np.int32)
    count = np.zeros((H, nqb), np.int32)
    for h in range(H):
        for r in range(nqb):
            c = int(rng.integers(0, cap))
            blocks[h, r, :c] = np.sort(rng.choice(L, c, replace=False))
            count[h, r] = c
    # head 1: blocks 3 and 40 select exactly the same keys -> they pair
    blocks[1, 40] = blocks[1, 3]
    count[1, 40] = count[1, 3] = max(count[1, 3], 60)
    blocks[1, 3, :60] = blocks[1, 40, :60] = np.arange(60)
    dev = torch.device("cuda")
    tb, tc = torch.from_numpy(blocks).to(dev), torch.from_numpy(count).to(dev)
    p1 = D.pair_qblocks(tb, tc, L).cpu().numpy()
    p2 = D.pair_qblocks(tb, tc, L).cpu().numpy()
    assert np.array_equal(p1, p2)
    for h in range(H):
        got = sorted(int(x) for x in p1[h] if x >= 0)
        assert got == list(range(nqb)), h
        assert (p1[h] < 0).sum() == 1  # 75 blocks -> 38 tiles, one empty half
    pairs = {tuple(sorted(p1[1, 2 * t:2 * t + 2])) for t in range(p1.shape[1] // 2)}
    assert (3, 40) in pairs


@pytest.mark.parametrize("chunk,s_i", [(7, 0.5), (7, 0.7), (14, 0.8)])
def test_select_plan_bitsets_pair_like_the_lists(lf, chunk, s_i):
    """lf_select_plan under geometry 2 pairs from the bitsets the selection
    kernel writes (staged in the segment buffer); lf_pair_qblocks gathers the
    lists.  Same pairing, and the plans built from it agree."""
    from paper_2602_04789_b200 import device as D
    H, f, n, d, topk = 3, 3, 1560, 128, 6
    bpf = -(-n // 64)
    qt = D.TilingSpec(f * n, n, 64)
    kt = D.TilingSpec(chunk * f * n, n, 64)
    P = (chunk - 1) * f
    g = torch.Generator(device="cuda").manual_seed(chunk)
    qb = torch.randn((H, qt.count, d), device="cuda", generator=g) * 0.125
    kb = torch.randn((H, kt.count, d), device="cuda", generator=g) * 0.125
    kf = torch.randn((H, P, d), device="cuda", generator=g) * 0.05
    with D.qtile_scope(2):
        sel, tiles, _ = D.select_plan(qb, kb, kf, bpf, chunk, f, topk, False, s_i, qt, kt,
                                      P * bpf)
        ref = D.pair_qblocks(sel.blocks, sel.count, P * bpf)
        ref_tiles = D.plan_tiles(sel.blocks, sel.count, qt, kt, P * bpf, qperm=ref)
    torch.cuda.synchronize()
    assert torch.equal(tiles.qperm, ref)
    assert torch.equal(tiles.seg_count, ref_tiles.seg_count)
    sc = tiles.seg_count.cpu().numpy()
    a_, b_ = tiles.segs.cpu().numpy(), ref_tiles.segs.cpu().numpy()
    for h in range(H):
        for t in range(sc.shape[1]):
            np.testing.assert_array_equal(a_[h, t, :sc[h, t]], b_[h, t, :sc[h, t]])


@pytest.mark.parametrize("i,s_i,topk,H", [(7, 0.5, 6, 3), (7, 0.7, 6, 2), (14, 0.8, 6, 2),
                                          (4, 0.3, 3, 2)])
def test_pipeline_paired_vs_oracle(lf, lfopt, i, s_i, topk, H):
    lfopt("qtile", 2)
    n, f, d = 1560, 3, 128
    lay = lf.ChunkLayout(f=f, n=n, b_q=64, b_kv=64, d=d, N=max(i, 7))
    q, k, v = O.synthetic_qkv(300 + i, f * n, i * f * n, d, heads=H)
    dev = torch.device("cuda")
    qd, kd, vd = (torch.from_numpy(a).to(dev, torch.bfloat16) for a in (q, k, v))
    pipe = lf.HsaPipeline(lay, H, i, lf.SelectionConfig(topk_frames=topk), framewise=True,
                          out_dtype=torch.float32)
    out = pipe(qd, kd, vd, s_i).cpu().numpy()
    torch.cuda.synchronize()
    assert pipe.errors() == 0
    masks = pipe.masks()
    for h in range(H):
        _, sel = O.select(q[h], k[h], i, s_i, f, n, 64, 64, topk, "global", framewise=True)
        np.testing.assert_array_equal(masks[h].bits, sel.bits)
        ref, _ = O.block_sparse_attention(q[h], k[h], v[h], sel.bits, O.q_tiling(f, n, 64, True),
                                          O.k_tiling(i, f, n, 64, True))
        assert_close_attn(out[h], ref, f"paired head {h}")


def test_rollout_paired_matches_blocks_geometry(lf):
    """The rollout driver under geometries 1 and 2: same masks, outputs equal to
    within the bf16 tolerance (different row grouping, same math per row), and
    geometry 2 issues no more key tiles."""
    import bench
    from paper_2602_04789_b200 import device as D
    H, f, n, d, N, i = 4, 3, 1560, 128, 7, 7
    lay = lf.ChunkLayout(f=f, n=n, b_q=64, b_kv=64, d=d, N=N)
    q, k, v = O.synthetic_qkv(77, f * n, i * f * n, d, heads=H)
    dev = torch.device("cuda")
    qd, kd, vd = (torch.from_numpy(a).to(dev, torch.bfloat16) for a in (q, k, v))
    res = {}
    for mode in (1, 2):
        D.set_qtile_mode(mode)
        try:
            ro = lf.HsaRollout(lay, H, cfg=lf.SelectionConfig(), framewise=True,
                               out_dtype=torch.float32)
            for c in range(1, i):
                sl = slice((c - 1) * f * n, c * f * n)
                ro.commit(kd[:, sl], vd[:, sl], c)
            cur = slice((i - 1) * f * n, i * f * n)
            pl = ro.prepare(qd, i, s_i=0.5)
            kk, vv = ro.kv_slot(i)
            kk.copy_(kd[:, cur])
            vv.copy_(vd[:, cur])
            out = ro.attend(pl).cpu().numpy()
            torch.cuda.synchronize()
            assert pl.qmode == mode
            sel = (pl.selection.blocks.cpu().numpy(), pl.selection.count.cpu().numpy())
            res[mode] = (out, sel, bench.issued_mma_flops(pl, d))
        finally:
            D.set_qtile_mode(-1)
    np.testing.assert_array_equal(res[1][1][1], res[2][1][1])
    cnt = res[1][1][1]
    for h in range(H):
        for r in range(cnt.shape[1]):
            np.testing.assert_array_equal(res[1][1][0][h, r, :cnt[h, r]],
                                          res[2][1][0][h, r, :cnt[h, r]])
    for h in range(H):
        assert_close_attn(res[2][0][h], res[1][0][h].astype(np.float64), f"head {h}")
    assert res[2][2] <= res[1][2], (res[1][2], res[2][2])
    print(f"issued tile FLOPs: blocks {res[1][2]:.3e}, paired {res[2][2]:.3e} "
          f"({100 * (res[2][2] / res[1][2] - 1):+.1f} %)")


def _pair_ref(blocks, count, L):
    """CPU restatement of pair_qblocks_kernel (pairing.cuh): overlaps, mutual-best
    rounds (key = overlap, nearer, lower index), tiles in serial-scan order."""
    H, n, _ = blocks.shape
    out = np.full((H, 2 * ((n + 1) // 2)), -1, np.int32)
    for h in range(H):
        sets = [set(int(b) for b in blocks[h, x, :count[h, x]] if 0 <= b < L) for x in range(n)]
        ov = [[min(len(sets[x] & sets[y]), 2047) for y in range(n)] for x in range(n)]
        mate = [-1] * n
        if any(sets):
            for _ in range(n):
                prop = [-1] * n
                for x in range(n):
                    if mate[x] >= 0:
                        continue
                    key = -1
                    for y in range(n):
                        if y != x and mate[y] < 0:
                            key = max(key, (ov[x][y] << 20) | ((1023 - abs(x - y)) << 10) | (1023 - y))
                    prop[x] = 1023 - (key & 1023) if key >= 0 else -1
                new = 0
                for x in range(n):
                    y = prop[x]
                    if y >= 0 and prop[y] == x:
                        mate[x] = y
                        new += x < y
                if new == 0:
                    break
        tiles, ul = [], []
        for x in range(n):
            if mate[x] > x:
                tiles.append((x, mate[x]))
            elif mate[x] < 0:
                ul.append(x)
                if len(ul) % 2 == 0:
                    tiles.append((ul[-2], ul[-1]))
        if len(ul) % 2:
            tiles.append((ul[-1], -1))
        out[h, :2 * len(tiles)] = np.asarray(tiles, np.int32).ravel()
    return out


@pytest.mark.parametrize("kind", ["random", "clustered", "empty"])
def test_pairing_matches_cpu_restatement(lf, kind):
    """Both pairing paths (lists: lf_pair_qblocks; bitsets + the overlap kernel:
    lf_select_plan) equal a CPU restatement of the mutual-best rounds."""
    from paper_2602_04789_b200 import device as D
    rng = np.random.default_rng({"random": 11, "clustered": 12, "empty": 13}[kind])
    H, nqb, cap, L = 2, 75, 150, 450
    blocks = np.full((H, nqb, cap), -1, np.int32)
    count = np.zeros((H, nqb), np.int32)
    if kind != "empty":
        for h in range(H):
            for r in range(nqb):
                if kind == "random":
                    c = int(rng.integers(0, cap))
                    sel = rng.choice(L, c, replace=False)
                else:  # groups of blocks share most of a frame range: long proposal chains
                    base = (r // 5) * 25 % L
                    pool = np.arange(base, base + 90) % L
                    c = int(rng.integers(40, 90))
                    sel = rng.choice(pool, c, replace=False)
                blocks[h, r, :c] = np.sort(sel)
                count[h, r] = c
    dev = torch.device("cuda")
    tb, tc = torch.from_numpy(blocks).to(dev), torch.from_numpy(count).to(dev)
    got = D.pair_qblocks(tb, tc, L).cpu().numpy()
    np.testing.assert_array_equal(got, _pair_ref(blocks, count, L))
