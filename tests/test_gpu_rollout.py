"""GPU rollout driver with incremental summary cache vs the per-call pipeline and the oracle."""

import numpy as np
import pytest
import torch

from oracle import lf_oracle as O

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,f,d,N,topk,plan", [(1560, 3, 128, 5, 6, (0.3, 0.6)),
                                               (256, 2, 64, 4, 2, (0.3, 0.5))])
def test_rollout_cache_matches_pipeline_and_oracle(n, f, d, N, topk, plan):
    import paper_2602_04789_b200 as lf
    from paper_2602_04789_b200.rollout import HsaRollout
    H = 2
    lay = lf.ChunkLayout(f=f, n=n, b_q=64, b_kv=64, d=d, N=N)
    pl = lf.allocate(plan[0], plan[1], N, 4, lay)
    cfg = lf.SelectionConfig(topk_frames=topk)
    ro = HsaRollout(lay, H, pl, cfg, out_dtype=torch.float32)
    dev = torch.device("cuda")
    L = f * n
    # clean K/V per chunk and the current chunk's (noisy) q/k/v per step
    clean = [O.synthetic_qkv(100 + i, L, L, d, heads=H) for i in range(N)]
    fw = not lay.aligned
    for i in range(1, N + 1):
        q, kc, vc = O.synthetic_qkv(500 + i, L, L, d, heads=H)
        qd, kcd, vcd = (torch.from_numpy(a).to(dev, torch.bfloat16) for a in (q, kc, vc))
        out = ro.step(qd, kcd, vcd, i).cpu().numpy()
        # same call through the per-call pipeline on the concatenated context
        kfull = np.concatenate([clean[t][1] for t in range(i - 1)] + [kc], axis=1)
        vfull = np.concatenate([clean[t][2] for t in range(i - 1)] + [vc], axis=1)
        kd, vd = (torch.from_numpy(a).to(dev, torch.bfloat16) for a in (kfull, vfull))
        pipe = lf.HsaPipeline(lay, H, i, cfg, framewise=fw, out_dtype=torch.float32)
        # s_host: both paths then pick the same query-tile geometry (bit-equal outputs)
        ref_gpu = pipe(qd, kd, vd, pl.s_device(i), s_host=float(pl.s[i - 1])).cpu().numpy()
        np.testing.assert_array_equal(out, ref_gpu)
        masks = pipe.masks()
        for h in range(H):
            _, sel = O.select(q[h], kfull[h], i, pl.s[i - 1], f, n, 64, 64, topk, "global",
                              framewise=fw)
            np.testing.assert_array_equal(masks[h].bits, sel.bits)
        # commit the clean chunk (rollout.py:306-308)
        ro.commit(torch.from_numpy(clean[i - 1][1]).to(dev, torch.bfloat16),
                  torch.from_numpy(clean[i - 1][2]).to(dev, torch.bfloat16), i) if i < N else None
    assert int(ro.err.item()) == 0
