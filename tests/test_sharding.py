"""World-size-2 gloo tests of the head-sharded path.

* CPU: each rank computes its own heads with the CPU oracle, the outputs are
  all-gathered exactly as bench.py / the sharded pipeline do, and compared
  with the single-process result.
* GPU (-m gpu): each rank runs the CUDA pipeline on its heads (masks checked
  on the rank), the device outputs are gathered and compared with the oracle.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2602_04789_b200.sharding import gather_heads, partition_heads


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, H, result_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import lf_oracle as O
    f, n, i, d = 2, 128, 3, 16
    q, k, v = O.synthetic_qkv(31, f * n, i * f * n, d, heads=H)
    shard = partition_heads(H, world, rank)
    outs = []
    for h in range(shard.h0, shard.h1):
        out, _, _ = O.hsa_attention(q[h], k[h], v[h], i, 0.5, f, n, 64, 64, 2, "global",
                                    threads=1)
        outs.append(out)
    local = torch.from_numpy(np.stack(outs))
    full = gather_heads(local, shard)
    if rank == 0:
        result_q.put(full.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_partition_rules():
    s = partition_heads(12, 4, 3)
    assert (s.mode, s.h0, s.h1, s.local_heads) == ("headshard", 9, 12, 3)
    assert partition_heads(12, 8, 5).mode == "replica"
    assert partition_heads(40, 8, 7).h0 == 35
    assert partition_heads(12, 1, 0).mode == "single"


def test_gloo_world2_head_gather_matches_single_process():
    H, world = 4, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, H, q)) for r in range(world)]
    for p in procs:
        p.start()
    full = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    from oracle import lf_oracle as O
    f, n, i, d = 2, 128, 3, 16
    qq, kk, vv = O.synthetic_qkv(31, f * n, i * f * n, d, heads=H)
    for h in range(H):
        ref, _, _ = O.hsa_attention(qq[h], kk[h], vv[h], i, 0.5, f, n, 64, 64, 2, "global",
                                    threads=1)
        np.testing.assert_array_equal(full[h], ref)


def _gpu_worker(rank, world, port, H, result_q):
    """One rank of the head-sharded GPU path: its heads through the CUDA
    pipeline (HsaPipeline -> lf_hsa_forward), masks checked against the oracle
    on the rank, outputs all-gathered (gloo, host copies) into [H, Lq, d]."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import datetime
    dist.init_process_group("gloo", rank=rank, world_size=world,
                            timeout=datetime.timedelta(seconds=180))
    try:
        import paper_2602_04789_b200 as lf
        from oracle import lf_oracle as O
        torch.cuda.set_device(rank % torch.cuda.device_count())
        f, n, i, d, s_i = 3, 1560, 5, 128, 0.5
        q, k, v = O.synthetic_qkv(77, f * n, i * f * n, d, heads=H)
        shard = partition_heads(H, world, rank)
        sl = slice(shard.h0, shard.h1)
        dev = torch.device("cuda", torch.cuda.current_device())
        qd, kd, vd = (torch.from_numpy(np.ascontiguousarray(a[sl])).to(dev, torch.bfloat16)
                      for a in (q, k, v))
        lay = lf.ChunkLayout(f=f, n=n, b_q=64, b_kv=64, d=d, N=7)
        pipe = lf.HsaPipeline(lay, shard.local_heads, i, lf.SelectionConfig(), framewise=True,
                              out_dtype=torch.float32)
        out = pipe(qd, kd, vd, s_i)
        torch.cuda.synchronize()
        assert pipe.errors() == 0
        masks = pipe.masks()
        for j, h in enumerate(range(shard.h0, shard.h1)):
            _, sel = O.select(q[h], k[h], i, s_i, f, n, 64, 64, 6, "global", framewise=True)
            assert np.array_equal(masks[j].bits, sel.bits), f"rank {rank} head {h}"
        full = gather_heads(out.cpu(), shard)
        if rank == 0:
            result_q.put(full.numpy())
        dist.barrier()
    except Exception as exc:  # surface the rank's failure instead of a queue timeout
        result_q.put(f"rank {rank}: {exc!r}")
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_gloo_world2_gpu_head_shards_match_oracle():
    """World size 2, each rank running the CUDA kernels on its half of the
    heads (both on cuda:0 when the box has one GPU), gathered head-major."""
    H, world = 4, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gpu_worker, args=(r, world, port, H, q)) for r in range(world)]
    for p in procs:
        p.start()
    full = q.get(timeout=600)
    assert not isinstance(full, str), full
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    from oracle import lf_oracle as O
    from tests.test_gpu_parity import assert_close_attn
    f, n, i, d, s_i = 3, 1560, 5, 128, 0.5
    qq, kk, vv = O.synthetic_qkv(77, f * n, i * f * n, d, heads=H)
    for h in range(H):
        _, sel = O.select(qq[h], kk[h], i, s_i, f, n, 64, 64, 6, "global", framewise=True)
        ref, _ = O.block_sparse_attention(qq[h], kk[h], vv[h], sel.bits, O.q_tiling(f, n, 64, True),
                                          O.k_tiling(i, f, n, 64, True))
        assert_close_attn(full[h], ref, f"gathered head {h}")
