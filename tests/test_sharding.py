"""World-size-2 gloo test of the head-sharded path (CPU).

Each rank computes its own heads with the CPU oracle (standing in for the
GPU kernels, which the -m gpu suite checks separately), then the outputs are
all-gathered exactly as bench.py / the sharded pipeline do, and compared with
the single-process result.
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
