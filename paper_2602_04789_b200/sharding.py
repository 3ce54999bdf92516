"""Multi-GPU plumbing for the hot path.

The hot path is independent per head (the reference is a per-head outer
loop), so one process per GPU owns a contiguous slice of heads
and the per-head outputs are all-gathered over NCCL into ``[H, Lq, d]``.
When the head count does not divide the world size (12 heads on 8 GPUs), the
ranks run independent videos instead (replicas, no collective).
"""

from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist


@dataclass(frozen=True)
class HeadShard:
    mode: str      # "single" | "headshard" | "replica"
    rank: int
    world: int
    heads: int     # total heads
    h0: int        # first owned head
    h1: int        # one past the last owned head

    @property
    def local_heads(self) -> int:
        return self.h1 - self.h0


def partition_heads(heads: int, world: int, rank: int) -> HeadShard:
    if world <= 1:
        return HeadShard("single", 0, 1, heads, 0, heads)
    if heads % world == 0:
        per = heads // world
        return HeadShard("headshard", rank, world, heads, rank * per, (rank + 1) * per)
    return HeadShard("replica", rank, world, heads, 0, heads)


def gather_heads(local: torch.Tensor, shard: HeadShard, out: torch.Tensor | None = None,
                 group=None) -> torch.Tensor:
    """All-gather per-head outputs [H/N, L, d] -> [H, L, d] (rank-major = head order)."""
    if shard.mode != "headshard":
        return local
    full_shape = (shard.heads,) + tuple(local.shape[1:])
    if out is None:
        out = torch.empty(full_shape, dtype=local.dtype, device=local.device)
    backend = dist.get_backend(group)
    if backend == "nccl":
        dist.all_gather_into_tensor(out, local.contiguous(), group=group)
    elif local.is_cuda:  # gloo with device tensors (functional checks): through host memory
        parts = [torch.empty(local.shape, dtype=local.dtype) for _ in range(shard.world)]
        dist.all_gather(parts, local.detach().cpu().contiguous(), group=group)
        out.copy_(torch.cat(parts, dim=0))
    else:  # gloo (CPU tests): list form
        parts = list(out.split(shard.local_heads, dim=0))
        dist.all_gather(parts, local.contiguous(), group=group)
    return out


def gather_heads_overlapped(local: torch.Tensor, shard: HeadShard, out: torch.Tensor,
                            comm_stream: torch.cuda.Stream, group=None) -> None:
    """gather_heads on ``comm_stream`` after the current stream's work so far:
    the next call's compute overlaps this call's all-gather over NVLink (the
    caller joins with ``current.wait_stream(comm_stream)`` before reading
    ``out``)."""
    if shard.mode != "headshard":
        return
    comm_stream.wait_stream(torch.cuda.current_stream())
    # both buffers are used on comm_stream: keep the caching allocator from
    # recycling them for the current stream while the all-gather runs
    local.record_stream(comm_stream)
    out.record_stream(comm_stream)
    with torch.cuda.stream(comm_stream):
        gather_heads(local, shard, out=out, group=group)
