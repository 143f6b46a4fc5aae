"""Batch-sharded data parallelism for the conv layer.

The minibatch is the only sharded dimension: rank r of G takes images
[r*N/G, (r+1)*N/G); updateOutput / updateGradInput are per-image independent and
need no communication; accGradParameters produces per-rank partial sums of
gradWeight / gradBias, so the single exchange step is an allreduce(sum) of those.
Each layer's gradients are packed into one flat bucket and all-reduced on a
communication stream that overlaps the next layer's backward kernels
(torch.distributed over NCCL/NVLink on GPUs; gloo on CPU for the tests).
"""
from __future__ import annotations

from typing import List, Optional, Sequence, Tuple

import torch
import torch.distributed as dist


def shard_range(n: int, rank: int, world: int) -> Tuple[int, int]:
    """[start, stop) of the images rank `rank` owns; remainders go to the low ranks."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} for world size {world}")
    base, extra = divmod(n, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


class GradBucket:
    """One flat buffer holding a layer's gradWeight and gradBias, so one collective
    moves both (fewer, larger messages)."""

    def __init__(self, shapes: Sequence[torch.Size], device, dtype=torch.float32):
        sizes = [int(torch.Size(s).numel()) for s in shapes]
        self.flat = torch.zeros(sum(sizes), device=device, dtype=dtype)
        self.views: List[torch.Tensor] = []
        off = 0
        for s, n in zip(shapes, sizes):
            self.views.append(self.flat[off:off + n].view(s))
            off += n


def allreduce_async(bucket: GradBucket, comm_stream: Optional["torch.cuda.Stream"] = None,
                    group=None):
    """Sum the bucket across ranks. On CUDA the collective is enqueued on `comm_stream`
    after the producer stream's current work, so it overlaps later compute; returns the
    event the consumer must wait on (None on CPU, where the call is synchronous)."""
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return None
    if bucket.flat.is_cuda and comm_stream is not None:
        ready = torch.cuda.Event()
        ready.record(torch.cuda.current_stream(bucket.flat.device))
        comm_stream.wait_event(ready)
        with torch.cuda.stream(comm_stream):
            dist.all_reduce(bucket.flat, op=dist.ReduceOp.SUM, group=group)
            done = torch.cuda.Event()
            done.record(comm_stream)
        return done
    dist.all_reduce(bucket.flat, op=dist.ReduceOp.SUM, group=group)
    return None
