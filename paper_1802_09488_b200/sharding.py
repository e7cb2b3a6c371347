"""Multi-GPU layout of the join: points shard by contiguous range, the index is
replicated, and the only collective is one sum of the per-polygon counts.

The split is the reference's worker split (join.cpp:264-265): rank r of W owns
points [n*r/W, n*(r+1)/W); global point indices are ``base_index + local``
(join.cpp:66-67).  Nothing on the probe path crosses GPUs.
"""
from __future__ import annotations


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    return n * rank // world, n * (rank + 1) // world


def allreduce_counts(counts):
    """Sum a per-polygon count tensor over all ranks (NCCL on GPUs, gloo in the
    CPU tests).  A no-op without an initialised process group."""
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(counts, op=dist.ReduceOp.SUM)
    return counts
