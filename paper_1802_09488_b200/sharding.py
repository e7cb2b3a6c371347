"""Multi-GPU layout of the join, one process per GPU (``torchrun``): points
shard by contiguous range, the index is replicated, and the only collective is
one sum of the per-polygon counts (and of the six JoinStats counters).

The split is the reference's worker split (join.cpp:264-265): rank r of W owns
points [n*r/W, n*(r+1)/W); global point indices are ``base_index + local``
(join.cpp:66-67); the merge is the reference's (join.cpp:280-284) with an
all-reduce (NCCL between GPUs, gloo in the CPU tests) in place of the serial
map merge.  First ids, overflow records and CSR rows stay sharded:
concatenated in rank order they are the global result.  Nothing on the probe
path crosses GPUs.

(The single-process counterpart — one host thread per GPU behind ONE call —
is ``join.IndexGroup`` / ``gj_group_*``.)
"""
from __future__ import annotations

import numpy as np

from . import capi


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    return n * rank // world, n * (rank + 1) // world


def _dist():
    import torch.distributed as dist

    return dist if dist.is_available() and dist.is_initialized() else None


def rank_world() -> tuple[int, int]:
    d = _dist()
    return (d.get_rank(), d.get_world_size()) if d else (0, 1)


def allreduce_counts(counts):
    """Sum a per-polygon count tensor over all ranks, in place.  A no-op
    without an initialised process group."""
    d = _dist()
    if d:  # also with one rank: the collective then runs (trivially) through the same backend
        d.all_reduce(counts, op=d.ReduceOp.SUM)
    return counts


def allreduce_sum_u64(values: np.ndarray, device=None) -> np.ndarray:
    """Sum of a small uint64 array over all ranks (as int64 on the wire; counts
    stay far below 2^63).  ``device``: where the tensor lives for the collective
    (a CUDA device for NCCL, None = host for gloo)."""
    import torch

    d = _dist()
    a = np.ascontiguousarray(values, np.uint64)
    if not d or d.get_world_size() == 1:
        return a.copy()
    t = torch.from_numpy(a.view(np.int64).copy())
    if device is not None:
        t = t.to(device)
    d.all_reduce(t, op=d.ReduceOp.SUM)
    return t.cpu().numpy().view(np.uint64)


class ShardedJoin:
    """This rank's share of a join over all ranks of the process group.

    ``session``: a ``join.Session`` on this rank's replica of the index (each
    rank loads the GJX1 file into its own GPU), or any object with the same
    ``join_count`` signature (the CPU tests pass the C oracle).  Results that
    are reductions (per-polygon counts, JoinStats) come back global; per-point
    results (first ids, overflow records) come back for this rank's range, with
    GLOBAL point indices."""

    def __init__(self, session, n_ids: int, collective_device=None):
        self.session = session
        self.n_ids = int(n_ids)
        self.collective_device = collective_device
        self.rank, self.world = rank_world()

    def range_of(self, n: int) -> tuple[int, int]:
        return shard_range(n, self.rank, self.world)

    def join_count(self, points, mode=capi.GJ_MODE_BUNDLE, stats=None, want_ids: bool = False,
                   base_index: int = 0):
        """``points``: the WHOLE input (every rank sees the same array, e.g. a
        memory-mapped file); this rank joins its range only."""
        begin, end = self.range_of(len(points))
        return self.join_count_shard(points[begin:end], base_index + begin, mode, stats, want_ids)

    def join_count_shard(self, local_points, base_index: int, mode=capi.GJ_MODE_BUNDLE, stats=None,
                         want_ids: bool = False):
        """``local_points``: this rank's range, whose first point has global
        index ``base_index``.  Returns (global counts u64[n_ids], local first
        ids | None, local (overflow point, overflow id) | None); ``stats``
        (a ``join.JoinStats``) receives the GLOBAL counters."""
        from .join import JoinStats

        local_stats = JoinStats() if stats is not None else None
        counts, first, ovf = self.session.join_count(local_points, mode, stats=local_stats, want_ids=want_ids,
                                                     base_index=base_index)
        packed = np.zeros(self.n_ids + 6, np.uint64)
        packed[:self.n_ids] = counts[:self.n_ids]
        if local_stats is not None:
            packed[self.n_ids:] = local_stats.as_tuple()
        total = allreduce_sum_u64(packed, self.collective_device)  # the ONE collective of the path
        if stats is not None:
            for name, v in zip(("probes", "pip_tests", "false_hits", "solely_true_hits", "refinement_entered",
                                "candidate_refs"), total[self.n_ids:]):
                setattr(stats, name, getattr(stats, name) + int(v))
        return total[:self.n_ids], first, ovf
