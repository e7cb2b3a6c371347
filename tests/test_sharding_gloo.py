"""The multi-GPU path on CPU: world_size-2 gloo processes shard points by
contiguous range exactly as bench.py does (the reference's worker split,
join.cpp:264-265), each joins its shard, and ONE all-reduce sums the
per-polygon counts.  The per-shard join here is the C oracle (test
infrastructure standing in for the GPU kernel); what is under test is the
host logic: range partition, global point indices via base_index, the count
reduction, and shard-count independence of the result."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1802_09488_b200 import sharding
from tests import golden_util


def test_shard_ranges_cover_and_match_reference_split():
    for n in (0, 1, 7, 100, 12345):
        for world in (1, 2, 3, 7, 8):
            ranges = [sharding.shard_range(n, r, world) for r in range(world)]
            assert ranges[0][0] == 0 and ranges[-1][1] == n
            for (a, b), (c, d) in zip(ranges, ranges[1:]):
                assert b == c and a <= b
            assert ranges == [(n * r // world, n * (r + 1) // world) for r in range(world)]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, name, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    fx = golden_util.load(name)
    ox = golden_util.oracle_index(fx)
    pts = fx["points"]
    begin, end = sharding.shard_range(len(pts), rank, world)
    pi, pid, stats, counts = ox.join(pts[begin:end], approx=False, base_index=begin)
    total = sharding.allreduce_counts(torch.from_numpy(counts.astype(np.int64)))
    st = sharding.allreduce_counts(torch.from_numpy(stats.astype(np.int64)))
    # pairs stay sharded: concatenation in rank order is the global order
    gathered = [None] * world
    dist.all_gather_object(gathered, (pi, pid))
    if rank == 0:
        np.savez(out_path, counts=total.numpy(), stats=st.numpy(),
                 pi=np.concatenate([g[0] for g in gathered]), pid=np.concatenate([g[1] for g in gathered]),
                 ids=ox.count_ids)
    dist.destroy_process_group()


@pytest.mark.parametrize("name", ["join_small_exact", "cfg3_tess16_exact_trained"])
def test_two_rank_join_equals_single(tmp_path, name):
    out = tmp_path / "r.npz"
    mp.spawn(_worker, args=(2, _free_port(), name, str(out)), nprocs=2, join=True)
    got = np.load(out)
    fx = golden_util.load(name)
    epi, epid = golden_util.pairs_of(fx, "exact")
    assert np.array_equal(got["pi"], epi) and np.array_equal(got["pid"], epid)
    assert tuple(got["stats"]) == tuple(int(v) for v in fx["exact_stats"])
    want = np.bincount(np.searchsorted(got["ids"], epid), minlength=len(got["ids"]))
    assert np.array_equal(got["counts"], want)
