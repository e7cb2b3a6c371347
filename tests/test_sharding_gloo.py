"""The one-process-per-GPU path (``sharding.ShardedJoin``, what ``bench.py
--gpus N`` runs under torchrun): world_size-2 process groups shard the points by
contiguous range (the reference's worker split, join.cpp:264-265), each rank
joins its range with global point indices (base_index), and ONE all-reduce sums
the per-polygon counts and JoinStats; pairs stay sharded and concatenate in rank
order.  The result must equal the single-worker result of the reference fixture
— the reference's thread-count independence test (tests/test_join.cpp:200-214)
with ranks as the workers.

Here (no GPU) each rank joins its shard with the C oracle — test
infrastructure standing in for the kernel; what is under test is the host logic.
On a GPU box the ``gpu``-marked variant runs the same two ranks through the real
library (both on cuda:0 when the box has one GPU — their kernels do not wait on
one another), including first ids and overflow records."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1802_09488_b200 import capi, join, sharding
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


class _OracleSession:
    """``join.Session.join_count`` served by the C oracle (CPU stand-in for one rank's GPU)."""

    def __init__(self, ox):
        self.ox = ox

    def join_count(self, points, mode, stats=None, want_ids=False, base_index=0):
        assert not want_ids
        _, _, st, counts = self.ox.join(points, approx=mode == capi.GJ_MODE_APPROX, base_index=base_index,
                                        want_pairs=False)
        if stats is not None:
            stats._add(capi.Stats(*[int(v) for v in st]))
        return counts, None, None


def _worker(rank, world, port, name, out_path, use_gpu):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    fx = golden_util.load(name)
    pts = fx["points"]
    extra = {}
    if use_gpu:
        n_dev = capi.lib().gj_device_count()
        assert n_dev > 0, "the gpu-marked test needs a device: there is no CPU fallback"
        bundle = join.IndexBundle.load(golden_util.bundle_file(name), device=rank % n_dev)
        session, ids = bundle.session(), bundle.ids
    else:
        ox = golden_util.oracle_index(fx)
        session, ids = _OracleSession(ox), ox.count_ids
    sj = sharding.ShardedJoin(session, len(ids))
    assert (sj.rank, sj.world) == (rank, world)
    st = join.JoinStats()
    counts, _, _ = sj.join_count(pts, capi.GJ_MODE_EXACT, stats=st)
    begin, end = sj.range_of(len(pts))
    if use_gpu:  # per-point results stay sharded, with global point indices
        _, first, (ovf_pt, ovf_id) = sj.join_count(pts, capi.GJ_MODE_EXACT, want_ids=True)
        row_ptr, pid = session.join_pairs(pts[begin:end], capi.GJ_MODE_EXACT)
        pi = begin + np.repeat(np.arange(end - begin, dtype=np.uint64), np.diff(row_ptr.astype(np.int64)))
        extra = dict(first=first, ovf_pt=ovf_pt, ovf_id=ovf_id)
    else:
        pi, pid, _, _ = session.ox.join(pts[begin:end], approx=False, base_index=begin)
    gathered = [None] * world
    dist.all_gather_object(gathered, (pi, pid, extra))
    if rank == 0:
        more = {k: np.concatenate([g[2][k] for g in gathered]) for k in extra}
        np.savez(out_path, counts=counts, stats=np.array(st.as_tuple(), np.uint64),
                 pi=np.concatenate([g[0] for g in gathered]), pid=np.concatenate([g[1] for g in gathered]),
                 ids=ids, **more)
    dist.destroy_process_group()


def _run(tmp_path, name, use_gpu):
    out = tmp_path / "r.npz"
    mp.spawn(_worker, args=(2, _free_port(), name, str(out), use_gpu), nprocs=2, join=True)
    got = np.load(out)
    fx = golden_util.load(name)
    epi, epid = golden_util.pairs_of(fx, "exact")
    assert np.array_equal(got["pi"], epi) and np.array_equal(got["pid"], epid)
    assert tuple(int(v) for v in got["stats"]) == tuple(int(v) for v in fx["exact_stats"])
    want = np.bincount(np.searchsorted(got["ids"], epid), minlength=len(got["ids"]))
    assert np.array_equal(got["counts"], want)
    return got, fx, epi, epid


@pytest.mark.parametrize("name", ["join_small_exact", "cfg3_tess16_exact_trained"])
def test_two_rank_join_equals_single(tmp_path, name):
    _run(tmp_path, name, use_gpu=False)


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["join_small_exact", "cfg3_tess16_exact_trained", "cfg5_stars_scaled"])
def test_two_rank_join_on_gpu_equals_single(tmp_path, name):
    got, fx, epi, epid = _run(tmp_path, name, use_gpu=True)
    # first ids + overflow records of the two ranks, concatenated in rank order, rebuild the global pair list
    first, opt, oid = got["first"], got["ovf_pt"], got["ovf_id"]
    assert len(first) == len(fx["points"]) and np.all(np.diff(opt.astype(np.int64)) >= 0)
    inline = (first != capi.GJ_NO_MATCH) & (first != capi.GJ_DEFERRED)
    pts = np.concatenate([np.nonzero(inline)[0].astype(np.uint64), opt])
    ids = np.concatenate([first[inline] & ~np.uint32(capi.GJ_MORE_FLAG), oid])
    seq = np.concatenate([np.zeros(int(inline.sum()), np.int64), 1 + np.arange(len(opt), dtype=np.int64)])
    order = np.lexsort((seq, pts))
    assert np.array_equal(pts[order], epi) and np.array_equal(ids[order], epid)
