"""GPU tests at BASELINE.json's full sizes (configs[1] / configs[2]: 289
polygons, 100 M points), through size-independent properties of the join —
no CPU oracle can finish these sizes in seconds:

  * conservation: per-polygon counts == histogram of (first ids + overflow ids);
  * JoinStats identities: probes == n, the three probe outcomes partition n,
    candidate_refs bounds the refined pairs;
  * linearity / shard invariance: the join of the whole input equals the sum of
    the joins of its ranges (what the multi-GPU split relies on), and global
    point indices (base_index) only relabel;
  * exact ⊆ approx: refining can only remove pairs;
  * the device-resident and the host-buffer entry points agree.

The indexes are the bench's cached reference-built bundles (.cache/, built
offline by tools/build_bundles.py); the tests skip when the cache is absent."""
import numpy as np
import pytest

from paper_1802_09488_b200 import capi, join, synth
from tools import build_bundles

pytestmark = pytest.mark.gpu

N_FULL = 100_000_000


def _bundle(config):
    name = build_bundles.workload_name(config)
    if not build_bundles.have_bundle(name):
        pytest.skip(f"no cached index for config {config} (tools/build_bundles.py needs the reference)")
    return join.IndexBundle.load(build_bundles.bundle_file(name), device=0)


def _hist(bundle, first, ovf_id):
    """Per-slot histogram of every emitted pair: first ids (flag stripped) + overflow ids."""
    hit = first[first < capi.GJ_DEFERRED] & np.uint32(~capi.GJ_MORE_FLAG & 0xFFFFFFFF)
    ids = np.concatenate([hit, ovf_id])
    return np.bincount(np.searchsorted(bundle.ids, ids), minlength=len(bundle.ids)).astype(np.uint64)


def test_config2_full_size_properties():
    bundle = _bundle(2)
    s = bundle.session()
    pts = synth.points_for(2, N_FULL, None)
    assert pts.shape == (N_FULL, 2)
    st = join.JoinStats()
    counts, first, (ovf_pt, ovf_id) = s.join_count(pts, capi.GJ_MODE_APPROX, stats=st, want_ids=True)
    # conservation
    assert np.array_equal(counts, _hist(bundle, first, ovf_id))
    assert not np.any(first == capi.GJ_DEFERRED)  # approx mode defers nothing
    more = (first != capi.GJ_NO_MATCH) & ((first & capi.GJ_MORE_FLAG) != 0)
    assert np.array_equal(np.unique(ovf_pt), np.flatnonzero(more).astype(np.uint64))
    assert np.all(np.diff(ovf_pt.astype(np.int64)) >= 0)  # overflow records ascend by point
    # JoinStats identities (join.hpp:77-84)
    probes, pip_tests, false_hits, solely_true, refined, cand_refs = st.as_tuple()
    assert probes == N_FULL and pip_tests == 0
    assert false_hits + solely_true + refined == N_FULL
    assert false_hits == int(np.count_nonzero(first == capi.GJ_NO_MATCH))
    assert int(counts.sum()) >= N_FULL - false_hits and cand_refs >= refined
    # linearity over ranges, with global indices
    cut = 37_123_457  # not a multiple of any tile or chunk size
    c0, f0, (p0, i0) = s.join_count(pts[:cut], capi.GJ_MODE_APPROX, want_ids=True)
    c1, f1, (p1, i1) = s.join_count(pts[cut:], capi.GJ_MODE_APPROX, want_ids=True, base_index=cut)
    assert np.array_equal(c0 + c1, counts)
    assert np.array_equal(np.concatenate([f0, f1]), first)
    assert np.array_equal(np.concatenate([p0, p1]), ovf_pt) and np.array_equal(np.concatenate([i0, i1]), ovf_id)
    # count-only entry point agrees
    c_only, _, _ = s.join_count(pts, capi.GJ_MODE_APPROX)
    assert np.array_equal(c_only, counts)


def _cpu_counts(path, pts, exact):
    """Per-polygon counts of the CPU join on all host threads: the compiled reference's own
    join_count_per_polygon when oracle/_ref travelled with the repo, else the C oracle port."""
    import os
    from oracle import ref
    threads = os.cpu_count() or 1
    if ref.available():
        rb = ref.RefBundle.load(path)
        assert rb.approx != exact  # join_count_per_polygon takes the mode from the bundle (join.cpp:257)
        return rb.join_count(pts, threads), "reference"
    from tests import golden_util
    ox = golden_util.oracle_index(golden_util.parse_gjx(open(path, "rb").read()))
    return ox.join_count(pts, approx=not exact, threads=threads)[0], "port"


@pytest.mark.parametrize("config,exact", [(2, False), (3, True)])
def test_full_size_counts_equal_the_cpu_reference(config, exact):
    """BASELINE configs[1] (approx) and configs[2] (exact, trained, ~1 % of the points on
    edges / vertices) at their full 100 M points: the per-polygon counts of the GPU join —
    host-buffer call and device-resident call — equal the reference's multithreaded CPU
    join_count_per_polygon on ALL points, polygon by polygon."""
    import torch
    bundle = _bundle(config)
    path = build_bundles.bundle_file(build_bundles.workload_name(config))
    polys = synth.polygons_for(config, 1.0) if synth.SPECS[config].boundary_fraction > 0 else None
    pts = synth.points_for(config, N_FULL, polys)
    want, kind = _cpu_counts(path, pts, exact)
    assert sum(want.values()) >= N_FULL * 0.99
    got = join.join_count_per_polygon(bundle, pts)  # mode from the bundle, like the reference
    assert got == want, f"GPU counts differ from the CPU {kind} join"
    s = bundle.session()
    d_pts = torch.from_numpy(pts).cuda()
    d_counts = torch.zeros(len(bundle.ids), dtype=torch.int64, device="cuda")
    torch.cuda.synchronize()
    s.join_count_device(d_pts.data_ptr(), N_FULL, d_counts.data_ptr(), capi.GJ_MODE_BUNDLE, sync=True)
    c = d_counts.cpu().numpy()
    assert {int(bundle.ids[k]): int(c[k]) for k in np.nonzero(c)[0]} == want
    # and all GPUs of the box behind one call (one replica per device, at least two replicas)
    devices = list(range(capi.lib().gj_device_count()))
    fleet = join.IndexGroup.load(path, devices if len(devices) > 1 else [0, 0])
    assert join.join_count_per_polygon(fleet, pts, 0) == want
    fleet.close()
    bundle.close()


def test_config2_device_resident_equals_host_path():
    import torch
    bundle = _bundle(2)
    s = bundle.session()
    n = N_FULL
    pts = synth.points_for(2, n, None)
    d_pts = torch.from_numpy(pts).cuda()
    d_counts = torch.zeros(len(bundle.ids), dtype=torch.int64, device="cuda")
    d_stats = torch.zeros(6, dtype=torch.int64, device="cuda")
    d_first = torch.empty(n, dtype=torch.int32, device="cuda")
    torch.cuda.synchronize()  # the session has its own stream: torch's fills and copies must have landed
    s.join_count_device(d_pts.data_ptr(), n, d_counts.data_ptr(), capi.GJ_MODE_APPROX,
                        d_stats_ptr=d_stats.data_ptr(), d_first_id_ptr=d_first.data_ptr(), sync=True)
    st = join.JoinStats()
    counts, first, _ = s.join_count(pts, capi.GJ_MODE_APPROX, stats=st, want_ids=True)
    assert np.array_equal(d_counts.cpu().numpy().astype(np.uint64), counts)
    assert np.array_equal(d_first.cpu().numpy().view(np.uint32), first)
    assert tuple(int(v) for v in d_stats.cpu().numpy()) == st.as_tuple()
    # idempotence: a second launch over the same input adds exactly the same counts
    s.join_count_device(d_pts.data_ptr(), n, d_counts.data_ptr(), capi.GJ_MODE_APPROX, sync=True)
    assert np.array_equal(d_counts.cpu().numpy().astype(np.uint64), 2 * counts)


def test_config3_exact_is_subset_of_approx_full_size():
    bundle = _bundle(3)
    s = bundle.session()
    polys = synth.polygons_for(3, 1.0)
    pts = synth.points_for(3, N_FULL, polys)
    se, sa = join.JoinStats(), join.JoinStats()
    ce, fe, (pe, ie) = s.join_count(pts, capi.GJ_MODE_EXACT, stats=se, want_ids=True)
    ca, fa, (pa, ia) = s.join_count(pts, capi.GJ_MODE_APPROX, stats=sa, want_ids=True)
    assert np.array_equal(ce, _hist(bundle, fe, ie)) and np.array_equal(ca, _hist(bundle, fa, ia))
    assert np.all(ce <= ca)  # refinement only removes pairs
    # probe-side counters do not depend on the mode; pip_tests == candidate_refs in exact mode (join.cpp:100-118)
    assert se.as_tuple()[0] == sa.as_tuple()[0] == N_FULL
    assert se.as_tuple()[2:] == sa.as_tuple()[2:]
    assert se.as_tuple()[1] == se.as_tuple()[5] and sa.as_tuple()[1] == 0
    assert int(ca.sum()) - int(ce.sum()) <= se.as_tuple()[1]  # at most one pair lost per PIP test
    # a point with no approx match has no exact match; exact first ids are approx pairs of that point
    assert np.all(fe[fa == capi.GJ_NO_MATCH] == capi.GJ_NO_MATCH)
    single = (fa != capi.GJ_NO_MATCH) & ((fa & capi.GJ_MORE_FLAG) == 0) & (fe < capi.GJ_DEFERRED)
    assert np.array_equal(fe[single] & np.uint32(0x7FFFFFFF), fa[single])
    # shard invariance in exact mode
    cut = 61_000_003
    c0, _, _ = s.join_count(pts[:cut], capi.GJ_MODE_EXACT)
    c1, _, _ = s.join_count(pts[cut:], capi.GJ_MODE_EXACT, base_index=cut)
    assert np.array_equal(c0 + c1, ce)


def test_one_billion_points_in_one_launch():
    """BASELINE configs[3] scale (1 B points per join): one device-resident
    launch over 16 GB of points (the 100 M config-2 points tiled 10 times in
    HBM) gives exactly 10x the counts and the same first ids in every copy —
    exercises point indices up to 2^30 and the 32-bit tile arithmetic."""
    import torch
    bundle = _bundle(2)
    s = bundle.session()
    reps = 10
    n = N_FULL * reps
    pts = synth.points_for(2, N_FULL, None)
    d_one = torch.from_numpy(pts).cuda()
    d_pts = d_one.repeat(reps, 1).contiguous()
    assert d_pts.shape == (n, 2)
    d_counts = torch.zeros(len(bundle.ids), dtype=torch.int64, device="cuda")
    d_first = torch.empty(n, dtype=torch.int32, device="cuda")
    d_counts1 = torch.zeros_like(d_counts)
    d_first1 = torch.empty(N_FULL, dtype=torch.int32, device="cuda")
    torch.cuda.synchronize()  # the session has its own stream: torch's fills and copies must have landed
    s.join_count_device(d_pts.data_ptr(), n, d_counts.data_ptr(), capi.GJ_MODE_APPROX,
                        d_first_id_ptr=d_first.data_ptr(), sync=True)
    s.join_count_device(d_one.data_ptr(), N_FULL, d_counts1.data_ptr(), capi.GJ_MODE_APPROX,
                        d_first_id_ptr=d_first1.data_ptr(), sync=True)
    assert torch.equal(d_counts, d_counts1 * reps)
    assert bool((d_first.view(reps, N_FULL) == d_first1.unsqueeze(0)).all())
    # a ragged total (not a multiple of the tile) ending inside the last copy
    m = n - 12_345
    d_counts.zero_()
    torch.cuda.synchronize()
    s.join_count_device(d_pts.data_ptr(), m, d_counts.data_ptr(), capi.GJ_MODE_APPROX, sync=True)
    tail, _, _ = s.join_count(pts[N_FULL - 12_345:], capi.GJ_MODE_APPROX)
    assert np.array_equal(d_counts.cpu().numpy().astype(np.uint64),
                          d_counts1.cpu().numpy().astype(np.uint64) * reps - tail)


def _scaled_bundle(config, scale):
    name = build_bundles.workload_name(config, scale)
    if not build_bundles.have_bundle(name):
        pytest.skip(f"no cached index {name} (tools/build_bundles.py needs the reference)")
    return build_bundles.bundle_file(name)


@pytest.mark.parametrize("config,scale,n,mode,opts", [
    (4, 0.04, 50_000_000, capi.GJ_MODE_APPROX, {}),
    # the full-size box's regime: shared-memory tier capped at its level (dead there), 16-bit flushed histogram ->
    # K1 picks its direct form and the sparse refinement by itself, as it does on the 37 GB index
    (4, 0.04, 50_000_000, capi.GJ_MODE_APPROX, {"dir16_level_max": 17, "hist16": 1}),
    (5, 0.03, 10_000_000, capi.GJ_MODE_EXACT, {})])
def test_density_matched_configs_4_and_5(config, scale, n, mode, opts):
    """The regimes of BASELINE configs[3] and configs[4] (run at full size by
    tools/fullsize.py: profiles/fullsize_r01_cfg*.json) on their density-matched
    stand-ins: 1 600 polygons at 1 m with k_max 56 (an id table beyond the
    shared-memory histogram when the tier is capped like the full-size box's, first ids
    written late), and 300 overlapping stars (every probe a lookup-table record, exact).
    Conservation, JoinStats identities, device-resident == host-buffer results, and
    — when the compiled reference travelled with the repo — counts and ordered pairs
    against the reference's own CPU join on a prefix."""
    import torch
    path = _scaled_bundle(config, scale)
    bundle = join.IndexBundle.load(path, device=0, options=capi.Options(**opts) if opts else None)
    if opts:
        assert bundle.info.k1_direct == 1 and bundle.info.link_records > 0
    s = bundle.session()
    polys = None
    pts = synth.points_for(config, n, polys, scale=scale)
    st = join.JoinStats()
    counts, first, (ovf_pt, ovf_id) = s.join_count(pts, mode, stats=st, want_ids=True)
    probes, pip_tests, false_hits, solely_true, refined, cand_refs = st.as_tuple()
    assert probes == n and false_hits + solely_true + refined == n
    if mode == capi.GJ_MODE_APPROX:
        assert pip_tests == 0
        assert np.array_equal(counts, _hist(bundle, first, ovf_id))
    else:
        assert pip_tests == cand_refs
    # device-resident call, in pieces that are not multiples of anything
    d_pts = torch.from_numpy(pts).cuda()
    d_counts = torch.zeros(len(bundle.ids), dtype=torch.int64, device="cuda")
    d_stats = torch.zeros(6, dtype=torch.int64, device="cuda")
    d_first = torch.empty(n, dtype=torch.int32, device="cuda")
    torch.cuda.synchronize()
    flat = d_pts.view(-1)
    piece = 7_654_321
    for a in range(0, n, piece):
        s.join_count_device(flat[2 * a:].data_ptr(), min(piece, n - a), d_counts.data_ptr(), mode,
                            d_stats_ptr=d_stats.data_ptr(), d_first_id_ptr=d_first[a:].data_ptr())
    s.sync()
    assert np.array_equal(d_counts.cpu().numpy().astype(np.uint64), counts)
    assert tuple(int(v) for v in d_stats.cpu().numpy()) == st.as_tuple()
    if mode == capi.GJ_MODE_APPROX:
        assert np.array_equal(d_first.cpu().numpy().view(np.uint32), first)
    # the reference itself on a prefix
    from oracle import ref
    if ref.available():
        rb = ref.RefBundle.load(path)
        m = 10_000_000 if opts else 1_000_000
        got, _, _ = s.join_count(pts[:m], mode)
        got_map = {int(bundle.ids[k]): int(got[k]) for k in np.nonzero(got)[0]}
        want = rb.join_exact_count_threads(pts[:m], 8) if mode == capi.GJ_MODE_EXACT else rb.join_count(pts[:m], 8)
        assert got_map == want
        mp = 100_000
        row_ptr, ids = s.join_pairs(pts[:mp], mode)
        pi, pid, rst = rb.join_pairs(pts[:mp], mode == capi.GJ_MODE_EXACT)
        gpi = np.repeat(np.arange(mp, dtype=np.uint64), np.diff(row_ptr.astype(np.int64)))
        assert np.array_equal(gpi, pi) and np.array_equal(ids, pid)
    bundle.close()
