"""GPU parity tests proper: the CUDA path, called through the C ABI, against
(a) the committed golden outputs of the compiled reference and (b) the C
oracle run live on the same inputs.  Bit-exact: entries, pairs (order
included), per-polygon counts and the six JoinStats counters."""
import numpy as np
import pytest

from paper_1802_09488_b200 import capi, join
from tests import golden_util

pytestmark = pytest.mark.gpu

JOIN_FIXTURES = [
    "join_small_exact", "join_small_approx", "acceptance_exact20", "cfg1_tess5_approx60m",
    "cfg2_tess16_approx4m", "cfg3_tess16_exact_trained", "cfg4_tess36_approx1m_k56",
    "cfg5_stars_scaled", "kmax60_sparse_ids", "world_stars", "empty_index",
    "kmax60_tiny_a", "kmax60_tiny_b",  # k_max 60 under a 48-bit prefix: the last node step ends below the leaf level
]

_cache = {}


def setup(name):
    if name not in _cache:
        fx = golden_util.load(name)
        bundle = join.IndexBundle.load(golden_util.bundle_file(name), device=0)
        _cache.clear()  # one resident index at a time
        _cache[name] = (fx, bundle)
    return _cache[name]


def pairs_from_csr(row_ptr, ids):
    n = len(row_ptr) - 1
    return np.repeat(np.arange(n, dtype=np.uint64), np.diff(row_ptr.astype(np.int64))), ids


@pytest.mark.parametrize("name", JOIN_FIXTURES)
def test_entries_match_reference(name):
    fx, bundle = setup(name)
    got = bundle.session().probe_points(fx["points"])
    assert np.array_equal(got, fx["entries"])  # bitwise Act::probe(cell_from_point(p))


@pytest.mark.parametrize("name", JOIN_FIXTURES)
def test_cell_probe_matches_point_probe_and_oracle(name):
    """The directory-free raw-id kernel (ProbeBatchFn contract) agrees with
    the directory path and the oracle's scalar walk."""
    from oracle import oracle
    fx, bundle = setup(name)
    k_max = int(fx["k_max"][0])
    raw = oracle.cell_from_point(fx["points"], k_max // 2)
    got = bundle.session().probe_cells(raw)
    assert np.array_equal(got, fx["entries"])
    ox = golden_util.oracle_index(fx)
    assert np.array_equal(got[:2000], ox.probe_raw(raw[:2000]))


@pytest.mark.parametrize("name", JOIN_FIXTURES)
@pytest.mark.parametrize("kind", ["exact", "approx"])
def test_pairs_match_reference(name, kind):
    fx, bundle = setup(name)
    mode = capi.GJ_MODE_EXACT if kind == "exact" else capi.GJ_MODE_APPROX
    st = join.JoinStats()
    pi, pid = pairs_from_csr(*bundle.session().join_pairs(fx["points"], mode, st))
    epi, epid = golden_util.pairs_of(fx, kind)
    assert np.array_equal(pi, epi)
    assert np.array_equal(pid, epid)  # order included
    assert st.as_tuple() == tuple(int(v) for v in fx[f"{kind}_stats"])


@pytest.mark.parametrize("name", JOIN_FIXTURES)
def test_counts_match_reference(name):
    """join_count_per_polygon: mode from the bundle, zero counts dropped."""
    fx, bundle = setup(name)
    got = join.join_count_per_polygon(bundle, fx["points"])
    want = {int(k): int(v) for k, v in zip(fx["count_ids"], fx["count_values"])}
    assert got == want
    assert bundle.approx == bool(fx["bundle_approx"][0])


@pytest.mark.parametrize("name", JOIN_FIXTURES)
def test_probe_stats_match_reference(name):
    fx, bundle = setup(name)
    st = join.JoinStats()
    join.accumulate_probe_stats(bundle, fx["points"], st)
    assert st.as_tuple() == tuple(int(v) for v in fx["probe_stats"])
    assert st.false_hits + st.solely_true_hits + st.refinement_entered == st.probes


@pytest.mark.parametrize("name", ["join_small_exact", "cfg3_tess16_exact_trained", "cfg5_stars_scaled"])
@pytest.mark.parametrize("kind", ["exact", "approx"])
def test_first_id_and_overflow(name, kind):
    fx, bundle = setup(name)
    mode = capi.GJ_MODE_EXACT if kind == "exact" else capi.GJ_MODE_APPROX
    counts, first, (opt, oid) = bundle.session().join_count(fx["points"], mode, want_ids=True)
    epi, epid = golden_util.pairs_of(fx, kind)
    n = len(fx["points"])
    inline = (first != capi.GJ_NO_MATCH) & (first != capi.GJ_DEFERRED)
    # rebuild the pair list: inline first ids + overflow records (already sorted)
    pts = np.concatenate([np.nonzero(inline)[0].astype(np.uint64), opt])
    ids = np.concatenate([first[inline] & ~np.uint32(capi.GJ_MORE_FLAG), oid])
    seq = np.concatenate([np.zeros(int(inline.sum()), np.int64), 1 + np.arange(len(opt), dtype=np.int64)])
    order = np.lexsort((seq, pts))
    assert np.array_equal(pts[order], epi)
    assert np.array_equal(ids[order], epid)
    want = np.bincount(np.searchsorted(bundle.ids, epid), minlength=len(bundle.ids))
    assert np.array_equal(counts, want.astype(np.uint64))
    more = (first & capi.GJ_MORE_FLAG) != 0
    per_point = np.bincount(epi.astype(np.int64), minlength=n)
    assert np.array_equal(more & inline, (per_point > 1) & inline)


@pytest.mark.parametrize("name", ["join_small_exact", "cfg2_tess16_approx4m", "cfg3_tess16_exact_trained",
                                  "cfg4_tess36_approx1m_k56", "cfg5_stars_scaled", "world_stars", "empty_index"])
@pytest.mark.parametrize("tier_sub", [0, 2])
def test_late_first_ids_equal_early_first_ids(name, tier_sub):
    """join_kernel's kLate variant (first-id words written where a point is settled
    instead of pre-written for every point; chosen by itself when the 16-bit tier
    resolves few cells) must produce the same first ids, overflow records, counts and
    stats as the default variant — host-buffer and device-resident calls, both modes,
    ragged sizes, with and without a refined tier."""
    import torch
    fx = golden_util.load(name)
    pts = np.ascontiguousarray(fx["points"])
    results = {}
    for late in ("0", "1"):
        b = join.IndexBundle.load(golden_util.bundle_file(name), device=0,
                                  options=capi.Options(ids_late=int(late), tier_sub=tier_sub))
        s = b.session()
        out = []
        for mode in (capi.GJ_MODE_EXACT, capi.GJ_MODE_APPROX):
            for n in (len(pts), min(len(pts), 4097), min(len(pts), 31)):
                st = join.JoinStats()
                counts, first, (opt, oid) = s.join_count(pts[:n], mode, stats=st, want_ids=True)
                out += [counts, first, opt, oid, np.array(st.as_tuple())]
                if n:
                    d_pts = torch.from_numpy(pts[:n]).cuda()
                    d_counts = torch.zeros(max(1, len(b.ids)), dtype=torch.int64, device="cuda")
                    d_first = torch.full((n,), 0x55555555, dtype=torch.int32, device="cuda")
                    torch.cuda.synchronize()
                    s.join_count_device(d_pts.data_ptr(), n, d_counts.data_ptr(), mode,
                                        d_first_id_ptr=d_first.data_ptr(), sync=True)
                    out += [d_counts.cpu().numpy(), d_first.cpu().numpy()]
        results[late] = out
        b.close()
    assert len(results["0"]) == len(results["1"])
    for a, c in zip(results["0"], results["1"]):
        assert np.array_equal(a, c)


def test_invalid_point_reports_first_index():
    fx, bundle = setup("join_small_exact")
    pts = fx["points"].copy()
    pts[777, 0] = 91.0
    pts[4242, 1] = np.nan
    with pytest.raises(join.InvalidArgument) as e:
        bundle.session().probe_points(pts)
    assert e.value.index == 777
    with pytest.raises(join.InvalidArgument) as e:
        join.join_count_per_polygon(bundle, pts)
    assert e.value.index == 777
    pts = fx["points"].copy()
    pts[5, 1] = np.inf
    with pytest.raises(join.InvalidArgument):
        join.join_exact(bundle, pts)


def test_edge_sizes():
    fx, bundle = setup("join_small_exact")
    s = bundle.session()
    assert len(s.probe_points(np.zeros((0, 2)))) == 0
    assert join.join_count_per_polygon(bundle, np.zeros((0, 2))) == {}
    for n in (1, 7, 8, 9, 1023, 4097):  # ragged tails around batch / tile sizes
        pi, pid = join.join_exact(bundle, fx["points"][:n])
        epi, epid = golden_util.pairs_of(fx, "exact")
        keep = epi < n
        assert np.array_equal(pi, epi[keep]) and np.array_equal(pid, epid[keep])


def test_from_arrays_equals_load_file():
    fx, bundle = setup("cfg2_tess16_approx4m")
    g = golden_util.parse_gjx(golden_util.gjx_bytes(fx))
    b2 = join.IndexBundle.from_arrays(g["arena"], g["lut"], g["roots"], g["prefixes"], g["prefix_bits"],
                                      g["k_max"], g["approx"], g["polygon_ids"], g["vtx_off"],
                                      g["vtx_latlng"], device=0)
    assert np.array_equal(b2.session().probe_points(fx["points"]), fx["entries"])
    assert b2.info.node_count == bundle.info.node_count and b2.info.dir_level == bundle.info.dir_level
    b2.close()


def test_cell_ids_match_reference_fixture():
    """cell_from_point: KATs, seed 0x5eed0001 cases, clamps and grid-line points."""
    fx = golden_util.load("cells")
    _, bundle = setup("join_small_exact")
    s = bundle.session()
    assert np.array_equal(s.cells_from_points(fx["points"], 24), fx["raw_l24"])
    assert np.array_equal(s.cells_from_points(fx["points"], 30), fx["raw_l30"])
    for level in (0, 1, 5, 12, 22, 30):
        sel = fx["levels"] == level
        if sel.any():
            assert np.array_equal(s.cells_from_points(fx["points"][sel], level), fx["raw"][sel])
    # literal KATs (test_cellgrid.cpp:25-33)
    assert int(s.cells_from_points([[0.0, 0.0]], 1)[0]) == (0b11 << 59) | (1 << 58)
    assert int(s.cells_from_points([[12.3, 45.6]], 0)[0]) == 1 << 60
    assert int(s.cells_from_points([[40.7, -74.0]], 24)[0]) == 0x1358F7810DB39000
    with pytest.raises(ValueError):
        s.cells_from_points([[0.0, 0.0]], 31)
    with pytest.raises(join.InvalidArgument):
        s.cells_from_points([[0.0, 181.0]], 5)


def test_cell_ids_adversarial_grid_lines_vs_oracle():
    """The division-free fast path must fall back exactly where truncation
    could differ: points on grid lines of every level and a few ulps around
    them, plus dense random points, bit-exact against the C oracle."""
    from oracle import oracle
    _, bundle = setup("join_small_exact")
    s = bundle.session()
    rng = np.random.default_rng(0xC311)
    pts = []
    for level in (30, 29, 24, 20, 16, 8):
        k = rng.integers(0, (1 << level) + 1, 40000)
        lat = k / float(1 << level) * 180.0 - 90.0
        lng = k[::-1] / float(1 << level) * 360.0 - 180.0
        for ulps in (0, 1, 2, 3, 4, 7, -1, -2, -3, -4, -7):
            a, o = lat.copy(), lng.copy()
            for _ in range(abs(ulps)):
                a = np.nextafter(a, np.inf if ulps > 0 else -np.inf)
                o = np.nextafter(o, np.inf if ulps > 0 else -np.inf)
            pts.append(np.stack([np.clip(a, -90.0, 90.0), np.clip(o, -180.0, 180.0)], axis=1))
    edge_lat = np.array([90.0, -90.0, 0.0, -0.0, 5e-324, -5e-324, 1e-300, np.nextafter(90.0, 0.0),
                         np.nextafter(-90.0, 0.0), 89.99999999999999, 45.0, 1e-17])
    edge_lng = np.array([180.0, -180.0, -0.0, 0.0, -5e-324, 5e-324, -1e-300, np.nextafter(180.0, 0.0),
                         np.nextafter(-180.0, 0.0), 179.99999999999997, -135.0, -1e-17])
    pts.append(np.stack([np.repeat(edge_lat, len(edge_lng)), np.tile(edge_lng, len(edge_lat))], axis=1))
    pts.append(np.stack([rng.uniform(-1e-7, 1e-7, 200_000), rng.uniform(-1e-7, 1e-7, 200_000)], axis=1))
    pts.append(np.stack([rng.uniform(-90, 90, 2_000_000), rng.uniform(-180, 180, 2_000_000)], axis=1))
    pts.append(np.stack([rng.uniform(40.5, 40.95, 2_000_000), rng.uniform(-74.25, -73.70, 2_000_000)], axis=1))
    pts = np.concatenate(pts)
    assert np.array_equal(s.cells_from_points(pts, 30), oracle.cell_from_point(pts, 30))


def test_multi_chunk_inputs_match_oracle():
    """Inputs larger than the internal chunk sizes (4 M points for pairs, 3 M
    for counts): chunk seams must not show in pairs, row offsets or counts."""
    fx, bundle = setup("join_small_exact")
    ox = golden_util.oracle_index(fx)
    rng = np.random.default_rng(0xC4A2)
    n = 9_000_000
    pts = np.stack([rng.uniform(-11.5, -4.5, n), rng.uniform(48.5, 55.5, n)], axis=1)
    s = bundle.session()
    want, total = ox.join_count(pts, approx=False, threads=16)
    assert join.join_count_per_polygon(bundle, pts) == want
    m = 4_500_000  # two pairs chunks
    st = join.JoinStats()
    row_ptr, ids = s.join_pairs(pts[:m], capi.GJ_MODE_EXACT, st)
    pi, pid, ost, _ = ox.join(pts[:m], approx=False)
    assert np.array_equal(np.repeat(np.arange(m, dtype=np.uint64), np.diff(row_ptr.astype(np.int64))), pi)
    assert np.array_equal(ids, pid)
    assert st.as_tuple() == tuple(int(v) for v in ost)
    assert int(row_ptr[-1]) == len(pid) and int(row_ptr[0]) == 0


@pytest.mark.parametrize("name", JOIN_FIXTURES)
def test_training_candidates_match_reference(name):
    """The training pre-pass (the probe half of Act::train, act.cpp:414-440):
    ordered indices equal to the compiled reference's fixture; the count equals
    JoinStats::refinement_entered of the reference's probe pass."""
    fx, bundle = setup(name)
    want = golden_util.load("training_candidates")[name].astype(np.uint64)
    s = bundle.session()
    got = s.training_candidates(fx["points"])
    assert np.array_equal(got, want)
    assert len(got) == int(fx["probe_stats"][4])
    n = len(fx["points"])
    assert join.expensive_fraction(bundle, fx["points"]) == (len(want) / n if n else 0.0)
    # a base index shifts the output; an empty input gives an empty list
    assert np.array_equal(s.training_candidates(fx["points"][:777], base_index=1 << 33),
                          want[want < 777] + np.uint64(1 << 33))
    assert len(s.training_candidates(np.zeros((0, 2)))) == 0


def test_training_candidates_multi_chunk_and_errors():
    fx, bundle = setup("cfg3_tess16_exact_trained")
    ox = golden_util.oracle_index(fx)
    rng = np.random.default_rng(0x7A12)
    lat, lng = fx["points"][:, 0], fx["points"][:, 1]
    n = 4_300_000  # more than one 4 M-point chunk
    pts = np.stack([rng.uniform(lat.min(), lat.max(), n), rng.uniform(lng.min(), lng.max(), n)], axis=1)
    s = bundle.session()
    assert np.array_equal(s.training_candidates(pts), ox.training_candidates(pts))
    pts[4_200_123, 0] = np.nan
    with pytest.raises(join.InvalidArgument) as e:
        s.training_candidates(pts)
    assert e.value.index == 4_200_123


def _write(tmp_path, name, data: bytes):
    p = tmp_path / name
    p.write_bytes(data)
    return p


def test_corrupt_index_files_are_rejected(tmp_path):
    """test_act.cpp:609-624 / test_join.cpp:317-318: empty, bad magic,
    truncated and garbage snapshots raise CorruptionError, never crash."""
    good = golden_util.gjx_bytes(golden_util.load("cfg2_tess16_approx4m"))
    for name, data in [("empty.gjx", b""), ("magic.gjx", b"XXXXYYYYZZZZ"), ("garbage.gjx", b"not an index"),
                       ("half.gjx", good[: len(good) // 2]), ("short.gjx", good[:100]),
                       ("almost.gjx", good[:-9])]:
        with pytest.raises(join.CorruptionError):
            join.IndexBundle.load(_write(tmp_path, name, data), device=0)
    with pytest.raises(OSError):
        join.IndexBundle.load(tmp_path / "missing.gjx", device=0)
    # the untouched bytes still load
    join.IndexBundle.load(_write(tmp_path, "good.gjx", good), device=0).close()


def test_structurally_corrupt_indexes_are_rejected():
    """What the reference would only hit lazily while probing (act.cpp:141-153,
    269, 667-669; join.cpp:111-114) is rejected when the index is created."""
    fx = golden_util.load("cfg5_stars_scaled")  # has lookup-table records
    g = golden_util.parse_gjx(golden_util.gjx_bytes(fx))

    def make(**over):
        a = dict(g)
        a.update(over)
        return join.IndexBundle.from_arrays(a["arena"], a["lut"], a["roots"], a["prefixes"], a["prefix_bits"],
                                            a["k_max"], a["approx"], a["polygon_ids"], a["vtx_off"],
                                            a["vtx_latlng"], device=0)

    make().close()  # the unmodified arrays are fine
    arena = g["arena"]
    n_nodes = len(arena) // 256
    links = np.flatnonzero(((arena & 3) == 0) & (arena != 0))
    offsets = np.flatnonzero((arena & 3) == 3)
    assert len(links) and len(offsets)

    bad = arena.copy()
    bad[links[0]] = np.uint64((n_nodes + 5) << 2)  # link past the arena
    with pytest.raises(join.CorruptionError):
        make(arena=bad)
    bad = arena.copy()
    bad[links[-1]] = np.uint64(1 << 2)  # link back to the root: not a forest
    with pytest.raises(join.CorruptionError):
        make(arena=bad)
    bad = arena.copy()
    bad[offsets[0]] = np.uint64(((len(g["lut"]) + 7) << 2) | 3)  # lookup-table offset out of range
    with pytest.raises(join.CorruptionError):
        make(arena=bad)
    lut = g["lut"].copy()
    off = int(arena[offsets[0]] >> np.uint64(2)) & 0x7FFFFFFF
    lut[off] = np.uint32(len(lut))  # record longer than the table
    with pytest.raises(join.CorruptionError):
        make(lut=lut)
    with pytest.raises(join.CorruptionError):
        make(k_max=50)  # validate_act_config, act.cpp:38-42
    roots = g["roots"].copy()
    roots[0] = n_nodes + 1
    with pytest.raises(join.CorruptionError):
        make(roots=roots)


def test_large_id_table_counts_through_private_copies():
    """Id tables too large for the shared-memory histograms (K1: forced here
    with the tuning knob; K2: more than 8192 ids) count into per-CTA copies in
    global memory that are folded afterwards: same counts, pairs and stats."""
    fx = golden_util.load("join_small_exact")
    g = golden_util.parse_gjx(golden_util.gjx_bytes(fx))
    extra = 9000  # far-away dummy triangles with sparse ids: referenced by no cell
    ids = np.concatenate([g["polygon_ids"], 100_000 + 7 * np.arange(extra, dtype=np.uint32)])
    tri = np.array([[-80.0, 10.0], [-80.0, 10.001], [-79.999, 10.0]])
    vtx = np.concatenate([g["vtx_latlng"].reshape(-1, 2), np.tile(tri, (extra, 1))])
    off = np.concatenate([g["vtx_off"], g["vtx_off"][-1] + 3 * np.arange(1, extra + 1, dtype=np.uint64)])
    b = join.IndexBundle.from_arrays(g["arena"], g["lut"], g["roots"], g["prefixes"], g["prefix_bits"], g["k_max"],
                                     g["approx"], ids, off, vtx, device=0,
                                     options=capi.Options(hist_rep_cap=0, hist16=0))
    assert len(b.ids) > 8192
    want = dict(zip(fx["count_ids"].tolist(), fx["count_values"].tolist()))
    for _ in range(2):  # the copies are left zero for the next launch
        assert join.join_count_per_polygon(b, fx["points"]) == want
    for kind, mode in (("exact", capi.GJ_MODE_EXACT), ("approx", capi.GJ_MODE_APPROX)):
        st = join.JoinStats()
        counts, first, (ovf_pt, ovf_id) = b.session().join_count(fx["points"], mode, stats=st, want_ids=True)
        epi, epid = golden_util.pairs_of(fx, kind)
        assert np.array_equal(counts, np.bincount(np.searchsorted(b.ids, epid), minlength=len(b.ids)).astype(np.uint64))
        assert st.as_tuple() == tuple(int(v) for v in fx[f"{kind}_stats"])
    b.close()


@pytest.mark.parametrize("name", ["cfg2_tess16_approx4m", "cfg3_tess16_exact_trained", "cfg4_tess36_approx1m_k56",
                                  "cfg5_stars_scaled", "kmax60_sparse_ids"])
def test_unpacked_queue_coding_matches_reference(name):
    """The fallback queue coding (window too wide for 32 bits, arenas of 2^24+
    nodes): the queue word is the tier index and population 3 re-reads the
    point.  Forced with the test hook; results must not change."""
    fx = golden_util.load(name)
    b = join.IndexBundle.load(golden_util.bundle_file(name), device=0, options=capi.Options(queue_unpacked=1))
    want = dict(zip(fx["count_ids"].tolist(), fx["count_values"].tolist()))
    assert join.join_count_per_polygon(b, fx["points"]) == want
    for kind, mode in (("exact", capi.GJ_MODE_EXACT), ("approx", capi.GJ_MODE_APPROX)):
        st = join.JoinStats()
        counts, first, _ = b.session().join_count(fx["points"], mode, stats=st, want_ids=True)
        epi, epid = golden_util.pairs_of(fx, kind)
        assert np.array_equal(counts, np.bincount(np.searchsorted(b.ids, epid), minlength=len(b.ids)).astype(np.uint64))
        assert st.as_tuple() == tuple(int(v) for v in fx[f"{kind}_stats"])
    b.close()


def _check_join_against_fixture(b, fx):
    want = dict(zip(fx["count_ids"].tolist(), fx["count_values"].tolist()))
    assert join.join_count_per_polygon(b, fx["points"]) == want
    for kind, mode in (("exact", capi.GJ_MODE_EXACT), ("approx", capi.GJ_MODE_APPROX)):
        st = join.JoinStats()
        counts, first, _ = b.session().join_count(fx["points"], mode, stats=st, want_ids=True)
        epi, epid = golden_util.pairs_of(fx, kind)
        assert np.array_equal(counts, np.bincount(np.searchsorted(b.ids, epid), minlength=len(b.ids)).astype(np.uint64))
        assert st.as_tuple() == tuple(int(v) for v in fx[f"{kind}_stats"])


@pytest.mark.parametrize("hi_bits", [1, 2])
@pytest.mark.parametrize("name", ["cfg2_tess16_approx4m", "cfg3_tess16_exact_trained", "cfg4_tess36_approx1m_k56",
                                  "cfg5_stars_scaled"])
def test_wide_arena_queue_coding_matches_reference(name, hi_bits):
    """Arenas of 2^24 / 2^25 nodes and more keep the packed queue coding by carrying
    1 / 2 high bits of the arena slot next to the point index (DevQueueCoding::index_bits).
    Forced on a small index with the test hook; results must not change."""
    fx = golden_util.load(name)
    b = join.IndexBundle.load(golden_util.bundle_file(name), device=0,
                              options=capi.Options(queue_slot_hi_bits=hi_bits))
    _check_join_against_fixture(b, fx)
    b.close()


@pytest.mark.parametrize("sub", [1, 2, 3])
@pytest.mark.parametrize("name", ["cfg2_tess16_approx4m", "cfg3_tess16_exact_trained", "cfg4_tess36_approx1m_k56",
                                  "cfg5_stars_scaled", "kmax60_sparse_ids", "world_stars", "join_small_exact"])
def test_refined_tier_matches_reference(name, sub):
    """K1's refined 32-bit tier (DevIndex::dirk): the deepest tier again, 1-3 grid
    levels finer, cells resolved from uniform slot runs of the linked nodes.  Built
    by itself only for indexes whose deepest tier is mostly links; forced here on
    every fixture shape, packed and unpacked queue coding.  Results must not change."""
    fx = golden_util.load(name)
    for unpacked in (False, True):
        b = join.IndexBundle.load(golden_util.bundle_file(name), device=0,
                                  options=capi.Options(tier_sub=sub, queue_unpacked=int(unpacked)))
        _check_join_against_fixture(b, fx)
        b.close()


def _everything(b, pts):
    """Every result form of the join, both modes, host-buffer and device-resident calls, ragged sizes."""
    import torch
    s = b.session()
    out = []
    for mode in (capi.GJ_MODE_EXACT, capi.GJ_MODE_APPROX):
        for n in (len(pts), min(len(pts), 4097), min(len(pts), 31)):
            st = join.JoinStats()
            counts, first, (opt, oid) = s.join_count(pts[:n], mode, stats=st, want_ids=True)
            out += [counts, first, opt, oid, np.array(st.as_tuple())]
            counts2, _, _ = s.join_count(pts[:n], mode)
            out += [counts2]
            if n:
                d_pts = torch.from_numpy(pts[:n]).cuda()
                d_counts = torch.zeros(max(1, len(b.ids)), dtype=torch.int64, device="cuda")
                d_first = torch.full((n,), 0x55555555, dtype=torch.int32, device="cuda")
                torch.cuda.synchronize()
                s.join_count_device(d_pts.data_ptr(), n, d_counts.data_ptr(), mode, d_first_id_ptr=d_first.data_ptr(), sync=True)
                out += [d_counts.cpu().numpy(), d_first.cpu().numpy()]
        row_ptr, ids = s.join_pairs(pts, mode)
        out += [row_ptr, ids]
    return out


@pytest.mark.parametrize("name", ["cfg1_tess5_approx60m", "cfg2_tess16_approx4m", "cfg3_tess16_exact_trained",
                                  "cfg4_tess36_approx1m_k56", "cfg5_stars_scaled", "kmax60_sparse_ids", "world_stars",
                                  "join_small_exact", "join_small_approx", "kmax60_tiny_a", "kmax60_tiny_b", "empty_index"])
def test_direct_form_matches_reference(name):
    """join_kernel's direct form (kDirect): every point gathers its own code of the 32-bit
    tier as an asynchronous copy into shared memory and is settled one tile later; chosen
    by itself when the shared-memory tier resolves nothing (BASELINE config 4).  Forced here
    on every fixture shape — the replicated histogram, general counting (hist_rep_cap=0 takes
    the histogram away), the 16-bit flushed histogram, packed / wide / unpacked queue codings,
    with the sparse refinement behind it — against the queued form.  Results must not change."""
    fx = golden_util.load(name)
    pts = np.ascontiguousarray(fx["points"])
    base = dict(tier_sub=0)
    plain = join.IndexBundle.load(golden_util.bundle_file(name), device=0, options=capi.Options(direct=0, link_sub=0, **base))
    want = _everything(plain, pts)
    plain.close()
    for extra in ({}, {"hist_rep_cap": 0}, {"hist16": 1}, {"link_sub": 1}, {"link_sub": 1, "hist16": 1, "queue_slot_hi_bits": 2},
                  {"queue_unpacked": 1, "hist_rep_cap": 0}):
        b = join.IndexBundle.load(golden_util.bundle_file(name), device=0, options=capi.Options(direct=1, **{**base, **extra}))
        _check_join_against_fixture(b, fx)
        got = _everything(b, pts)
        assert len(got) == len(want)
        for k, (a, c) in enumerate(zip(want, got)):
            assert np.array_equal(a, c), (extra, k)
        b.close()


@pytest.mark.parametrize("name", ["cfg2_tess16_approx4m", "cfg3_tess16_exact_trained", "cfg4_tess36_approx1m_k56",
                                  "cfg5_stars_scaled", "kmax60_sparse_ids", "world_stars", "join_small_exact",
                                  "kmax60_tiny_a", "kmax60_tiny_b"])
def test_sparse_refinement_matches_reference(name):
    """K1's sparse refinement (DevIndex::link_sub): one 64-byte record per LINK cell of
    the deepest tier, a code per 16-slot run of the linked node.  Built by itself only for
    trees too large for palette nodes (BASELINE config 4 at full size); forced here on
    every fixture shape, with and without palette nodes behind it, with the wide-arena
    queue coding, and with the unpacked coding (where it must be dropped).  Results must
    not change."""
    fx = golden_util.load(name)
    pts = np.ascontiguousarray(fx["points"])
    everything = lambda b: _everything(b, pts)
    plain = join.IndexBundle.load(golden_util.bundle_file(name), device=0, options=capi.Options(link_sub=0, tier_sub=0))
    assert plain.info.link_records == 0
    want = everything(plain)
    plain.close()
    built = 0
    for extra in ({}, {"node_pal_max_mb": 0}, {"queue_slot_hi_bits": 2}, {"queue_unpacked": 1}, {"ids_late": 1}):
        b = join.IndexBundle.load(golden_util.bundle_file(name), device=0, options=capi.Options(link_sub=1, tier_sub=0, **extra))
        if extra.get("queue_unpacked"):
            assert b.info.link_records == 0
        built += b.info.link_records
        _check_join_against_fixture(b, fx)
        got = everything(b)
        assert len(got) == len(want)
        for a, c in zip(want, got):
            assert np.array_equal(a, c)
        b.close()
    if name.startswith("cfg"):
        assert built > 0  # the fixture does exercise the records


def test_arena_beyond_2_24_nodes_matches_reference():
    """A REAL arena of more than 2^24 nodes (34 GB): the nodes of a fixture index
    renumbered to sit above 2^24 empty, unreachable nodes, so every arena slot the
    join touches needs more than 32 bits.  Entries, counts and stats must equal the
    fixture's.  (BASELINE config 4 at full size has 18.3 M nodes.)"""
    import torch
    shift = 1 << 24
    free_dev, _ = torch.cuda.mem_get_info()
    try:
        avail_host = int([l for l in open("/proc/meminfo") if l.startswith("MemAvailable")][0].split()[1]) * 1024
    except Exception:
        avail_host = 0
    if free_dev < 60 << 30 or avail_host < 60 << 30:
        pytest.skip("needs 60 GB of free device and host memory")
    _cache.clear()
    fx = golden_util.load("cfg4_tess36_approx1m_k56")
    g = golden_util.parse_gjx(golden_util.gjx_bytes(fx))
    small = np.asarray(g["arena"], np.uint64)
    k = len(small) // 256
    arena = np.zeros((shift + k) * 256, np.uint64)  # untouched pages are not backed by memory
    link = ((small & np.uint64(3)) == 0) & (small != 0)
    moved = small.copy()
    moved[link] += np.uint64(shift << 2)  # a link is node id << 2 (act.hpp:55-60)
    arena[shift * 256:] = moved
    roots = np.asarray(g["roots"], np.uint64).copy()
    roots[roots != 0] += np.uint64(shift)
    b = join.IndexBundle.from_arrays(arena, g["lut"], roots, g["prefixes"], g["prefix_bits"], g["k_max"], g["approx"],
                                     g["polygon_ids"], g["vtx_off"], g["vtx_latlng"], device=0)
    del arena
    assert b.info.node_count == shift + k
    assert np.array_equal(b.session().probe_points(fx["points"]), fx["entries"])
    _check_join_against_fixture(b, fx)
    b.close()


def test_device_resident_call_is_split_into_launches():
    """A device-resident call longer than one launch may be (the cap depends on the
    arena size) runs as several launches: same counts, first ids and stats, and the
    smallest offending index of the whole call survives the later pieces."""
    import torch
    fx = golden_util.load("cfg3_tess16_exact_trained")
    b = join.IndexBundle.load(golden_util.bundle_file("cfg3_tess16_exact_trained"), device=0)
    pts = np.ascontiguousarray(fx["points"])
    n = len(pts)
    # the same index again (a device-to-device replica would inherit the knob), capped at a seventh of the call per launch
    b_split = join.IndexBundle.load(golden_util.bundle_file("cfg3_tess16_exact_trained"), device=0,
                                    options=capi.Options(max_launch_points=n // 7 + 1))
    d_pts = torch.from_numpy(pts).cuda()

    def run(mode, s):
        d_counts = torch.zeros(len(b.ids), dtype=torch.int64, device="cuda")
        d_stats = torch.zeros(6, dtype=torch.int64, device="cuda")
        d_first = torch.empty(n, dtype=torch.int32, device="cuda")
        torch.cuda.synchronize()
        s.join_count_device(d_pts.data_ptr(), n, d_counts.data_ptr(), mode, d_stats_ptr=d_stats.data_ptr(),
                            d_first_id_ptr=d_first.data_ptr(), sync=True)
        return d_counts.cpu().numpy(), d_stats.cpu().numpy(), d_first.cpu().numpy()

    for mode in (capi.GJ_MODE_EXACT, capi.GJ_MODE_APPROX):
        s = b.session()
        l0 = s.launches
        one = run(mode, s)
        per_call = s.launches - l0
        s = b_split.session()
        l0 = s.launches
        many = run(mode, s)
        assert s.launches - l0 == 7 * per_call
        for a, c in zip(one, many):
            assert np.array_equal(a, c)
    bad = pts.copy()
    bad[n // 7 - 3, 0] = 95.0   # in the first piece
    bad[n - 5, 1] = np.nan      # in the last piece
    d_bad = torch.from_numpy(bad).cuda()
    d_counts = torch.zeros(len(b.ids), dtype=torch.int64, device="cuda")
    torch.cuda.synchronize()
    with pytest.raises(join.InvalidArgument) as e:
        s.join_count_device(d_bad.data_ptr(), n, d_counts.data_ptr(), capi.GJ_MODE_APPROX)
        s.sync()
    assert e.value.index == n // 7 - 3
    b.close()
    b_split.close()


def test_index_and_session_lifecycle_releases_device_memory():
    """Create / use / destroy indexes and sessions repeatedly: HBM comes back."""
    import torch
    fx = golden_util.load("cfg2_tess16_approx4m")
    path = golden_util.bundle_file("cfg2_tess16_approx4m")
    _cache.clear()
    torch.cuda.synchronize()

    def cycle():
        b = join.IndexBundle.load(path, device=0)
        s = b.session()
        s.join_count(fx["points"], capi.GJ_MODE_EXACT, want_ids=True)
        s.join_pairs(fx["points"][:5000], capi.GJ_MODE_APPROX)
        s.training_candidates(fx["points"][:5000])
        s.points_from_csv(b"lat,lng\n1,2\n")
        s.close()
        b.close()

    cycle()  # first use may create the context's own pools
    free0, _ = torch.cuda.mem_get_info()
    for _ in range(20):
        cycle()
    free1, _ = torch.cuda.mem_get_info()
    assert free0 - free1 < (8 << 20), (free0, free1)


def test_concurrent_sessions_on_one_index_and_on_two_indexes():
    """An index is immutable and shared; sessions are per thread.
    Threads joining at the same time — on one index and on indexes with
    different shared-memory plans — get the serial results."""
    import threading
    from paper_1802_09488_b200.join import Session
    fxa, fxb = golden_util.load("cfg2_tess16_approx4m"), golden_util.load("cfg5_stars_scaled")
    ba = join.IndexBundle.load(golden_util.bundle_file("cfg2_tess16_approx4m"), device=0)
    bb = join.IndexBundle.load(golden_util.bundle_file("cfg5_stars_scaled"), device=0)
    want = {}
    for key, (b, fx) in {"a": (ba, fxa), "b": (bb, fxb)}.items():
        c, f, (op, oi) = b.session().join_count(fx["points"], capi.GJ_MODE_EXACT, want_ids=True)
        want[key] = (c.copy(), f.copy(), op.copy(), oi.copy())
    errors = []

    def worker(key, b, fx):
        try:
            s = Session(b)
            for _ in range(25):
                c, f, (op, oi) = s.join_count(fx["points"], capi.GJ_MODE_EXACT, want_ids=True)
                w = want[key]
                if not (np.array_equal(c, w[0]) and np.array_equal(f, w[1]) and np.array_equal(op, w[2])
                        and np.array_equal(oi, w[3])):
                    errors.append(key)
            s.close()
        except Exception as exc:  # noqa: BLE001
            errors.append(repr(exc))

    threads = [threading.Thread(target=worker, args=(k, b, fx))
               for k, b, fx in [("a", ba, fxa), ("b", bb, fxb), ("a", ba, fxa), ("b", bb, fxb)]]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert errors == []
    ba.close()
    bb.close()


def _fleet_devices():
    """Every GPU of the box, topped up to three replicas with device 0 (replicas
    on one device share nothing, and their kernels do not wait on one another)."""
    devices = list(range(capi.lib().gj_device_count()))
    while len(devices) < 3:
        devices.append(0)
    return devices


@pytest.mark.parametrize("name", ["join_small_exact", "cfg2_tess16_approx4m", "cfg3_tess16_exact_trained",
                                  "cfg5_stars_scaled", "kmax60_sparse_ids", "empty_index"])
def test_index_group_equals_single_device(name):
    """The all-GPUs-for-one-input call (gj_group_*: the reference's worker fan-out,
    join.cpp:255-285, with index replicas as the workers): counts, stats, first ids,
    overflow records and ordered pairs equal the one-device results and the reference
    fixture for every worker count — tests/test_join.cpp:200-214 (threads in {1,2,3,7})."""
    fx = golden_util.load(name)
    pts = np.ascontiguousarray(fx["points"])
    one = join.IndexBundle.load(golden_util.bundle_file(name), device=0)
    fleet = join.IndexGroup.load(golden_util.bundle_file(name), _fleet_devices())
    assert len(fleet) == len(_fleet_devices()) and np.array_equal(fleet.ids, one.ids)
    want = {int(k): int(v) for k, v in zip(fx["count_ids"], fx["count_values"])}
    for threads in (1, 2, 3, 7):
        assert join.join_count_per_polygon(fleet, pts, threads) == want
    for kind, mode in (("exact", capi.GJ_MODE_EXACT), ("approx", capi.GJ_MODE_APPROX)):
        s1, sg = join.JoinStats(), join.JoinStats()
        c1, f1, (p1, i1) = one.session().join_count(pts, mode, stats=s1, want_ids=True, base_index=1000)
        for workers in (0, 2):
            sg = join.JoinStats()
            cg, fg, (pg, ig) = fleet.session(workers).join_count(pts, mode, stats=sg, want_ids=True, base_index=1000)
            assert np.array_equal(c1, cg) and np.array_equal(f1, fg)
            assert np.array_equal(p1, pg) and np.array_equal(i1, ig)
            assert s1.as_tuple() == sg.as_tuple() == tuple(int(v) for v in fx[f"{kind}_stats"])
        st = join.JoinStats()
        pi, pid = (join.join_exact if kind == "exact" else join.join_approx)(fleet, pts, st)
        epi, epid = golden_util.pairs_of(fx, kind)
        assert np.array_equal(pi, epi) and np.array_equal(pid, epid)
        assert st.as_tuple() == tuple(int(v) for v in fx[f"{kind}_stats"])
    if len(pts) > 10:  # the smallest offending index wins, wherever its range runs
        bad = pts.copy()
        bad[len(pts) - 2, 1] = 200.0
        with pytest.raises(join.InvalidArgument) as e:
            fleet.session().join_count(bad, capi.GJ_MODE_APPROX)
        assert e.value.index == len(pts) - 2
        bad[3, 0] = np.inf
        with pytest.raises(join.InvalidArgument) as e:
            fleet.session().join_count(bad, capi.GJ_MODE_EXACT, want_ids=True)
        assert e.value.index == 3
        with pytest.raises(join.InvalidArgument) as e:
            join.join_exact(fleet, bad)
        assert e.value.index == 3
    fleet.close()
    one.close()


def test_replica_is_independent_of_its_source():
    """gj_index_replicate: a device-to-device copy keeps working after the index it was
    copied from is destroyed, and gives the same entries and join results."""
    fx = golden_util.load("cfg3_tess16_exact_trained")
    src = join.IndexBundle.load(golden_util.bundle_file("cfg3_tess16_exact_trained"), device=0,
                                options=capi.Options(tier_sub=1))
    n_dev = capi.lib().gj_device_count()
    rep = src.replicate(n_dev - 1)
    assert rep.info.device == n_dev - 1 and rep.info.node_count == src.info.node_count
    src.close()
    filler = join.IndexBundle.load(golden_util.bundle_file("cfg5_stars_scaled"), device=0)  # reuse the freed HBM
    assert np.array_equal(rep.session().probe_points(fx["points"]), fx["entries"])
    _check_join_against_fixture(rep, fx)
    filler.close()
    rep.close()


@pytest.mark.parametrize("name", ["join_small_exact", "cfg4_tess36_approx1m_k56", "cfg5_stars_scaled", "kmax60_sparse_ids"])
def test_flushed_16bit_histogram_matches_reference(name):
    """Id tables beyond the 32-bit shared-memory histogram count in a 16-bit one that the CTA flushes every
    kHist16FlushTiles tiles (forced here on small tables): the fixture's results, then launches long enough for
    many flushes per CTA — random points, and the worst case of every point in ONE polygon (a counter that would
    wrap 30 times without the flushes) — against the default counting path."""
    import torch
    fx = golden_util.load(name)
    b16 = join.IndexBundle.load(golden_util.bundle_file(name), device=0, options=capi.Options(hist16=1))
    b32 = join.IndexBundle.load(golden_util.bundle_file(name), device=0)
    _check_join_against_fixture(b16, fx)
    rng = np.random.default_rng(0x16B1)
    pts = np.ascontiguousarray(fx["points"])
    n = 20_000_000
    big = pts[rng.integers(0, len(pts), n)]
    hit = pts[np.flatnonzero(b32.session().join_count(pts, capi.GJ_MODE_APPROX, want_ids=True)[1] < capi.GJ_DEFERRED)[0]]
    same = np.tile(hit, (n, 1))
    for arr in (big, same):
        d_pts = torch.from_numpy(arr).cuda()
        for mode in (capi.GJ_MODE_APPROX, capi.GJ_MODE_EXACT):
            if mode == capi.GJ_MODE_EXACT and name == "cfg5_stars_scaled":
                continue  # 2^32 candidate tasks in one launch: the call is refused, see test_device_resident_call_is_split_into_launches
            res = []
            for b in (b16, b32):
                d_counts = torch.zeros(len(b.ids), dtype=torch.int64, device="cuda")
                d_first = torch.empty(n, dtype=torch.int32, device="cuda")
                torch.cuda.synchronize()
                b.session().join_count_device(d_pts.data_ptr(), n, d_counts.data_ptr(), mode,
                                              d_first_id_ptr=d_first.data_ptr(), sync=True)
                res.append((d_counts.cpu().numpy(), d_first.cpu().numpy()))
            assert np.array_equal(res[0][0], res[1][0]) and np.array_equal(res[0][1], res[1][1])
            assert int(res[0][0].sum()) >= (n if arr is same else 1)
    b16.close()
    b32.close()


@pytest.mark.parametrize("name", ["join_small_exact", "cfg3_tess16_exact_trained", "cfg5_stars_scaled", "empty_index"])
@pytest.mark.parametrize("chunk", [0, 4096])
def test_csr_into_caller_arrays_host_and_device(name, chunk):
    """join_exact / join_approx -> CSR in ONE call: gj_join_pairs_host_into (caller's host arrays, pageable and
    pinned, streamed chunk by chunk) and gj_join_pairs_device (points, row offsets and ids all in HBM) give the
    fixture's ordered pairs and stats, with many small chunks as well; an id array that is too small returns the
    size needed and complete row offsets."""
    import torch
    fx = golden_util.load(name)
    pts = np.ascontiguousarray(fx["points"])
    n = len(pts)
    b = join.IndexBundle.load(golden_util.bundle_file(name), device=0,
                              options=capi.Options(chunk_points=chunk) if chunk else None)
    s = b.session()
    for kind, mode in (("exact", capi.GJ_MODE_EXACT), ("approx", capi.GJ_MODE_APPROX)):
        epi, epid = golden_util.pairs_of(fx, kind)
        want_rows = np.concatenate([[0], np.cumsum(np.bincount(epi.astype(np.int64), minlength=n))]).astype(np.uint64)
        want_stats = tuple(int(v) for v in fx[f"{kind}_stats"])
        for pinned in (False, True):
            row_ptr = join.pinned_array(n + 1, np.uint64) if pinned else np.empty(n + 1, np.uint64)
            ids = join.pinned_array(len(epid) + 5, np.uint32) if pinned else np.empty(len(epid) + 5, np.uint32)
            st = join.JoinStats()
            total = s.join_pairs_into(pts, mode, row_ptr, ids, st)
            assert total == len(epid) and np.array_equal(row_ptr, want_rows) and np.array_equal(ids[:total], epid)
            assert st.as_tuple() == want_stats
        if len(epid) > 3:  # too small: the size comes back, and the rows
            row_ptr = np.zeros(n + 1, np.uint64)
            with pytest.raises(join.CapacityError) as e:
                s.join_pairs_into(pts, mode, row_ptr, np.empty(len(epid) // 2, np.uint32))
            assert e.value.needed == len(epid) and np.array_equal(row_ptr, want_rows)
        # everything in HBM
        d_pts = torch.from_numpy(pts).cuda() if n else torch.zeros((1, 2), dtype=torch.float64, device="cuda")
        d_rows = torch.full((n + 1,), -1, dtype=torch.int64, device="cuda")
        d_ids = torch.full((len(epid) + 7,), -1, dtype=torch.int32, device="cuda")
        torch.cuda.synchronize()
        st = join.JoinStats()
        total = s.join_pairs_device(d_pts.data_ptr(), n, mode, d_rows.data_ptr(), d_ids.data_ptr(), len(d_ids), st)
        assert total == len(epid) and st.as_tuple() == want_stats
        assert np.array_equal(d_rows.cpu().numpy().view(np.uint64), want_rows)
        got = d_ids.cpu().numpy().view(np.uint32)
        assert np.array_equal(got[:total], epid) and np.all(got[total:] == 0xFFFFFFFF)  # nothing written past the end
        if len(epid) > 3:
            with pytest.raises(join.CapacityError) as e:
                s.join_pairs_device(d_pts.data_ptr(), n, mode, d_rows.data_ptr(), d_ids.data_ptr(), len(epid) - 1)
            assert e.value.needed == len(epid)
            with pytest.raises(join.CapacityError) as e:  # sizing call
                s.join_pairs_device(d_pts.data_ptr(), n, mode, d_rows.data_ptr(), 0, 0)
            assert e.value.needed == len(epid)
            assert np.array_equal(d_rows.cpu().numpy().view(np.uint64), want_rows)
    if n > 10:
        bad = pts.copy()
        bad[n // 2, 0] = -90.5
        with pytest.raises(join.InvalidArgument) as e:
            s.join_pairs_into(bad, capi.GJ_MODE_EXACT, np.empty(n + 1, np.uint64), np.empty(16, np.uint32))
        assert e.value.index == n // 2
    b.close()


@pytest.mark.parametrize("name", ["cfg5_stars_scaled", "join_small_exact", "cfg3_tess16_exact_trained", "world_stars",
                                  "kmax60_sparse_ids"])
def test_staged_lookup_table_records_match_reference(name):
    """Lookup-table-heavy indexes stage the records of a population-3 batch in shared memory (stage_records: a
    warp-cooperative, coalesced copy in 16-byte chunks) instead of walking them word by word per lane.  Forced on
    here; counts, stats, first ids and overflow records must equal the fixture's and the unstaged path's, with
    batches that fit the staging buffer and — small chunk budget — batches that do not."""
    import torch
    fx = golden_util.load(name)
    pts = np.ascontiguousarray(fx["points"])
    plain = join.IndexBundle.load(golden_util.bundle_file(name), device=0, options=capi.Options(stage_lut=0))
    for extra in ({}, {"smem_pad": 60000}):  # the padding leaves the staging buffer only its minimum size
        b = join.IndexBundle.load(golden_util.bundle_file(name), device=0, options=capi.Options(stage_lut=1, **extra))
        _check_join_against_fixture(b, fx)
        for mode in (capi.GJ_MODE_EXACT, capi.GJ_MODE_APPROX):
            sa, sb = join.JoinStats(), join.JoinStats()
            ca, fa, (pa, ia) = plain.session().join_count(pts, mode, stats=sa, want_ids=True)
            cb, fb, (pb, ib) = b.session().join_count(pts, mode, stats=sb, want_ids=True)
            assert np.array_equal(ca, cb) and np.array_equal(fa, fb) and np.array_equal(pa, pb) and np.array_equal(ia, ib)
            assert sa.as_tuple() == sb.as_tuple()
            n = len(pts)
            d_pts = torch.from_numpy(pts).cuda()
            d_counts = torch.zeros(max(1, len(b.ids)), dtype=torch.int64, device="cuda")
            torch.cuda.synchronize()
            b.session().join_count_device(d_pts.data_ptr(), n, d_counts.data_ptr(), mode, sync=True)
            assert np.array_equal(d_counts.cpu().numpy()[:len(ca)].astype(np.uint64), ca)
        b.close()
    plain.close()


@pytest.mark.parametrize("name", ["join_small_exact", "acceptance_exact20", "cfg3_tess16_exact_trained", "cfg5_stars_scaled",
                                  "kmax60_sparse_ids", "world_stars", "kmax60_tiny_a"])
def test_indexed_strip_lists_match_reference(name):
    """Large polygon sets give the refine kernel strip lists of vertex indices instead of 32-byte edge records
    (gj_options.strip_index; automatic beyond ~32 MB of records).  Forced here: exact pairs, counts and stats must
    equal the fixture's."""
    fx = golden_util.load(name)
    b = join.IndexBundle.load(golden_util.bundle_file(name), device=0, options=capi.Options(strip_index=1))
    _check_join_against_fixture(b, fx)
    st = join.JoinStats()
    pi, pid = pairs_from_csr(*b.session().join_pairs(fx["points"], capi.GJ_MODE_EXACT, st))
    epi, epid = golden_util.pairs_of(fx, "exact")
    assert np.array_equal(pi, epi) and np.array_equal(pid, epid)
    assert st.as_tuple() == tuple(int(v) for v in fx["exact_stats"])
    b.close()
