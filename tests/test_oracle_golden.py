"""CPU tests: the plain-C oracle (oracle/geojoin_oracle.c) is PINNED against the
reference — its own known-answer vectors (re-expressed literally) and the
committed fixtures that the compiled reference produced (tests/golden/).  These
tests are what entitles the GPU parity tests to use the oracle as a checker."""
import ctypes as C

import numpy as np
import pytest

from oracle import oracle
from tests import golden_util

JOIN_FIXTURES = [
    "join_small_exact", "acceptance_exact20", "cfg1_tess5_approx60m", "cfg2_tess16_approx4m",
    "cfg3_tess16_exact_trained", "cfg4_tess36_approx1m_k56", "cfg5_stars_scaled", "kmax60_sparse_ids",
    "world_stars", "empty_index", "kmax60_tiny_a", "kmax60_tiny_b",
]


# ---- cellgrid -------------------------------------------------------------------------
def test_cell_kats():
    """test_cellgrid.cpp:25-33 and the survey's verified value."""
    root = 1 << 60
    assert int(oracle.cell_from_point([[12.3, 45.6]], 0)[0]) == root
    assert int(oracle.cell_from_point([[-90.0, -180.0]], 0)[0]) == root
    assert int(oracle.cell_from_point([[0.0, 0.0]], 1)[0]) == (0b11 << 59) | (1 << 58)
    assert int(oracle.cell_from_point([[40.7, -74.0]], 24)[0]) == 0x1358F7810DB39000


def test_cells_match_reference_fixture():
    """test_cellgrid.cpp:35-48 (seed 0x5eed0001), clamps and grid-line points."""
    fx = golden_util.load("cells")
    L = oracle.lib()
    raw = C.c_uint64(0)
    got = np.empty(len(fx["points"]), np.uint64)
    for k, ((lat, lng), level) in enumerate(zip(fx["points"], fx["levels"])):
        assert L.gjo_cell_from_point(float(lat), float(lng), int(level), C.byref(raw)) == oracle.OK
        got[k] = raw.value
    assert np.array_equal(got, fx["raw"])
    assert np.array_equal(oracle.cell_from_point(fx["points"], 24), fx["raw_l24"])
    assert np.array_equal(oracle.cell_from_point(fx["points"], 30), fx["raw_l30"])


def test_cells_vs_bitwise_encoder():
    """An independent bit-by-bit encoder (the idea of oracles.hpp:54-72): grid
    discretisation then one quadrant pair at a time, MSB first."""
    rng = np.random.default_rng(5)
    pts = np.stack([rng.uniform(-90, 90, 3000), rng.uniform(-180, 180, 3000)], axis=1)
    for level in (0, 1, 7, 24, 30):
        got = oracle.cell_from_point(pts, level)
        for (lat, lng), g in zip(pts[:300], got[:300]):
            ys = min(int(max((lat + 90.0) / 180.0 * 1073741824.0, 0.0)), 0x3FFFFFFF)
            xs = min(int(max((lng + 180.0) / 360.0 * 1073741824.0, 0.0)), 0x3FFFFFFF)
            raw = 0
            for b in range(level):
                bit = 29 - b
                raw = (raw << 2) | (((ys >> bit) & 1) << 1) | ((xs >> bit) & 1)
            raw = ((raw << 1) | 1) << (60 - 2 * level)
            assert int(g) == raw


def test_invalid_points_and_levels():
    """test_cellgrid.cpp:50-61."""
    L = oracle.lib()
    raw = C.c_uint64(0)
    for lat, lng in ((91.0, 0.0), (0.0, 181.0), (float("nan"), 0.0), (0.0, float("inf"))):
        assert L.gjo_cell_from_point(lat, lng, 5, C.byref(raw)) == oracle.INVALID_POINT
    assert L.gjo_cell_from_point(0.0, 0.0, 31, C.byref(raw)) == oracle.INVALID_LEVEL
    assert L.gjo_cell_from_point(0.0, 0.0, -1, C.byref(raw)) == oracle.INVALID_LEVEL
    with pytest.raises(oracle.OracleError) as e:
        oracle.cell_from_point([[1.0, 1.0], [2.0, 2.0], [95.0, 0.0]], 10)
    assert e.value.status == oracle.INVALID_POINT and e.value.bad_index == 2


# ---- PIP --------------------------------------------------------------------------------
def test_pip_unit_square_kats():
    """test_geometry.cpp:69-78: edges and vertices count as inside (ST_Covers)."""
    fx = golden_util.load("pip")
    got = oracle.pip_test(fx["square"], fx["square_points"])
    assert got.tolist() == [True, True, True, True, False, False, False]
    assert np.array_equal(got, fx["square_inside"].astype(bool))


def test_pip_matches_reference_fixture():
    """test_geometry.cpp:80-102 shapes (seed 0x6eed0002) + on-edge / on-vertex probes."""
    fx = golden_util.load("pip")
    want = np.unpackbits(fx["inside"])[: len(fx["points"])].astype(bool)
    ro, po = fx["ring_off"].astype(np.int64), fx["point_off"].astype(np.int64)
    got = np.concatenate([oracle.pip_test(fx["ring_latlng"][ro[r]:ro[r + 1]], fx["points"][po[r]:po[r + 1]])
                          for r in range(len(ro) - 1)])
    assert np.array_equal(got, want)
    assert want.any() and not want.all()


# ---- tagged entries ---------------------------------------------------------------------
def test_tag_decode_forms():
    """test_act.cpp:80-107,245-284: payload forms and the lookup-table record
    [1, 5, 2, 1, 3] = one true hit (5) then candidates (1, 3)."""
    lut = np.array([1, 5, 2, 1, 3], np.uint32)
    ix = oracle.OracleIndex(np.zeros(0, np.uint64), lut, np.zeros(8), np.zeros(8), np.zeros(8), 48,
                            np.zeros(0, np.uint32), np.zeros(1, np.uint64), np.zeros((0, 2)))
    one = ((5 << 1 | 1) << 2) | 1
    assert ix.decode(one) == [(5, True)]
    two = ((8 << 1 | 1) << 33) | ((2 << 1) << 2) | 2
    assert ix.decode(two) == [(8, True), (2, False)]
    assert ix.decode(0) == []
    assert ix.decode((0 << 2) | 3) == [(5, True), (1, False), (3, False)]
    with pytest.raises(oracle.OracleError) as e:
        ix.decode((100 << 2) | 3)  # offset past the table end
    assert e.value.status == oracle.CORRUPT_INDEX
    big = ((((1 << 30) - 1) << 1) << 2) | 1  # kMaxPolygonId candidate
    assert ix.decode(big) == [((1 << 30) - 1, False)]


# ---- probe + join vs the compiled reference's outputs -----------------------------------
@pytest.mark.parametrize("name", JOIN_FIXTURES)
def test_probe_entries_match_reference(name):
    fx = golden_util.load(name)
    ox = golden_util.oracle_index(fx)
    assert np.array_equal(ox.probe_points(fx["points"]), fx["entries"])


@pytest.mark.parametrize("name", ["join_small_exact", "cfg2_tess16_approx4m", "world_stars", "empty_index"])
def test_batch_equals_scalar_and_node_bound(name):
    """test_act.cpp:311-343 (lockstep kernel == scalar walk) and :226-243
    (at most 1 + k_max/8 node accesses)."""
    fx = golden_util.load(name)
    ox = golden_util.oracle_index(fx)
    k_max = int(fx["k_max"][0])
    rng = np.random.default_rng(11)
    pts = fx["points"][:4000].copy()
    far = rng.random(len(pts)) < 0.2  # mix in global points: prefix mismatches and misses
    pts[far] = np.stack([rng.uniform(-90, 90, far.sum()), rng.uniform(-180, 180, far.sum())], axis=1)
    raw = oracle.cell_from_point(pts, k_max // 2)
    scalar, acc = ox.probe_raw(raw, count_accesses=True)
    assert np.array_equal(ox.probe_batch8(raw), scalar)
    assert acc.max() <= 1 + (k_max + 7) // 8


@pytest.mark.parametrize("name", JOIN_FIXTURES)
@pytest.mark.parametrize("kind", ["exact", "approx"])
def test_join_matches_reference(name, kind):
    fx = golden_util.load(name)
    ox = golden_util.oracle_index(fx)
    pi, pid, stats, counts = ox.join(fx["points"], approx=(kind == "approx"))
    epi, epid = golden_util.pairs_of(fx, kind)
    assert np.array_equal(pi, epi) and np.array_equal(pid, epid)
    assert tuple(int(v) for v in stats) == tuple(int(v) for v in fx[f"{kind}_stats"])
    assert int(counts.sum()) == len(epid)


@pytest.mark.parametrize("name", JOIN_FIXTURES)
def test_count_matches_reference_for_any_thread_count(name):
    """test_join.cpp:200-214: streaming counts are independent of the worker count."""
    fx = golden_util.load(name)
    ox = golden_util.oracle_index(fx)
    want = {int(k): int(v) for k, v in zip(fx["count_ids"], fx["count_values"])}
    approx = bool(fx["bundle_approx"][0])
    for threads in (1, 2, 3, 7):
        got, total = ox.join_count(fx["points"], approx, threads)
        assert got == want and total == sum(want.values())


def test_join_stops_at_invalid_point():
    fx = golden_util.load("join_small_exact")
    ox = golden_util.oracle_index(fx)
    pts = fx["points"][:100].copy()
    pts[37, 0] = np.nan
    with pytest.raises(oracle.OracleError) as e:
        ox.join(pts, approx=False)
    assert e.value.status == oracle.INVALID_POINT and e.value.bad_index == 37


def test_oracle_against_live_reference(ref_available):
    """Where the compiled reference is present, random fresh inputs as well."""
    if not ref_available:
        pytest.skip("oracle/_ref not built")
    from oracle import ref
    from tests.refrng import Rng, random_points_in, random_star_polygon
    rng = Rng(0xBEEF)
    rings = [random_star_polygon(rng, rng.uniform(10, 12), rng.uniform(20, 22), rng.uniform(0.2, 0.8),
                                 rng.uniform_int(5, 30)) for _ in range(7)]
    polys = ref.Polygons.from_rings(rings, ids=[3, 5, 8, 13, 21, 34, 55])
    pts = random_points_in(rng, 9.0, 13.0, 19.0, 23.0, 20000)
    for cfg in (ref.default_config(mode_approx=0), ref.default_config(mode_approx=1, precision_m=200.0)):
        b = ref.RefBundle.build(polys, cfg)
        ox = oracle.OracleIndex.from_ref_bundle(b)
        assert np.array_equal(ox.probe_points(pts), b.probe_points(pts))
        for exact in (True, False):
            pi, pid, st = b.join_pairs(pts, exact)
            opi, opid, ost, _ = ox.join(pts, approx=not exact)
            assert np.array_equal(pi, opi) and np.array_equal(pid, opid) and np.array_equal(st, ost)
        assert ox.join_count(pts, b.approx, 4)[0] == b.join_count(pts, 4)


# ---- training pre-pass (act.cpp:414-440) ---------------------------------------------
@pytest.mark.parametrize("name", JOIN_FIXTURES)
def test_training_candidates_match_reference_fixture(name):
    """The oracle's restatement of Act::train's any_candidate test against the
    indices the compiled reference produced (tests/golden/make_training_golden.py),
    and against JoinStats::refinement_entered of the same reference run."""
    fx = golden_util.load(name)
    want = golden_util.load("training_candidates")[name].astype(np.uint64)
    got = golden_util.oracle_index(fx).training_candidates(fx["points"])
    assert np.array_equal(got, want)
    assert len(got) == int(fx["probe_stats"][4])


def test_training_candidates_match_live_reference():
    from oracle import ref
    if not ref.available():
        pytest.skip("oracle/_ref not built")
    fx = golden_util.load("cfg3_tess16_exact_trained")
    b = ref.RefBundle.load(golden_util.bundle_file("cfg3_tess16_exact_trained"))
    rng = np.random.default_rng(0x7A11)
    lat = fx["points"][:, 0]
    lng = fx["points"][:, 1]
    pts = np.stack([rng.uniform(lat.min(), lat.max(), 50_000), rng.uniform(lng.min(), lng.max(), 50_000)], axis=1)
    assert np.array_equal(golden_util.oracle_index(fx).training_candidates(pts), b.training_candidates(pts))
