"""Generates tests/golden/*.npz by running the UNMODIFIED reference (compiled
by oracle/build.py into oracle/_ref) on seeded inputs.  Run in the build
container only (needs /root/reference):

    python tests/golden/make_golden.py

Scenarios re-express the reference's own test cases (same RNG recipe, seeds
and shapes; tests/oracles.hpp, tests/test_cellgrid.cpp:35-48,
tests/test_geometry.cpp:69-102, tests/test_act.cpp:245-284,311-343,
tests/test_join.cpp:115-134,160-214, tests/acceptance.cpp:156-174) plus
scaled-down versions of the five BASELINE.json configs.  Every expected
value in the fixtures is an output of the reference itself.
"""
from __future__ import annotations

import sys
import tempfile
import zlib
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle import ref  # noqa: E402
from paper_1802_09488_b200 import synth  # noqa: E402
from tests.refrng import Rng, random_points_in, random_star_polygon  # noqa: E402

OUT = Path(__file__).resolve().parent


def save(name: str, **arrays):
    path = OUT / f"{name}.npz"
    np.savez_compressed(path, **arrays)
    print(f"{name}: {path.stat().st_size / 1024:.0f} KB")


def bundle_bytes(b: ref.RefBundle) -> np.ndarray:
    with tempfile.NamedTemporaryFile(suffix=".gjx") as f:
        b.save(f.name)
        raw = Path(f.name).read_bytes()
    return np.frombuffer(zlib.compress(raw, 9), dtype=np.uint8)


def join_fixture(name: str, polys: ref.Polygons, cfg, points: np.ndarray, training=None, extra=None):
    b = ref.RefBundle.build(polys, cfg, training)
    i = b.info
    print(f"  [{name}] mode={'approx' if i.mode_approx else 'exact'} nodes={i.node_count} lut={i.lut_len} "
          f"bound={i.achieved_precision_m:.3f} trained_splits={i.train_cells_split}")
    points = np.ascontiguousarray(points, np.float64)
    entries = b.probe_points(points)
    epi, epid, est = b.join_pairs(points, exact=True)
    api, apid, ast = b.join_pairs(points, exact=False)
    counts = b.join_count(points, threads=3)
    pst = b.accumulate_probe_stats(points)
    out = dict(
        gjx_z=bundle_bytes(b), points=points, entries=entries,
        exact_pi=epi.astype(np.uint32), exact_pid=epid, exact_stats=est,
        approx_pi=api.astype(np.uint32), approx_pid=apid, approx_stats=ast,
        count_ids=np.array(sorted(counts), np.uint32),
        count_values=np.array([counts[k] for k in sorted(counts)], np.uint64),
        probe_stats=pst, bundle_approx=np.array([i.mode_approx], np.int32),
        k_max=np.array([i.k_max], np.int32))
    if extra:
        out.update(extra)
    save(name, **out)
    return b


def star_set(rng: Rng, n, lat_rng, lng_rng, rad_rng, vtx_rng, ids=None):
    rings = []
    for _ in range(n):
        clat = rng.uniform(*lat_rng)
        clng = rng.uniform(*lng_rng)
        rad = rng.uniform(*rad_rng)
        nv = rng.uniform_int(*vtx_rng)
        rings.append(random_star_polygon(rng, clat, clng, rad, nv))
    for r in rings:
        ref.validate_polygon(r)
    return ref.Polygons.from_rings(rings, ids)


def main():
    # ---- cellgrid: test_cellgrid.cpp:35-48 (seed 0x5eed0001) + clamps + grid-line points
    rng = Rng(0x5EED0001)
    pts, levels = [], []
    for _ in range(20000):
        pts.append((rng.uniform(-90.0, 90.0), rng.uniform(-180.0, 180.0)))
        levels.append(rng.uniform_int(0, 30))
    pts += [(90.0, 180.0), (90.0, 180.0), (-90.0, -180.0), (0.0, 0.0), (12.3, 45.6), (40.7, -74.0)]
    levels += [30, 5, 30, 1, 0, 24]
    # points exactly on and one ulp around level-30 grid lines (truncation edge)
    g = np.random.default_rng(7)
    k = g.integers(1, 1 << 30, 2000)
    lat_line = k / float(1 << 30) * 180.0 - 90.0
    lng_line = k / float(1 << 30) * 360.0 - 180.0
    for arr_lat, arr_lng in ((lat_line, lng_line), (np.nextafter(lat_line, 100), np.nextafter(lng_line, 200)),
                             (np.nextafter(lat_line, -100), np.nextafter(lng_line, -200))):
        for a, o in zip(arr_lat, arr_lng):
            pts.append((float(a), float(o)))
            levels.append(30)
    pts = np.array(pts)
    levels = np.array(levels, np.int32)
    save("cells", points=pts, levels=levels, raw=ref.cell_from_point_levels(pts, levels),
         raw_l24=ref.cell_from_point(pts, 24), raw_l30=ref.cell_from_point(pts, 30))

    # ---- pip: test_geometry.cpp:69-102 (unit square KATs + seed 0x6eed0002)
    square = np.array([[0, 0], [0, 1], [1, 1], [1, 0]], float)
    sq_pts = np.array([[0.5, 0.5], [0.0, 0.5], [0.5, 0.0], [1.0, 1.0], [1.5, 0.5], [-0.1, 0.5], [0.5, 1.0000001]])
    rng = Rng(0x6EED0002)
    rings = [random_star_polygon(rng, 10.0, 20.0, 1.0, 12)]
    points = [random_points_in(rng, 8.0, 12.0, 18.0, 22.0, 1000)]
    for _ in range(100):
        clat, clng = rng.uniform(-70, 70), rng.uniform(-150, 150)
        rad = rng.uniform(0.05, 3.0)
        nv = rng.uniform_int(3, 40)
        ring = random_star_polygon(rng, clat, clng, rad, nv)
        rings.append(ring)
        lo, hi = ring.min(0), ring.max(0)
        points.append(random_points_in(rng, lo[0] - 1, hi[0] + 1, lo[1] - 1, hi[1] + 1, 1000))
    # boundary probes: vertices verbatim and points on edges
    for r in range(len(rings)):
        ring = rings[r]
        t = np.linspace(0.0, 1.0, 7)[None, :, None]
        a = ring[:, None, :]
        b = np.roll(ring, -1, axis=0)[:, None, :]
        on_edge = (a + t * (b - a)).reshape(-1, 2)[:200]
        points[r] = np.concatenate([points[r], on_edge])
    polys = ref.Polygons.from_rings(rings)
    expected = np.concatenate([ref.pip_test(rings[r], points[r]) for r in range(len(rings))])
    save("pip", ring_off=polys.vtx_off, ring_latlng=polys.latlng,
         point_off=np.cumsum([0] + [len(p) for p in points]).astype(np.uint64),
         points=np.concatenate(points), inside=np.packbits(expected),
         square=square, square_points=sq_pts, square_inside=ref.pip_test(square, sq_pts))

    # ---- join_small_exact: test_join.cpp:115-134 (seed 0x10e0002), exact default config
    rng = Rng(0x10E0002)
    polys = star_set(rng, 8, (-10.0, -6.0), (50.0, 54.0), (0.2, 1.2), (8, 24))
    pts = random_points_in(rng, -11.5, -4.5, 48.5, 55.5, 10000)
    # a few on-boundary points as well
    ring = polys.ring(3)
    pts[:16] = ring[:16] if len(ring) >= 16 else pts[:16]
    pts[16:24] = (ring[:8] + np.roll(ring, -1, axis=0)[:8]) * 0.5
    join_fixture("join_small_exact", polys, ref.default_config(mode_approx=0), pts)

    # ---- join_small_approx: test_join.cpp:160-189 (seed 0x10e0003), approx 25 m
    rng = Rng(0x10E0003)
    polys = star_set(rng, 6, (-10.0, -6.0), (50.0, 54.0), (0.2, 1.2), (8, 24))
    pts = random_points_in(rng, -11.5, -4.5, 48.5, 55.5, 10000)
    join_fixture("join_small_approx", polys, ref.default_config(mode_approx=1, precision_m=25.0,
                                                                memory_budget_bytes=4 << 30), pts)

    # ---- acceptance criterion 1 shape: acceptance.cpp:156-174 (seed 0xacce0001), 20 polygons
    rng = Rng(0xACCE0001)
    polys = star_set(rng, 20, (30.0, 36.0), (-100.0, -94.0), (0.2, 1.0), (6, 32))
    pts = random_points_in(rng, 29.0, 37.0, -101.0, -93.0, 20000)
    join_fixture("acceptance_exact20", polys, ref.default_config(mode_approx=0), pts)

    # ---- lookup-table shape: overlapping stars -> records with >= 3 refs (config 5 scaled)
    sub = (40.60, 40.66, -74.05, -73.98)
    stars = synth.star_polygons(60, synth.seed_for(5, 0), box=sub)
    pts = synth.uniform_points(20000, synth.seed_for(5, 2), box=sub)
    join_fixture("cfg5_stars_scaled", ref.Polygons(stars.ids, stars.vtx_off, stars.latlng),
                 ref.default_config(mode_approx=1, precision_m=15.0, k_max=48, memory_budget_bytes=4 << 30), pts)

    # ---- tessellations: configs 1-4 scaled
    t1 = synth.voronoi_tessellation(5, synth.seed_for(1, 0), mean_vertices=300.0)
    pts = synth.uniform_points(30000, synth.seed_for(1, 2))
    join_fixture("cfg1_tess5_approx60m", ref.Polygons(t1.ids, t1.vtx_off, t1.latlng),
                 ref.default_config(mode_approx=1, precision_m=60.0, k_max=48), pts)

    sub2 = (40.70, 40.79, -74.02, -73.91)  # straddles the level-7 latitude line 40.78125
    t2 = synth.voronoi_tessellation(16, synth.seed_for(2, 0), mean_vertices=60.0, box=sub2)
    pts = synth.uniform_points(30000, synth.seed_for(2, 2), box=(40.69, 40.80, -74.03, -73.90))
    join_fixture("cfg2_tess16_approx4m", ref.Polygons(t2.ids, t2.vtx_off, t2.latlng),
                 ref.default_config(mode_approx=1, precision_m=4.0, k_max=48, memory_budget_bytes=4 << 30), pts)

    mix = synth.gaussian_mixture(synth.seed_for(3, 1), components=8, sigma=(0.004, 0.02), box=sub2)
    train = synth.mixture_points(100000, synth.seed_for(3, 1), mix, box=sub2)
    pts = synth.mixture_points(30000, synth.seed_for(3, 2), mix, box=sub2)
    synth.plant_boundary_points(pts, t2, synth.seed_for(3, 2), 0.02)
    join_fixture("cfg3_tess16_exact_trained", ref.Polygons(t2.ids, t2.vtx_off, t2.latlng),
                 ref.default_config(mode_approx=0, k_max=48, memory_budget_bytes=256 << 20,
                                    training_point_limit=100000), pts, training=train)

    sub4 = (40.700, 40.712, -74.000, -73.985)
    t4 = synth.voronoi_tessellation(36, synth.seed_for(4, 0), mean_vertices=15.0, max_depth=3, box=sub4)
    pts = synth.uniform_points(30000, synth.seed_for(4, 2), box=(40.699, 40.713, -74.001, -73.984))
    join_fixture("cfg4_tess36_approx1m_k56", ref.Polygons(t4.ids, t4.vtx_off, t4.latlng),
                 ref.default_config(mode_approx=1, precision_m=1.0, k_max=56, memory_budget_bytes=8 << 30), pts)

    # ---- k_max = 60 (full key) and sparse polygon ids
    rng = Rng(0xAC70060)
    polys = star_set(rng, 3, (1.0, 1.002), (1.0, 1.002), (0.0004, 0.0008), (5, 9),
                     ids=[7, 1000, (1 << 30) - 1])
    pts = random_points_in(rng, 0.998, 1.004, 0.998, 1.004, 5000)
    join_fixture("kmax60_sparse_ids", polys,
                 ref.default_config(mode_approx=1, precision_m=0.5, k_max=60, memory_budget_bytes=4 << 30), pts)

    # ---- world-spanning polygons: short prefix, coarse directory
    rng = Rng(0xAC70004)
    polys = star_set(rng, 5, (-40.0, 40.0), (-120.0, 120.0), (8.0, 25.0), (6, 24))
    pts = np.concatenate([random_points_in(rng, -90.0, 90.0, -180.0, 180.0, 9990),
                          np.array([[90.0, 180.0], [-90.0, -180.0], [0.0, 0.0], [90.0, -180.0], [-90.0, 180.0],
                                    [45.0, 90.0], [-45.0, -90.0], [0.0, 180.0], [0.0, -180.0], [89.999999, 179.999999]])])
    join_fixture("world_stars", polys, ref.default_config(mode_approx=0, k_max=48), pts)

    # ---- empty index: test_act.cpp:109-123
    rng = Rng(0xAC70002)
    pts = random_points_in(rng, -90.0, 90.0, -180.0, 180.0, 1000)
    join_fixture("empty_index", ref.Polygons.from_rings([]), ref.default_config(mode_approx=0), pts)


if __name__ == "__main__":
    main()
