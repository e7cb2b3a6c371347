"""TEST INFRASTRUCTURE — adversarial inputs for the point-in-polygon refine
(pip_test, proj/src/geometry.cpp:184-204; point_segment_dist_sq :63-75; the
reference's own cases: tests/test_geometry.cpp:69-102).

The GPU refine kernel adds three exactness arguments of its own on top of the
reference's arithmetic — rejection by the edge's bounding box widened by 1e-9
degrees, "certain crossing" without the division when the point lies left of
the edge's x range, and per-polygon latitude strips — so the points here sit
exactly where those could go wrong: on and a few ulps around every vertex and
edge, on rays through vertices (point latitude == vertex latitude), at 0.5e-12 …
2e-9 degrees from edges (either side of the 1e-12 boundary tolerance and of
the 1e-9 margin), and on the seams between latitude strips."""
from __future__ import annotations

import numpy as np

ULPS = (0, 1, -1, 2, -2, 4, -4, 7, -7)


def ulp_shift(a: np.ndarray, k: int) -> np.ndarray:
    """k representable doubles further from zero (k > 0) or closer to it (k < 0)."""
    return (np.ascontiguousarray(a, np.float64).view(np.int64) + np.int64(k)).view(np.float64)


def rings_of(vtx_off, vtx_latlng):
    ll = np.asarray(vtx_latlng, np.float64).reshape(-1, 2)
    return [ll[int(vtx_off[i]):int(vtx_off[i + 1])] for i in range(len(vtx_off) - 1)]


def adversarial_points(rings, rng: np.random.Generator, per_ring_cap: int = 150_000) -> np.ndarray:
    """(lat, lng) probes around every ring (array of (lat, lng) vertices, not closed)."""
    out = []
    for ring in rings:
        v = np.asarray(ring, np.float64)
        n = len(v)
        if n < 3:
            continue
        a, b = v, np.roll(v, -1, axis=0)
        pts = []
        # 1. vertices +- ulps in each axis (a ray through a vertex, the vertex itself)
        for dk in ULPS:
            for dl in ULPS:
                pts.append(np.stack([ulp_shift(v[:, 0], dk), ulp_shift(v[:, 1], dl)], axis=1))
        # 2. points of the edges (what "a + t (b - a)" rounds to) +- ulps
        for t in (0.5, 0.25, 1.0 / 3.0, 0.999999, 1e-9):
            p = a + t * (b - a)
            for dk in (0, 1, -1, 4, -4):
                for dl in (0, 1, -1, 4, -4):
                    pts.append(np.stack([ulp_shift(p[:, 0], dk), ulp_shift(p[:, 1], dl)], axis=1))
        # 3. at a given distance from the edge, both sides: around the 1e-12 tolerance and the 1e-9 margin
        d = b - a
        length = np.hypot(d[:, 0], d[:, 1])
        ok = length > 0
        nrm = np.zeros_like(d)
        nrm[ok] = np.stack([-d[ok, 1], d[ok, 0]], axis=1) / length[ok, None]
        for dist in (0.5e-12, 0.99e-12, 1.01e-12, 1.5e-12, 2e-12, 0.5e-9, 0.99e-9, 1.01e-9, 2e-9, 1e-7):
            for side in (1.0, -1.0):
                for t in (0.5, 0.1, 0.0, 1.0):
                    pts.append(a + t * d + side * dist * nrm)
        # 4. rays through vertices: the latitude of a vertex (+- ulps), x elsewhere — left of, between and
        #    right of the polygon, and just beside the x of other vertices
        x_lo, x_hi = v[:, 1].min(), v[:, 1].max()
        span = max(x_hi - x_lo, 1e-9)
        for dk in (0, 1, -1, 2, -2):
            y = ulp_shift(v[:, 0], dk)
            for x in (np.full(n, x_lo - 0.25 * span), np.full(n, x_hi + 0.25 * span),
                      rng.uniform(x_lo, x_hi, n), rng.uniform(x_lo, x_hi, n),
                      np.roll(v[:, 1], 1) - 1e-9, np.roll(v[:, 1], -1) + 1e-9, np.roll(v[:, 1], 2),
                      np.roll(v[:, 1], n // 2), 0.5 * (v[:, 1] + np.roll(v[:, 1], n // 3))):
                pts.append(np.stack([y, x], axis=1))
        # 5. latitude-strip seams of the refine kernel (gj_index.cu: k = 2 * edges strips over the polygon's
        #    latitude range widened by 2e-9): seam latitudes +- ulps, x across the polygon
        k = min(65536, max(1, 2 * n))
        y_lo, y_hi = v[:, 0].min() - 2e-9, v[:, 0].max() + 2e-9
        seams = y_lo + np.arange(k + 1) * ((y_hi - y_lo) / k)
        seams2 = y_lo + np.arange(k + 1) / (k / (y_hi - y_lo))
        for s in (seams, seams2):
            for dk in (0, 1, -1, 2, -2, 8, -8):
                for x in (rng.uniform(x_lo, x_hi, k + 1), rng.uniform(x_lo, x_hi, k + 1)):
                    pts.append(np.stack([ulp_shift(s, dk), x], axis=1))
        p = np.concatenate(pts)
        if len(p) > per_ring_cap:
            p = p[rng.choice(len(p), per_ring_cap, replace=False)]
        out.append(p)
    p = np.concatenate(out) if out else np.zeros((0, 2))
    good = (np.abs(p[:, 0]) <= 90.0) & (np.abs(p[:, 1]) <= 180.0) & np.isfinite(p).all(axis=1)
    return np.ascontiguousarray(p[good])


def special_polygons():
    """Hand-made rings (lat, lng) around (40.7, -74.0) with the shapes random stars never
    have: exactly horizontal and vertical edges, edges whose end latitudes differ by 1-3
    ulps, many vertices on one latitude (a ray through all of them), collinear vertices
    in the middle of a straight edge, a very long flat edge, and a sliver."""
    y0, x0 = 40.7, -74.0
    up = lambda y, k: float(ulp_shift(np.array([y]), k)[0])
    rings = []
    # 0: axis-aligned rectangle with collinear mid-edge vertices
    rings.append([(y0, x0), (y0, x0 + 0.005), (y0, x0 + 0.01), (y0 + 0.004, x0 + 0.01), (y0 + 0.008, x0 + 0.01),
                  (y0 + 0.008, x0 + 0.005), (y0 + 0.008, x0), (y0 + 0.004, x0)])
    # 1: "rectangle" whose horizontal edges are off by 1 and 3 ulps end to end
    b = y0 + 0.02
    rings.append([(b, x0), (up(b, 1), x0 + 0.01), (up(b + 0.006, 3), x0 + 0.01), (b + 0.006, x0)])
    # 2: comb — the teeth tips share one latitude, the notches another (rays through many vertices)
    c, teeth = y0 + 0.04, 12
    comb = [(c, x0)]
    for t in range(teeth):
        xa = x0 + 0.001 * (2 * t)
        comb += [(c + 0.003, xa), (c + 0.003, xa + 0.001), (c + 0.001, xa + 0.001), (c + 0.001, xa + 0.002)]
    comb += [(c + 0.003, x0 + 0.001 * 2 * teeth), (c + 0.003, x0 + 0.001 * 2 * teeth + 0.001),
             (c, x0 + 0.001 * 2 * teeth + 0.001)]
    rings.append(comb)
    # 3: sliver triangle with a tiny-slope long edge
    s = y0 - 0.02
    rings.append([(s, x0), (s + 1e-9, x0 + 0.02), (s + 0.0005, x0 + 0.01)])
    # 4: diamond whose left and right vertices share a latitude with rectangle 0's top edge
    d = y0 + 0.008
    rings.append([(d, x0 + 0.02), (d - 0.003, x0 + 0.023), (d, x0 + 0.026), (d + 0.003, x0 + 0.023)])
    # 5: staircase: alternating exactly horizontal / exactly vertical edges
    q, stair = y0 - 0.01, [(y0 - 0.01, x0 + 0.03)]
    for t in range(8):
        stair += [(q + 0.0005 * t, x0 + 0.03 + 0.0007 * (t + 1)), (q + 0.0005 * (t + 1), x0 + 0.03 + 0.0007 * (t + 1))]
    stair += [(q + 0.0005 * 8, x0 + 0.03)]
    rings.append(stair)
    return [np.array(r, np.float64) for r in rings]


def special_points(rings, rng: np.random.Generator) -> np.ndarray:
    """adversarial_points plus dense samples ON the horizontal / vertical edges and a
    random background."""
    pts = [adversarial_points(rings, rng)]
    for ring in rings:
        v = np.asarray(ring)
        a, b = v, np.roll(v, -1, axis=0)
        for i in range(len(v)):
            t = rng.uniform(-0.05, 1.05, 300)[:, None]
            on = a[i] + t * (b[i] - a[i])
            for dk in (0, 1, -1, 3, -3):
                pts.append(np.stack([ulp_shift(on[:, 0], dk), on[:, 1]], axis=1))
                pts.append(np.stack([on[:, 0], ulp_shift(on[:, 1], dk)], axis=1))
    lo = np.min([r.min(axis=0) for r in rings], axis=0) - 0.002
    hi = np.max([r.max(axis=0) for r in rings], axis=0) + 0.002
    pts.append(np.stack([rng.uniform(lo[0], hi[0], 200_000), rng.uniform(lo[1], hi[1], 200_000)], axis=1))
    return np.ascontiguousarray(np.concatenate(pts))
