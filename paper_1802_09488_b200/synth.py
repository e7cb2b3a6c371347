"""Seeded synthetic workloads standing in for the paper's NYC datasets.

The paper measures on NYC taxi points joined with boroughs / neighbourhoods /
census blocks; none of those files are available, so
BASELINE.json's five configs are reproduced here as seeded synthetic inputs
with the same polygon counts, extent and point skew:

* jittered-Voronoi tessellations of a 0.45° x 0.55° box whose shared edges are
  replaced by midpoint-displacement polylines (identical vertices in both
  neighbours, so the tessellation stays gap- and overlap-free);
* star-shaped overlapping polygons (the family of the reference's
  ``random_star_polygon`` test helper, tests/oracles.hpp:161-174);
* uniform / Gaussian-mixture / on-boundary probe points.

Everything is a pure function of its seed.  Points are AoS float64
``(lat, lng)`` pairs — the reference's ``LatLng`` layout (latlng.hpp:26-29).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

# SW corner (40.50, -74.25) -> NE corner (40.95, -73.70): SURVEY.md §8d.
BOX = (40.50, 40.95, -74.25, -73.70)  # lat_lo, lat_hi, lng_lo, lng_hi
BASE_SEED = 0x180209488
METERS_PER_DEG = 111195.0


def seed_for(config: int, stream: int) -> int:
    """stream: 0 polygons, 1 training points, 2 probe points."""
    return BASE_SEED + 1000 * config + stream


def _rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seed))


@dataclass
class PolygonSet:
    """CSR polygons: ids[P], vtx_off[P+1], latlng[sum V, 2] (ring, first vertex not repeated)."""
    ids: np.ndarray
    vtx_off: np.ndarray
    latlng: np.ndarray

    def ring(self, i: int) -> np.ndarray:
        return self.latlng[int(self.vtx_off[i]):int(self.vtx_off[i + 1])]

    def __len__(self) -> int:
        return len(self.ids)

    @property
    def vertex_counts(self) -> np.ndarray:
        return np.diff(self.vtx_off.astype(np.int64))

    @staticmethod
    def from_rings(rings, ids=None) -> "PolygonSet":
        ids = np.arange(len(rings), dtype=np.uint32) if ids is None else np.asarray(ids, np.uint32)
        off = np.zeros(len(rings) + 1, np.uint64)
        off[1:] = np.cumsum([len(r) for r in rings])
        ll = np.concatenate(rings).astype(np.float64) if len(rings) else np.zeros((0, 2))
        return PolygonSet(ids, off, np.ascontiguousarray(ll))


# ----------------------------------------------------------------------------
# ring validity (planar, x = lng, y = lat)
# ----------------------------------------------------------------------------
def ring_is_simple(ring: np.ndarray) -> bool:
    """True when no two non-adjacent edges touch or cross and no consecutive
    vertices repeat (the reference's validate_polygon rejects both)."""
    n = len(ring)
    if n < 3:
        return False
    a = ring
    b = np.roll(ring, -1, axis=0)
    if np.any(np.all(a == b, axis=1)):
        return False
    ax, ay, bx, by = a[:, 1], a[:, 0], b[:, 1], b[:, 0]
    # bounding-box prefilter on all pairs, then orientation tests on survivors
    lox, hix = np.minimum(ax, bx), np.maximum(ax, bx)
    loy, hiy = np.minimum(ay, by), np.maximum(ay, by)
    for i0 in range(0, n, 512):  # blocks keep the broadcast memory bounded
        i1 = min(n, i0 + 512)
        ov = ((lox[i0:i1, None] <= hix[None, :]) & (lox[None, :] <= hix[i0:i1, None]) &
              (loy[i0:i1, None] <= hiy[None, :]) & (loy[None, :] <= hiy[i0:i1, None]))
        ii, jj = np.nonzero(ov)
        ii = ii + i0
        keep = (jj > ii + 1) & ~((ii == 0) & (jj == n - 1))
        ii, jj = ii[keep], jj[keep]
        if len(ii) == 0:
            continue

        def orient(px, py, qx, qy, rx, ry):
            return (qx - px) * (ry - py) - (qy - py) * (rx - px)

        d1 = orient(ax[ii], ay[ii], bx[ii], by[ii], ax[jj], ay[jj])
        d2 = orient(ax[ii], ay[ii], bx[ii], by[ii], bx[jj], by[jj])
        d3 = orient(ax[jj], ay[jj], bx[jj], by[jj], ax[ii], ay[ii])
        d4 = orient(ax[jj], ay[jj], bx[jj], by[jj], bx[ii], by[ii])
        cross = (d1 * d2 <= 0) & (d3 * d4 <= 0)
        if np.any(cross):
            return False
    return True


# ----------------------------------------------------------------------------
# Voronoi tessellation with fractal shared edges
# ----------------------------------------------------------------------------
def _sites(n: int, rng: np.random.Generator, box) -> np.ndarray:
    lat_lo, lat_hi, lng_lo, lng_hi = box
    g = int(round(np.sqrt(n)))
    if g * g == n and n >= 16:  # jittered grid
        iy, ix = np.divmod(np.arange(n), g)
        u = (ix + 0.5 + rng.uniform(-0.38, 0.38, n)) / g
        v = (iy + 0.5 + rng.uniform(-0.38, 0.38, n)) / g
    else:  # few sites: rejection-sample a minimum spacing
        pts = []
        min_d = 0.45 / np.sqrt(n)
        while len(pts) < n:
            c = rng.uniform(0.08, 0.92, 2)
            if all(np.hypot(*(c - p)) >= min_d for p in pts):
                pts.append(c)
        u, v = np.array(pts)[:, 0], np.array(pts)[:, 1]
    return np.stack([lat_lo + v * (lat_hi - lat_lo), lng_lo + u * (lng_hi - lng_lo)], axis=1)


def _displace(p0: np.ndarray, p1: np.ndarray, depth: int, amp: float,
              rng: np.random.Generator) -> np.ndarray:
    """Midpoint-displacement polyline from p0 to p1 with 2**depth segments."""
    pts = np.stack([p0, p1])
    for _ in range(depth):
        a, b = pts[:-1], pts[1:]
        d = b - a
        normal = np.stack([-d[:, 1], d[:, 0]], axis=1)  # |normal| == |d|
        mid = (a + b) * 0.5 + normal * (amp * rng.uniform(-1.0, 1.0, len(a)))[:, None]
        out = np.empty((2 * len(a) + 1, 2))
        out[0::2] = pts
        out[1::2] = mid
        pts = out
    return pts


def voronoi_tessellation(n_sites: int, seed: int, mean_vertices: float,
                         max_depth: int = 9, amp: float = 0.22, box=BOX) -> PolygonSet:
    """n_sites non-overlapping simple polygons tiling ``box``."""
    from scipy.spatial import Voronoi

    rng = _rng(seed)
    lat_lo, lat_hi, lng_lo, lng_hi = box
    sites = _sites(n_sites, rng, box)
    # Mirror the sites across the four box edges: the cells of the original
    # sites then end exactly on the box (standard bounded-Voronoi trick).
    m = [sites]
    for axis, lo, hi in ((0, lat_lo, lat_hi), (1, lng_lo, lng_hi)):
        for edge in (lo, hi):
            r = sites.copy()
            r[:, axis] = 2 * edge - r[:, axis]
            m.append(r)
    vor = Voronoi(np.concatenate(m))
    verts = vor.vertices.copy()
    # snap the vertices that lie on the box to it exactly
    for axis, lo, hi in ((0, lat_lo, lat_hi), (1, lng_lo, lng_hi)):
        for edge in (lo, hi):
            near = np.abs(verts[:, axis] - edge) < 1e-9
            verts[near, axis] = edge

    ridge_sites = vor.ridge_points
    ridge_verts = np.asarray(vor.ridge_vertices)
    inner = (ridge_sites < n_sites).any(axis=1)
    assert (ridge_verts[inner] >= 0).all(), "bounded cells expected"
    shared = (ridge_sites < n_sites).all(axis=1)
    length = np.zeros(len(ridge_verts))
    length[inner] = np.hypot(*(verts[ridge_verts[inner, 0]] - verts[ridge_verts[inner, 1]]).T)

    # Pick the segment length so the mean ring size lands near mean_vertices:
    # every shared ridge of length L gets 2**d segments, d = round(log2(L/seg)).
    def depths(seg):
        d = np.zeros(len(length), np.int64)
        ok = shared & (length > 0)
        d[ok] = np.clip(np.round(np.log2(length[ok] / seg)), 0, max_depth).astype(np.int64)
        return d

    def mean_ring(seg):
        d = depths(seg)
        per_site = np.zeros(n_sites)
        for k in (0, 1):
            s = ridge_sites[inner, k]
            mask = s < n_sites
            np.add.at(per_site, s[mask], (2.0 ** d[inner])[mask])
        return per_site.mean()

    lo_s, hi_s = 1e-7, 1.0
    for _ in range(60):  # bisection on a monotone step function
        mid = np.sqrt(lo_s * hi_s)
        if mean_ring(mid) > mean_vertices:
            lo_s = mid
        else:
            hi_s = mid
    seg = hi_s
    depth = depths(seg)

    # Several passes with shrinking amplitude until every ring is simple.
    cur_amp = amp
    for _attempt in range(12):
        lines: dict[tuple[int, int], np.ndarray] = {}
        for r in np.nonzero(inner)[0]:
            v0, v1 = sorted(ridge_verts[r])
            if v0 == v1:
                continue
            if shared[r] and depth[r] > 0:
                rr = _rng((seed * 1000003 + int(v0) * 7919 + int(v1)) & 0x7FFFFFFFFFFFFFFF)
                lines[(v0, v1)] = _displace(verts[v0], verts[v1], int(depth[r]), cur_amp, rr)
            else:
                lines[(v0, v1)] = np.stack([verts[v0], verts[v1]])
        rings = []
        ok = True
        for s in range(n_sites):
            region = [v for v in vor.regions[vor.point_region[s]]]
            assert -1 not in region
            rv = verts[region]
            ang = np.arctan2(rv[:, 0] - sites[s, 0], rv[:, 1] - sites[s, 1])
            order = [region[k] for k in np.argsort(ang)]
            parts = []
            for k, va in enumerate(order):
                vb = order[(k + 1) % len(order)]
                if va == vb:
                    continue
                key = (min(va, vb), max(va, vb))
                line = lines.get(key)
                if line is None:  # coincident vertices collapsed a ridge
                    line = np.stack([verts[key[0]], verts[key[1]]])
                parts.append(line[:-1] if va < vb else line[::-1][:-1])
            ring = np.concatenate(parts)
            keep = np.ones(len(ring), bool)
            keep[1:] = np.any(ring[1:] != ring[:-1], axis=1)
            if np.all(ring[0] == ring[-1]):
                keep[-1] = False
            ring = ring[keep]
            if not ring_is_simple(ring):
                ok = False
                break
            rings.append(ring)
        if ok:
            return PolygonSet.from_rings(rings)
        cur_amp *= 0.7
    raise RuntimeError("could not build a simple tessellation")


# ----------------------------------------------------------------------------
# overlapping star polygons (BASELINE config 5)
# ----------------------------------------------------------------------------
def star_polygons(n: int, seed: int, vertices=(16, 128), radius_m=(50.0, 2000.0),
                  box=BOX) -> PolygonSet:
    """Star-shaped rings: strictly increasing vertex angles, so simple by
    construction (same family as tests/oracles.hpp:161-174)."""
    rng = _rng(seed)
    lat_lo, lat_hi, lng_lo, lng_hi = box
    rings = []
    for _ in range(n):
        clat = rng.uniform(lat_lo, lat_hi)
        clng = rng.uniform(lng_lo, lng_hi)
        k = int(rng.integers(vertices[0], vertices[1] + 1))
        r_m = rng.uniform(radius_m[0], radius_m[1])
        ang = (np.arange(k) + 0.2 + 0.6 * rng.random(k)) * (2.0 * np.pi / k)
        rad = r_m * rng.uniform(0.55, 1.45, k)
        dlat = rad * np.sin(ang) / METERS_PER_DEG
        dlng = rad * np.cos(ang) / (METERS_PER_DEG * np.cos(np.deg2rad(clat)))
        rings.append(np.stack([clat + dlat, clng + dlng], axis=1))
    return PolygonSet.from_rings(rings)


# ----------------------------------------------------------------------------
# points
# ----------------------------------------------------------------------------
def uniform_points(n: int, seed: int, box=BOX, out: np.ndarray | None = None) -> np.ndarray:
    rng = _rng(seed)
    lat_lo, lat_hi, lng_lo, lng_hi = box
    pts = np.empty((n, 2), np.float64) if out is None else out
    chunk = 1 << 22
    for b in range(0, n, chunk):
        e = min(n, b + chunk)
        u = rng.random((e - b, 2))
        pts[b:e, 0] = lat_lo + (lat_hi - lat_lo) * u[:, 0]
        pts[b:e, 1] = lng_lo + (lng_hi - lng_lo) * u[:, 1]
    return pts


@dataclass
class Mixture:
    centres: np.ndarray
    sigma: np.ndarray
    weights: np.ndarray
    background: float


def gaussian_mixture(seed: int, components: int = 40, sigma=(0.002, 0.02), zipf: float = 1.1,
                     background: float = 0.10, box=BOX) -> Mixture:
    rng = _rng(seed ^ 0x5A5A5A5A)
    lat_lo, lat_hi, lng_lo, lng_hi = box
    centres = np.stack([rng.uniform(lat_lo, lat_hi, components),
                        rng.uniform(lng_lo, lng_hi, components)], axis=1)
    sig = rng.uniform(sigma[0], sigma[1], components)
    w = 1.0 / np.arange(1, components + 1) ** zipf
    return Mixture(centres, sig, w / w.sum(), background)


def mixture_points(n: int, seed: int, mix: Mixture, box=BOX, out: np.ndarray | None = None) -> np.ndarray:
    """Zipf-weighted isotropic Gaussians + uniform background; samples are
    clamped into valid lat/lng (never needed for this box) so every point is
    a legal reference input."""
    rng = _rng(seed)
    lat_lo, lat_hi, lng_lo, lng_hi = box
    pts = np.empty((n, 2), np.float64) if out is None else out
    chunk = 1 << 22
    for b in range(0, n, chunk):
        e = min(n, b + chunk)
        m = e - b
        comp = rng.choice(len(mix.weights), size=m, p=mix.weights)
        z = rng.standard_normal((m, 2))
        p = mix.centres[comp] + z * mix.sigma[comp][:, None]
        bg = rng.random(m) < mix.background
        nb = int(bg.sum())
        if nb:
            u = rng.random((nb, 2))
            p[bg, 0] = lat_lo + (lat_hi - lat_lo) * u[:, 0]
            p[bg, 1] = lng_lo + (lng_hi - lng_lo) * u[:, 1]
        np.clip(p[:, 0], -90.0, 90.0, out=p[:, 0])
        np.clip(p[:, 1], -180.0, 180.0, out=p[:, 1])
        pts[b:e] = p
    return pts


def plant_boundary_points(points: np.ndarray, polys: PolygonSet, seed: int, fraction: float = 0.01) -> np.ndarray:
    """Overwrite ``fraction`` of the points with exact boundary points: half a
    polygon vertex verbatim, half ``a + t*(b-a)`` on an edge — ST_Covers counts
    both as inside every adjacent polygon (geometry.cpp:28-29,184-193).
    Returns the indices that were replaced."""
    rng = _rng(seed ^ 0xB0DA)
    n = len(points)
    k = int(n * fraction)
    if k == 0:
        return np.zeros(0, np.int64)
    idx = rng.choice(n, size=k, replace=False)
    nv = len(polys.latlng)
    off = polys.vtx_off.astype(np.int64)
    v = rng.integers(0, nv, size=k)
    poly_of = np.searchsorted(off, v, side="right") - 1
    nxt = v + 1
    wrap = nxt >= off[poly_of + 1]
    nxt[wrap] = off[poly_of[wrap]]
    a = polys.latlng[v]
    b = polys.latlng[nxt]
    t = rng.random(k)
    t[: k // 2] = 0.0  # vertex verbatim
    points[idx] = a + t[:, None] * (b - a)
    return idx


# ----------------------------------------------------------------------------
# BASELINE.json configs (polygons + index parameters + point distribution)
# ----------------------------------------------------------------------------
@dataclass
class WorkloadSpec:
    name: str
    config: int
    n_points: int
    exact: bool            # join mode
    build_approx: bool     # JoinConfig::mode handed to build_index
    precision_m: float
    k_max: int
    budget_bytes: int
    training_points: int
    distribution: str      # "uniform" | "mixture"
    boundary_fraction: float


SPECS = {
    1: WorkloadSpec("cfg1_5poly_approx60m", 1, 1_000_000, False, True, 60.0, 48, 1 << 30, 0, "uniform", 0.0),
    2: WorkloadSpec("cfg2_289poly_approx4m", 2, 100_000_000, False, True, 4.0, 48, 8 << 30, 0, "uniform", 0.0),
    3: WorkloadSpec("cfg3_289poly_exact_trained", 3, 100_000_000, True, False, 10.0, 48, 4 << 30,
                    10_000_000, "mixture", 0.01),
    4: WorkloadSpec("cfg4_40kpoly_approx1m", 4, 1_000_000_000, False, True, 1.0, 56, 64 << 30, 0, "mixture", 0.0),
    5: WorkloadSpec("cfg5_10kstars_exact15m", 5, 500_000_000, True, True, 15.0, 48, 16 << 30, 0, "uniform", 0.0),
}


def box_for(config: int, scale: float = 1.0):
    """Configs 4 and 5 scale down DENSITY-MATCHED: ``scale`` of the polygons in
    ``scale`` of the area (a centred sub-box), so polygon size, overlap and the
    index depth per point stay those of the full config."""
    if scale >= 1.0 or config not in (4, 5):
        return BOX
    lat_lo, lat_hi, lng_lo, lng_hi = BOX
    f = float(np.sqrt(scale))
    clat, clng = (lat_lo + lat_hi) / 2, (lng_lo + lng_hi) / 2
    hlat, hlng = (lat_hi - lat_lo) / 2 * f, (lng_hi - lng_lo) / 2 * f
    return (clat - hlat, clat + hlat, clng - hlng, clng + hlng)


def polygons_for(config: int, scale: float = 1.0) -> PolygonSet:
    """Polygons of a BASELINE config; ``scale`` < 1 shrinks the polygon COUNT
    (for configs 4 and 5 together with the box, see box_for)."""
    s = seed_for(config, 0)
    if config == 1:
        return voronoi_tessellation(5, s, mean_vertices=1100.0, max_depth=9)
    if config in (2, 3):
        n = max(4, int(round(289 * scale)))
        g = int(round(np.sqrt(n)))
        return voronoi_tessellation(g * g if g * g >= 16 else n, seed_for(2, 0), mean_vertices=150.0)
    if config == 4:
        n = max(16, int(round(40_000 * scale)))
        g = int(round(np.sqrt(n)))
        return voronoi_tessellation(g * g, s, mean_vertices=15.0, max_depth=3, box=box_for(4, scale))
    if config == 5:
        return star_polygons(max(4, int(round(10_000 * scale))), s, box=box_for(5, scale))
    raise ValueError(config)


def points_for(config: int, n: int, polys: PolygonSet | None = None, stream: int = 2,
               out: np.ndarray | None = None, scale: float = 1.0) -> np.ndarray:
    spec = SPECS[config]
    s = seed_for(config, stream)
    box = box_for(config, scale)
    if spec.distribution == "uniform":
        pts = uniform_points(n, s, box=box, out=out)
    else:
        f = float(np.sqrt(scale)) if box is not BOX else 1.0
        mix = gaussian_mixture(seed_for(3, 1), sigma=(0.002 * f, 0.02 * f), box=box)
        pts = mixture_points(n, s, mix, box=box, out=out)
    if spec.boundary_fraction > 0 and polys is not None and stream == 2:
        plant_boundary_points(pts, polys, s, spec.boundary_fraction)
    return pts
