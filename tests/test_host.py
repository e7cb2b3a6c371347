"""CPU tests of the host side: the C-ABI library loads and exports every
declared symbol, fails loudly without a GPU, the GJX1 reader used by the test
infrastructure agrees with the reference's in-memory views, the synthetic
generators are deterministic and produce valid polygons."""
import ctypes as C
import re
from pathlib import Path

import numpy as np
import pytest

from paper_1802_09488_b200 import capi, join, synth
from tests import golden_util
from tests.refrng import Rng

ROOT = Path(__file__).resolve().parent.parent


def test_library_exports_every_declared_symbol():
    header = (ROOT / "include" / "geojoin_b200.h").read_text()
    declared = set(re.findall(r"GJ_API\s+[\w\s\*]+?\b(gj_\w+)\s*\(", header))
    assert declared, "no declarations parsed"
    assert declared == set(capi.EXPORTS)
    L = capi.lib()
    for name in declared:
        assert getattr(L, name) is not None


def test_header_structs_match_ctypes_layout():
    assert C.sizeof(capi.IndexDesc) == 8 + 8 + 8 + 8 + 3 * 64 + 4 + 4 + 8 + 3 * 8
    assert C.sizeof(capi.Stats) == 48
    assert C.sizeof(capi.IndexInfo) == 5 * 8 + 18 * 4
    assert C.sizeof(capi.Overflow) == 32
    assert C.sizeof(capi.Options) == 17 * 4 + 4 + 2 * 8  # 17 words, padding, two u64
    o = capi.Options(tier_sub=2)  # gj_options_default + overrides
    assert o.struct_size == C.sizeof(capi.Options) and o.tier_sub == 2
    assert (o.ids_late, o.hist_rep_cap, o.node_pal_max_mb, o.max_launch_points, o.chunk_points) == (-1, -1, -1, 0, 0)


def test_library_reads_no_environment_variable():
    """Tuning knobs and test hooks travel in gj_options; a stray variable in a user's
    environment must not change kernel variants or launch splitting."""
    for f in (ROOT / "paper_1802_09488_b200" / "csrc").iterdir():
        assert "getenv" not in f.read_text(), f"{f.name} reads the environment"


def test_no_gpu_means_loud_failure():
    """There is no CPU fallback: without a device every entry point errors."""
    L = capi.lib()
    if L.gj_device_count() > 0:
        pytest.skip("a GPU is present")
    with pytest.raises(join.CudaError):
        join.IndexBundle.load(golden_util.bundle_file("join_small_exact"))
    fx = golden_util.load("join_small_exact")
    g = golden_util.parse_gjx(golden_util.gjx_bytes(fx))
    with pytest.raises(join.CudaError):
        join.IndexBundle.from_arrays(g["arena"], g["lut"], g["roots"], g["prefixes"], g["prefix_bits"],
                                     g["k_max"], g["approx"], g["polygon_ids"], g["vtx_off"], g["vtx_latlng"])


def test_product_package_does_not_use_the_oracle():
    """Only tests/, smoke() and bench.py's CPU legs may import, link or execute
    anything under oracle/; the product package must not."""
    bad = re.compile(r"(^\s*(from|import)\s+oracle\b)|libgeojoin_oracle|libgeojoin_ref|oracle/|geojoin_oracle\.h",
                     re.MULTILINE)
    for path in list((ROOT / "paper_1802_09488_b200").rglob("*")) + list((ROOT / "include").rglob("*")):
        if path.suffix in (".py", ".cu", ".cuh", ".hpp", ".h"):
            m = bad.search(path.read_text())
            assert m is None, f"{path} references the oracle: {m.group(0)!r}"


def test_gjx_parser_matches_reference_views(ref_available):
    if not ref_available:
        pytest.skip("oracle/_ref not built")
    from oracle import ref
    fx = golden_util.load("cfg2_tess16_approx4m")
    g = golden_util.parse_gjx(golden_util.gjx_bytes(fx))
    b = ref.RefBundle.load(golden_util.bundle_file("cfg2_tess16_approx4m"))
    arena, lut, roots, prefixes, pbits = b.view()
    assert np.array_equal(g["arena"], arena) and np.array_equal(g["lut"], lut)
    assert np.array_equal(g["roots"], roots) and np.array_equal(g["prefixes"], prefixes)
    assert np.array_equal(g["prefix_bits"], pbits)
    polys = b.polygons()
    assert np.array_equal(g["polygon_ids"], polys.ids) and np.array_equal(g["vtx_latlng"], polys.latlng)
    assert g["k_max"] == b.k_max and g["approx"] == b.approx


def test_mt19937_64_check_value():
    """The C++ standard's check value: the 10000th output of a default-seeded mt19937_64."""
    r = Rng(5489)
    v = 0
    for _ in range(10000):
        v = r.u64()
    assert v == 9981545732273789042


def test_synth_is_deterministic_and_valid():
    a = synth.voronoi_tessellation(16, 1234, mean_vertices=60.0)
    b = synth.voronoi_tessellation(16, 1234, mean_vertices=60.0)
    assert np.array_equal(a.latlng, b.latlng) and np.array_equal(a.vtx_off, b.vtx_off)
    lat_lo, lat_hi, lng_lo, lng_hi = synth.BOX
    assert a.latlng[:, 0].min() >= lat_lo and a.latlng[:, 0].max() <= lat_hi
    assert a.latlng[:, 1].min() >= lng_lo and a.latlng[:, 1].max() <= lng_hi
    for i in range(len(a)):
        assert synth.ring_is_simple(a.ring(i))
    # shared edges carry identical vertices in both neighbours: the rings tile
    # the box, so signed areas add up to the box area
    def area(r):
        x, y = r[:, 1], r[:, 0]
        return 0.5 * abs(np.dot(x, np.roll(y, -1)) - np.dot(y, np.roll(x, -1)))
    total = sum(area(a.ring(i)) for i in range(len(a)))
    assert abs(total - (lat_hi - lat_lo) * (lng_hi - lng_lo)) < 1e-9
    stars = synth.star_polygons(20, 99)
    assert all(synth.ring_is_simple(stars.ring(i)) for i in range(len(stars)))
    assert 16 <= stars.vertex_counts.min() and stars.vertex_counts.max() <= 128


def test_synth_points():
    p = synth.uniform_points(10000, 7)
    assert np.array_equal(p, synth.uniform_points(10000, 7))
    lat_lo, lat_hi, lng_lo, lng_hi = synth.BOX
    assert (p[:, 0] >= lat_lo).all() and (p[:, 0] <= lat_hi).all()
    mix = synth.gaussian_mixture(3)
    q = synth.mixture_points(20000, 8, mix)
    assert np.isfinite(q).all() and (np.abs(q[:, 0]) <= 90).all() and (np.abs(q[:, 1]) <= 180).all()
    polys = synth.voronoi_tessellation(9, 5, mean_vertices=30.0)
    idx = synth.plant_boundary_points(q, polys, 9, 0.05)
    assert len(idx) == 1000
    verts = {tuple(v) for v in polys.latlng}
    assert sum(tuple(q[i]) in verts for i in idx) >= 400  # about half are vertices verbatim


def test_ring_is_simple_rejects_bowtie():
    bow = np.array([[0.0, 0.0], [1.0, 1.0], [0.0, 1.0], [1.0, 0.0]])
    assert not synth.ring_is_simple(bow)
    assert synth.ring_is_simple(np.array([[0.0, 0.0], [0.0, 1.0], [1.0, 1.0], [1.0, 0.0]]))


def _fma_exact(v: float, r: float, c: float) -> float:
    """RN(v*r + c) with one rounding, like the device fma: exact rational
    arithmetic, then Fraction -> float (correctly rounded int true division)."""
    from fractions import Fraction
    return float(Fraction(v) * Fraction(r) + Fraction(c))


def test_fast_grid_coordinates_claim():
    """The arithmetic claim behind csrc/gj_device.cuh::grid_xy_try, checked on
    the CPU without any CUDA: t = fma(v, RN(2^30/span), 2^31 + 2^29); whenever t
    has exponent 0x41E with a clear top mantissa bit and its 21-bit fraction
    field lies in [2, 2^21 - 3], v is inside [lo, hi] and the 30 bits above the
    fraction are exactly trunc(((v - lo) / span) * 2^30) as the reference
    computes it (cell_id.cpp:50-56); otherwise the fast path must refuse."""
    import struct
    rng = np.random.default_rng(0xF4A)
    accepted = refused = 0
    for lo, span in ((-90.0, 180.0), (-180.0, 360.0)):
        hi = lo + span
        r = 1073741824.0 / span
        vals = []
        for level in (30, 27, 24, 16, 3):
            k = rng.integers(0, (1 << level) + 1, 300)
            base = k / float(1 << level) * span + lo
            for ulps in range(-4, 5):
                v = base.copy()
                for _ in range(abs(ulps)):
                    v = np.nextafter(v, np.inf if ulps > 0 else -np.inf)
                vals.append(v)
        vals.append(rng.uniform(lo, hi, 4000))
        vals.append(rng.uniform(-1e-9, 1e-9, 200))
        vals.append(np.array([lo, hi, 0.0, -0.0, 5e-324, -5e-324, np.nextafter(hi, np.inf), np.nextafter(lo, -np.inf),
                              hi + 1.0, lo - 1.0, 1e300, -1e300, np.inf, -np.inf, np.nan]))
        for v in np.concatenate(vals):
            v = float(v)
            valid = lo <= v <= hi  # False for NaN
            if np.isfinite(v):
                t = _fma_exact(v, r, 2147483648.0 + 536870912.0)
            else:
                t = v * r  # inf / nan propagate
            bits = struct.unpack("<Q", struct.pack("<d", t))[0]
            hi_word, frac = bits >> 32, bits & 0x1FFFFF
            ok = ((hi_word ^ 0x41E00000) >> 19) == 0 and 2 <= frac <= (1 << 21) - 3
            if not ok:
                refused += 1
                continue
            accepted += 1
            assert valid, v
            cell = (bits >> 21) & 0x3FFFFFFF
            want = int(np.float64(v - lo) / np.float64(span) * np.float64(1073741824.0))  # the reference's order
            assert cell == min(want, (1 << 30) - 1), (v, cell, want)
    assert accepted > 5000 and refused > 2000
