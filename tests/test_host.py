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
    assert C.sizeof(capi.IndexInfo) == 5 * 8 + 16 * 4
    assert C.sizeof(capi.Overflow) == 32


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
