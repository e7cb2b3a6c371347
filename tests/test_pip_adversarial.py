"""Adversarial parity of the PIP refine path (K2) with the reference's pip_test /
join_exact (proj/src/geometry.cpp:28-39,63-75,184-204; the reference's own cases:
tests/test_geometry.cpp:69-102).  Inputs: tests/pip_adversarial.py; expected
values: tests/golden/pip_adversarial.npz, outputs of the compiled reference
(tests/golden/make_pip_golden.py).

CPU (`not gpu`): the C oracle restatement equals the reference on these inputs —
the golden digests, and pip_test polygon by polygon against the live compiled
reference where it is present.  GPU: join_exact through the C ABI equals the C
oracle pair for pair, and the golden counts / stats / digest."""
import hashlib
import tempfile
import zlib
from pathlib import Path

import numpy as np
import pytest

from paper_1802_09488_b200 import capi, join
from tests import golden_util, pip_adversarial as adv

FIXTURES = ["join_small_exact", "acceptance_exact20", "cfg3_tess16_exact_trained", "cfg5_stars_scaled", "world_stars"]
SEED = 0x9121AD5
_tmp = tempfile.TemporaryDirectory(prefix="gj_pip_")


def _digest(pi, pid):
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(pi, np.uint64).tobytes())
    h.update(np.ascontiguousarray(pid, np.uint32).tobytes())
    return np.frombuffer(h.digest(), np.uint8)


def _case(name):
    """(GJX1 path, parsed bundle, adversarial points, golden dict, key prefix)."""
    gold = golden_util.load("pip_adversarial")
    if name == "special":
        raw = zlib.decompress(gold["special_gjx_z"].tobytes())
        path = Path(_tmp.name) / "special.gjx"
        if not path.exists():
            path.write_bytes(raw)
        g = golden_util.parse_gjx(raw)
        rings = adv.special_polygons()
        assert np.array_equal(np.concatenate(rings), g["vtx_latlng"].reshape(-1, 2))
        pts = adv.special_points(rings, np.random.default_rng(SEED))
    else:
        path = golden_util.bundle_file(name)
        g = golden_util.parse_gjx(golden_util.gjx_bytes(golden_util.load(name)))
        pts = adv.adversarial_points(adv.rings_of(g["vtx_off"], g["vtx_latlng"]),
                                     np.random.default_rng(SEED + 1 + FIXTURES.index(name)), per_ring_cap=60_000)
    assert len(pts) == int(gold[f"{name}_n_points"][0]), "the seeded generator changed: regenerate the golden file"
    return path, g, pts, gold, name


def _check_against_golden(gold, name, pi, pid, stats):
    assert len(pid) == int(gold[f"{name}_n_pairs"][0])
    assert tuple(int(v) for v in stats) == tuple(int(v) for v in gold[f"{name}_stats"])
    ids, cnt = np.unique(pid, return_counts=True)
    assert np.array_equal(ids, gold[f"{name}_count_ids"]) and np.array_equal(cnt.astype(np.uint64), gold[f"{name}_count_values"])
    assert np.array_equal(_digest(pi, pid), gold[f"{name}_digest"])  # every pair, in the reference's order


@pytest.mark.parametrize("name", ["special"] + FIXTURES)
def test_oracle_equals_reference_on_adversarial_points(name):
    path, g, pts, gold, name = _case(name)
    ox = golden_util.oracle_index(g)
    pi, pid, st, _ = ox.join(pts, approx=False)
    _check_against_golden(gold, name, pi, pid, st)


def test_oracle_pip_equals_live_reference_polygon_by_polygon(ref_available):
    """pip_test itself (no index in between): every special polygon against every special point."""
    if not ref_available:
        pytest.skip("oracle/_ref not built")
    from oracle import oracle, ref
    rings = adv.special_polygons()
    pts = adv.special_points(rings, np.random.default_rng(SEED))
    for ring in rings:
        ref.validate_polygon(ring)
        assert np.array_equal(oracle.pip_test(ring, pts), ref.pip_test(ring, pts))
    # the unit-square KATs of tests/test_geometry.cpp:69-78: edge, vertex, just outside
    sq = np.array([[0.0, 0.0], [0.0, 1.0], [1.0, 1.0], [1.0, 0.0]])
    kat = np.array([[0.5, 0.5], [0.0, 0.5], [0.5, 0.0], [1.0, 1.0], [0.5, 1.0000001], [1.5, 0.5], [-1e-13, 0.5]])
    want = np.array([True, True, True, True, False, False, True])
    assert np.array_equal(oracle.pip_test(sq, kat), want) and np.array_equal(ref.pip_test(sq, kat), want)


@pytest.mark.gpu
@pytest.mark.parametrize("strip_index", [0, 1])  # K2's strip lists as 32-byte edge records / as vertex indices
@pytest.mark.parametrize("name", ["special"] + FIXTURES)
def test_gpu_exact_join_on_adversarial_points(name, strip_index):
    path, g, pts, gold, name = _case(name)
    bundle = join.IndexBundle.load(path, device=0, options=capi.Options(strip_index=strip_index))
    s = bundle.session()
    st = join.JoinStats()
    row_ptr, pid = s.join_pairs(pts, capi.GJ_MODE_EXACT, st)
    pi = np.repeat(np.arange(len(pts), dtype=np.uint64), np.diff(row_ptr.astype(np.int64)))
    ox = golden_util.oracle_index(g)
    opi, opid, ost, _ = ox.join(pts, approx=False)
    assert np.array_equal(pi, opi) and np.array_equal(pid, opid)  # pair for pair against the C oracle
    _check_against_golden(gold, name, pi, pid, st.as_tuple())      # and the reference's golden values
    # the streaming join (K1 -> K2 -> counts / first ids / overflow records) on the same points
    st2 = join.JoinStats()
    counts, first, (ovf_pt, ovf_id) = s.join_count(pts, capi.GJ_MODE_EXACT, stats=st2, want_ids=True)
    assert st2.as_tuple() == st.as_tuple()
    assert np.array_equal(counts, np.bincount(np.searchsorted(bundle.ids, pid), minlength=len(bundle.ids)).astype(np.uint64))
    inline = (first != capi.GJ_NO_MATCH) & (first != capi.GJ_DEFERRED)
    p2 = np.concatenate([np.nonzero(inline)[0].astype(np.uint64), ovf_pt])
    i2 = np.concatenate([first[inline] & ~np.uint32(capi.GJ_MORE_FLAG), ovf_id])
    seq = np.concatenate([np.zeros(int(inline.sum()), np.int64), 1 + np.arange(len(ovf_pt), dtype=np.int64)])
    order = np.lexsort((seq, p2))
    assert np.array_equal(p2[order], pi) and np.array_equal(i2[order], pid)
    bundle.close()
