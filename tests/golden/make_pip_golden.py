"""Generates tests/golden/pip_adversarial.npz by running the UNMODIFIED reference
(oracle/_ref) on the adversarial point-in-polygon inputs of
tests/pip_adversarial.py.  Run in the build container only (needs /root/reference):

    python tests/golden/make_pip_golden.py

Holds (a) the GJX1 bundle the reference's build_index makes (exact mode) of the
hand-made special polygons — horizontal / vertical / 1-ulp-slanted edges, many
vertices on one latitude, collinear vertices, slivers — and (b), for that bundle
and for the polygon sets of committed join fixtures, what the reference's
join_exact returns on the seeded adversarial points: per-polygon counts, the six
JoinStats counters, the number of pairs and a SHA-256 of the ordered pair arrays.
The points themselves are regenerated from the seed by the tests (same numpy).
Mirrors tests/test_geometry.cpp:69-102 (pip_test KATs, pip vs winding oracle)."""
from __future__ import annotations

import hashlib
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle import ref  # noqa: E402
from tests import golden_util, pip_adversarial as adv  # noqa: E402
from tests.golden.make_golden import bundle_bytes, save  # noqa: E402

FIXTURES = ["join_small_exact", "acceptance_exact20", "cfg3_tess16_exact_trained", "cfg5_stars_scaled", "world_stars"]
SEED = 0x9121AD5


def pairs_digest(pi: np.ndarray, pid: np.ndarray) -> np.ndarray:
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(pi, np.uint64).tobytes())
    h.update(np.ascontiguousarray(pid, np.uint32).tobytes())
    return np.frombuffer(h.digest(), np.uint8).copy()


def expected(prefix: str, rb: ref.RefBundle, pts: np.ndarray, out: dict):
    pi, pid, st = rb.join_pairs(pts, exact=True)
    ids, cnt = np.unique(pid, return_counts=True)
    out[f"{prefix}_n_points"] = np.array([len(pts)], np.uint64)
    out[f"{prefix}_n_pairs"] = np.array([len(pid)], np.uint64)
    out[f"{prefix}_digest"] = pairs_digest(pi, pid)
    out[f"{prefix}_stats"] = st
    out[f"{prefix}_count_ids"] = ids.astype(np.uint32)
    out[f"{prefix}_count_values"] = cnt.astype(np.uint64)
    print(f"  {prefix}: {len(pts)} points, {len(pid)} pairs, {int(st[1])} pip tests")


def main():
    out = {}
    rings = adv.special_polygons()
    for r in rings:
        ref.validate_polygon(r)
    polys = ref.Polygons.from_rings(rings)
    rb = ref.RefBundle.build(polys, ref.default_config(mode_approx=0, k_max=48))
    assert not rb.approx
    out["special_gjx_z"] = bundle_bytes(rb)
    expected("special", rb, adv.special_points(rings, np.random.default_rng(SEED)), out)
    for k, name in enumerate(FIXTURES):
        g = golden_util.parse_gjx(golden_util.gjx_bytes(golden_util.load(name)))
        fr = adv.rings_of(g["vtx_off"], g["vtx_latlng"])
        pts = adv.adversarial_points(fr, np.random.default_rng(SEED + 1 + k), per_ring_cap=60_000)
        expected(name, ref.RefBundle.load(golden_util.bundle_file(name)), pts, out)
    save("pip_adversarial", **out)


if __name__ == "__main__":
    main()
