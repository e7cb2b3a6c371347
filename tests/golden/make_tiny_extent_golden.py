"""Generates tests/golden/kmax60_tiny_*.npz from the compiled reference (build container only):

    python tests/golden/make_tiny_extent_golden.py

k_max = 60 indexes over extents so small that the face prefix takes its maximum of 48 bits (act.cpp:62-68: the
prefix stops 8 bits short of the shortest key): the trie is one or two node steps deep and its LAST step ends at
"level 32", two grid levels below the leaf level (a k_max-60 node under 56 key bits uses 4 of its 8 slot bits).
The device index must not take a directory tier there (such an index was rejected as corrupt
although the reference loads and probes it)."""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle import ref  # noqa: E402
from tests import golden_util  # noqa: E402
from tests.golden.make_golden import join_fixture  # noqa: E402
from tests.refrng import Rng, random_points_in, random_star_polygon  # noqa: E402


def main():
    lat_cell24 = 180.0 / (1 << 24)
    lng_cell24 = 360.0 / (1 << 24)
    for name, radius, fine in (("kmax60_tiny_a", 1.6e-6, False), ("kmax60_tiny_b", 1.1e-7, True)):
        rng = Rng(0x7171 + int(fine))
        # centre of a level-24 cell (so the polygon does not straddle a coarser cell boundary)
        clat = (int((1.0 + 90.0) / lat_cell24) + 0.5) * lat_cell24 - 90.0
        clng = (int((1.0 + 180.0) / lng_cell24) + 0.5) * lng_cell24 - 180.0
        if fine:  # centre of a level-28 cell
            clat = (int((1.0 + 90.0) / (lat_cell24 / 16)) + 0.5) * (lat_cell24 / 16) - 90.0
            clng = (int((1.0 + 180.0) / (lng_cell24 / 16)) + 0.5) * (lng_cell24 / 16) - 180.0
        ring = random_star_polygon(rng, clat, clng, radius, 7)
        ref.validate_polygon(ring)
        polys = ref.Polygons.from_rings([ring], ids=[5])
        pts = random_points_in(rng, clat - 4 * radius, clat + 4 * radius, clng - 4 * radius, clng + 4 * radius, 4000)
        pts[:7] = ring
        pts[7:14] = (ring + np.roll(ring, -1, axis=0)) * 0.5
        b = join_fixture(name, polys, ref.default_config(mode_approx=0, k_max=60, memory_budget_bytes=1 << 30), pts)
        g = golden_util.parse_gjx(golden_util.gjx_bytes(golden_util.load(name)))
        print(f"  {name}: prefix_bits {int(g['prefix_bits'][0])} nodes {len(g['arena']) // 256}")
        assert int(g["prefix_bits"][0]) == 48, "choose another extent"


if __name__ == "__main__":
    main()
