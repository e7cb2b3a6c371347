"""Times Session.points_from_csv (gj_points_from_csv_host) on synthetic rows;
under ncu it yields the per-kernel split.    python tools/csv_probe.py [ROWS]"""
from __future__ import annotations

import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_1802_09488_b200 import join  # noqa: E402
from tests import golden_util  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 3_000_000
    rng = np.random.default_rng(1)
    lat = rng.uniform(40.5, 40.95, n)
    lng = rng.uniform(-74.25, -73.70, n)
    text = ("id,lat,lng\n" + "\n".join(f"{k},{a!r},{o:.6f}" for k, (a, o) in enumerate(zip(lat.tolist(), lng.tolist())))
            + "\n").encode()
    bundle = join.IndexBundle.load(golden_util.bundle_file("join_small_exact"), device=0)
    s = bundle.session()
    s.points_from_csv(text[:1 << 20].rsplit(b"\n", 1)[0])
    for _ in range(3):
        t0 = time.time()
        pts, sk = s.points_from_csv(text)
        dt = time.time() - t0
        print(f"{len(text) / 1e6:.0f} MB, {len(pts)} points, {sk} skipped: {dt * 1e3:.1f} ms = "
              f"{len(text) / dt / 1e9:.2f} GB/s, {n / dt / 1e6:.1f} M rows/s", flush=True)


if __name__ == "__main__":
    main()
