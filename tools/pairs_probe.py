"""Times Session.join_pairs (gj_join_pairs_host + gj_pairs_copy) on a BASELINE
config; under ncu it yields the per-kernel split of the CSR pipeline.

    python tools/pairs_probe.py CONFIG [--scale S] [--points N]
"""
from __future__ import annotations

import argparse
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_1802_09488_b200 import capi, join, synth  # noqa: E402
from tools import build_bundles  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", type=int)
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--points", type=int, default=20_000_000)
    args = ap.parse_args()
    spec = synth.SPECS[args.config]
    path = build_bundles.ensure_workload_bundle(args.config, args.scale)
    bundle = join.IndexBundle.load(path, device=0)
    s = bundle.session()
    polys = synth.polygons_for(args.config, args.scale) if spec.boundary_fraction > 0 else None
    pts = synth.points_for(args.config, args.points, polys, scale=args.scale)
    mode = capi.GJ_MODE_EXACT if spec.exact else capi.GJ_MODE_APPROX
    s.join_pairs(pts[:1_000_000], mode)
    for _ in range(2):
        t0 = time.time()
        row_ptr, ids = s.join_pairs(pts, mode)
        dt = time.time() - t0
        print(f"config {args.config}: {len(pts)} points, {int(row_ptr[-1])} pairs, {dt:.3f} s, "
              f"{len(pts) / dt / 1e6:.1f} M points/s, {int(row_ptr[-1]) / dt / 1e6:.1f} M pairs/s", flush=True)


if __name__ == "__main__":
    main()
