"""Times the materialised join (CSR) on a BASELINE config three ways: the two-call
API (gj_join_pairs_host + gj_pairs_copy, pageable arrays), the one-call streaming API
(gj_join_pairs_host_into; pageable and pinned arrays) and the device-resident one
(gj_join_pairs_device), against the PCIe floor of the bytes moved; under ncu it
yields the per-kernel split of the CSR pipeline.

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
    import json

    import numpy as np
    import torch
    n = len(pts)
    res = {"config": args.config, "scale": args.scale, "points": n}
    s.join_pairs(pts[:1_000_000], mode)
    for _ in range(2):
        t0 = time.time()
        row_ptr, ids = s.join_pairs(pts, mode)
        dt = time.time() - t0
    pairs = int(row_ptr[-1])
    res["pairs"] = pairs
    res["two_call_pageable_s"] = dt
    bytes_moved = 16 * n + 8 * (n + 1) + 4 * pairs
    res["pcie_floor_s_at_55GBps_d2h"] = (8 * (n + 1) + 4 * pairs) / 55e9  # D2H dominates; H2D overlaps on its own engine
    print(f"config {args.config}: {n} points, {pairs} pairs; two calls, pageable: {dt:.3f} s = {pairs / dt / 1e6:.0f} M pairs/s",
          flush=True)
    for label, alloc in (("pageable", lambda k, t: np.empty(k, t)), ("pinned", join.pinned_array)):
        rp, out = alloc(n + 1, np.uint64), alloc(pairs, np.uint32)
        src = pts
        if label == "pinned":
            src = join.pinned_array(2 * n, np.float64).reshape(n, 2)
            src[:] = pts
        s.join_pairs_into(src[:1_000_000], mode, rp, out)
        best = 1e9
        for _ in range(3):
            t0 = time.time()
            total = s.join_pairs_into(src, mode, rp, out)
            best = min(best, time.time() - t0)
        assert total == pairs and np.array_equal(rp, row_ptr) and np.array_equal(out, ids)
        res[f"one_call_{label}_s"] = best
        print(f"  one call, {label} arrays: {best:.3f} s = {pairs / best / 1e6:.0f} M pairs/s "
              f"({best / res['pcie_floor_s_at_55GBps_d2h']:.2f}x the D2H floor)", flush=True)
    d_pts = torch.from_numpy(pts).cuda()
    d_rows = torch.empty(n + 1, dtype=torch.int64, device="cuda")
    d_ids = torch.empty(pairs, dtype=torch.int32, device="cuda")
    torch.cuda.synchronize()
    s.join_pairs_device(d_pts.data_ptr(), n, mode, d_rows.data_ptr(), d_ids.data_ptr(), pairs)
    best = 1e9
    for _ in range(3):
        t0 = time.time()
        total = s.join_pairs_device(d_pts.data_ptr(), n, mode, d_rows.data_ptr(), d_ids.data_ptr(), pairs)
        best = min(best, time.time() - t0)
    assert total == pairs and np.array_equal(d_ids.cpu().numpy().view(np.uint32), ids)
    res["device_resident_s"] = best
    res["device_resident_algorithmic_GBps"] = bytes_moved / best / 1e9
    print(f"  device-resident: {best * 1e3:.2f} ms = {pairs / best / 1e9:.1f} G pairs/s, {n / best / 1e9:.2f} G points/s", flush=True)
    (ROOT / "gpurun_out").mkdir(exist_ok=True)
    (ROOT / "gpurun_out" / f"pairs_probe_cfg{args.config}.json").write_text(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
