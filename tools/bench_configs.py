"""Secondary measurements: the device-resident join on the other BASELINE
configs (bench.py is the headline, config 2).  For each config: load the
cached reference-built index, generate the seeded points, time the join in the
config's mode (first id per point + per-polygon counts + JoinStats) with CUDA
events, and check a prefix against the CPU oracle (test infrastructure).

    python tools/bench_configs.py [configs...] [--points N]
"""
from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_1802_09488_b200 import capi, join, synth  # noqa: E402
from tools import build_bundles  # noqa: E402


def run_config(config: int, n_points: int, scale: float, reps: int, check: int, want_ids: bool = True,
               pairs_points: int = 0, want_stats: bool = True, force_mode: str | None = None, options=None):
    import torch

    spec = synth.SPECS[config]
    name = build_bundles.workload_name(config, scale)
    path = build_bundles.ensure_workload_bundle(config, scale, log=lambda *a: print(*a, file=sys.stderr))
    bundle = join.IndexBundle.load(path, device=0, options=options)
    sess = bundle.session()
    info = bundle.info
    polys = synth.polygons_for(config, scale) if spec.boundary_fraction > 0 else None
    n = min(n_points, spec.n_points)
    t0 = time.time()
    pts = synth.points_for(config, n, polys, scale=scale)
    gen_s = time.time() - t0
    exact = spec.exact if force_mode is None else force_mode == "exact"
    mode = capi.GJ_MODE_EXACT if exact else capi.GJ_MODE_APPROX

    d_pts = torch.from_numpy(pts).cuda()
    n_ids = len(bundle.ids)
    d_counts = torch.zeros(max(1, n_ids), dtype=torch.int64, device="cuda")
    d_stats = torch.zeros(6, dtype=torch.int64, device="cuda")
    d_first = torch.empty(n, dtype=torch.int32, device="cuda")
    stream = torch.cuda.ExternalStream(sess.stream)

    def step():
        sess.join_count_device(d_pts.data_ptr(), n, d_counts.data_ptr(), mode,
                               d_stats_ptr=d_stats.data_ptr() if want_stats else 0,
                               d_first_id_ptr=d_first.data_ptr() if want_ids else 0)

    for _ in range(3):
        step()
    sess.sync()
    d_counts.zero_()
    d_stats.zero_()
    torch.cuda.synchronize()
    launches0 = sess.launches
    launches1 = None
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        e0.record()
        for _ in range(reps):
            step()
        e1.record()
    sess.sync()
    launches1 = sess.launches
    ms = e0.elapsed_time(e1) / reps
    stats = (d_stats.cpu().numpy() // reps).tolist()
    counts = d_counts.cpu().numpy() // reps

    # parity on a prefix against the CPU oracle
    from tests import golden_util
    m = min(check, n)
    ox = golden_util.oracle_index(golden_util.parse_gjx(Path(path).read_bytes()))
    t0 = time.time()
    want, total = ox.join_count(pts[:m], approx=not exact, threads=16)
    cpu_s = time.time() - t0
    got, _, _ = sess.join_count(pts[:m], mode)
    got_map = {int(bundle.ids[k]): int(got[k]) for k in np.nonzero(got)[0]}
    ok = got_map == want
    # ordered pairs on a smaller prefix
    mp = min(200_000, n)
    row_ptr, ids = sess.join_pairs(pts[:mp], mode)
    pi, pid, ost, _ = ox.join(pts[:mp], approx=not exact)
    gpi = np.repeat(np.arange(mp, dtype=np.uint64), np.diff(row_ptr.astype(np.int64)))
    ok_pairs = bool(np.array_equal(gpi, pi) and np.array_equal(ids, pid))

    pairs_res = None
    if pairs_points:  # throughput of the materialised-pairs call (CSR), host buffers in and out
        mq = min(pairs_points, n)
        sess.join_pairs(pts[:min(mq, 1_000_000)], mode)
        t0 = time.time()
        rp, pid2 = sess.join_pairs(pts[:mq], mode)
        dt = time.time() - t0
        pairs_res = {"points": mq, "pairs": int(rp[-1]), "seconds": dt, "mpoints_per_s": mq / dt / 1e6,
                     "mpairs_per_s": int(rp[-1]) / dt / 1e6}
    res = {
        "config": config, "name": name, "mode": "exact" if exact else "approx", "points": n,
        "ms": ms, "gpoints_per_s": n / ms / 1e6, "launches_per_step": (launches1 - launches0) // reps, "ids": want_ids, "stats_collected": want_stats,
        "index_nodes": int(info.node_count), "index_mb": info.device_bytes / 1e6, "n_polygons": int(info.n_polygons),
        "dir1_level": info.dir_level, "dir2_level": info.dir2_level, "dir16_level": info.dir16_level,
        "link_records": int(info.link_records), "k1_direct": int(info.k1_direct), "dir16_cells": [info.dir16_width, info.dir16_height], "dir2_cells": [info.dir2_width, info.dir2_height],
        "stats": dict(zip(["probes", "pip_tests", "false_hits", "solely_true_hits", "refinement_entered",
                           "candidate_refs"], stats)),
        "pairs_per_point": float(counts.sum()) / n,
        "oracle_counts_equal": bool(ok), "oracle_pairs_equal": ok_pairs, "oracle_prefix": m,
        "cpu_oracle_prefix_mpts_per_s_16thr": m / cpu_s / 1e6, "gen_s": gen_s,
        "join_pairs_host": pairs_res,
    }
    print(json.dumps(res), flush=True)
    sess.close()
    bundle.close()
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="*", type=int, default=[1, 2, 3])
    ap.add_argument("--points", type=int, default=100_000_000)
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--check", type=int, default=5_000_000)
    ap.add_argument("--no-ids", action="store_true", help="counts + stats only (no first id per point)")
    ap.add_argument("--no-stats", action="store_true", help="do not collect JoinStats")
    ap.add_argument("--mode", choices=["approx", "exact"], default=None, help="override the config's join mode")
    ap.add_argument("--dir16-level", type=int, default=0,
                    help="cap the shared-memory tier at this grid level (a stand-in over a scaled-down box otherwise "
                         "gets a finer first tier than the full-size box would: level 17 for the BASELINE box)")
    ap.add_argument("--pairs", type=int, default=0, help="also time gj_join_pairs_host on this many points")
    ap.add_argument("--opt", default="", help="comma-separated gj_options fields, e.g. hist_rep_cap=0,hist16=0")
    args = ap.parse_args()
    kw = {k: int(v) for k, v in (kv.split("=", 1) for kv in args.opt.split(",") if kv)}
    if args.dir16_level:
        kw["dir16_level_max"] = args.dir16_level
    options = capi.Options(**kw) if kw else None
    out = [run_config(c, args.points, args.scale, args.reps, args.check, not args.no_ids, args.pairs, not args.no_stats,
                      args.mode, options) for c in args.configs]
    (ROOT / "gpurun_out").mkdir(exist_ok=True)
    (ROOT / "gpurun_out" / "bench_configs.json").write_text(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
