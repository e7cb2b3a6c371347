"""BASELINE configs 4 and 5 at (or near) FULL size, in one process on the GPU box.

The indexes of these configs (tens of GB) are too large for the compressed
``.cache/`` route of ``tools/build_bundles.py``, so this tool builds the index
in place with the UNMODIFIED compiled reference (``oracle/_ref``: its
``build_index``, join.cpp:152-235 — offline, outside every timed region), hands
the reference's own flat arrays (``ActProbeView``, act.hpp:108-116) to
``gj_index_create``, and then

  1. times the device-resident join over ALL the config's points (CUDA events on
     the session stream; exact mode: launches of ``--launch`` points, because one
     launch reserves ``points x max candidate refs`` PIP tasks),
  2. times the host-buffer call (``gj_join_count_host``, pageable numpy points),
  3. checks per-polygon counts against the reference's own multithreaded CPU join
     on ``--check`` points, and the ordered pairs on a 200 K prefix.

    python tools/fullsize.py 4 --scale 1.0
    python tools/fullsize.py 5 --scale 1.0 --launch 20000000

The reference is test infrastructure here: it builds the index (offline) and is
the checker; nothing it computes reaches the timed path.
"""
from __future__ import annotations

import argparse
import json
import os
import resource
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_1802_09488_b200 import capi, join, synth  # noqa: E402
from tools import build_bundles  # noqa: E402


def log(*a):
    print("[fullsize]", *a, file=sys.stderr, flush=True)


def rss_gb() -> float:
    return resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 1e6


def run(config: int, scale: float, n_points: int, launch: int, check: int, reps: int, threads: int,
        want_ids: bool, want_stats: bool, host_points: int, pairs_points: int = 0, save_index: str = "",
        load_index: str = "", variants=()):
    import torch
    from oracle import ref

    spec = synth.SPECS[config]
    name = build_bundles.workload_name(config, scale)
    res = {"config": config, "name": name, "scale": scale}

    # ---- index: offline, reference builder ----
    t0 = time.time()
    polys = synth.polygons_for(config, scale)
    res["polygon_gen_s"] = round(time.time() - t0, 1)
    log(f"{len(polys)} polygons generated in {res['polygon_gen_s']}s")
    t0 = time.time()
    if load_index and Path(load_index).exists():
        rb = ref.RefBundle.load(load_index)
        res["index_source"] = "GJX1 file written by an earlier run of this tool (reference build_index + IndexBundle::save)"
    elif build_bundles.have_bundle(name):
        rb = ref.RefBundle.load(build_bundles.bundle_file(name))
        res["index_source"] = "cached GJX1 file (reference build_index + IndexBundle::save), loaded by the reference"
    else:
        cfg = ref.default_config(mode_approx=int(spec.build_approx), precision_m=spec.precision_m, k_max=spec.k_max,
                                 memory_budget_bytes=spec.budget_bytes,
                                 training_point_limit=max(1, spec.training_points))
        rb = ref.RefBundle.build(ref.Polygons(polys.ids, polys.vtx_off, polys.latlng), cfg, None)
        res["index_source"] = "reference build_index in this process"
    res["index_build_s"] = round(time.time() - t0, 1)
    if save_index and not Path(save_index).exists():
        t0 = time.time()
        rb.save(save_index)
        log(f"index saved to {save_index} in {time.time() - t0:.1f}s")
    i = rb.info
    if spec.build_approx and not i.mode_approx:
        raise RuntimeError("approximate build fell back to exact (SURVEY.md trap 11)")
    log(f"index: {res['index_build_s']}s nodes={i.node_count} lut={i.lut_len} mem={i.memory_bytes / 1e9:.2f}GB "
        f"bound={i.achieved_precision_m:.3f}m peak_rss={rss_gb():.1f}GB")
    arena, lut, roots, prefixes, pbits = rb.view()
    rp = rb.polygons()
    t0 = time.time()
    bundle = join.IndexBundle.from_arrays(arena, lut, roots, prefixes, pbits, rb.k_max, rb.approx,
                                          rp.ids, rp.vtx_off, rp.latlng, device=0)
    res["index_create_s"] = round(time.time() - t0, 1)
    info = bundle.info
    sess = bundle.session()
    res.update({
        "index_nodes": int(info.node_count), "index_lut_words": int(i.lut_len), "index_device_gb": info.device_bytes / 1e9,
        "n_polygons": int(info.n_polygons), "k_max": int(rb.k_max), "bound_m": float(i.achieved_precision_m),
        "dir1_level": info.dir_level, "dir2_level": info.dir2_level, "dir16_level": info.dir16_level,
        "link_records": int(info.link_records), "k1_direct": int(info.k1_direct),
    })
    log(f"device index created in {res['index_create_s']}s: {res['index_device_gb']:.2f} GB in HBM, tiers "
        f"{info.dir16_level}/{info.dir_level}/{info.dir2_level}, {info.link_records} sparse refinement records, direct form {info.k1_direct}")

    # ---- points ----
    n = min(n_points, spec.n_points)
    exact = spec.exact
    mode = capi.GJ_MODE_EXACT if exact else capi.GJ_MODE_APPROX
    t0 = time.time()
    pts = np.empty((n, 2), np.float64)
    piece = 50_000_000
    d_pts = torch.empty((n, 2), dtype=torch.float64, device="cuda")
    for a in range(0, n, piece):
        b = min(n, a + piece)
        # one seeded stream per piece: the same bytes whatever the total
        pts[a:b] = synth.points_for(config, b - a, polys if spec.boundary_fraction > 0 else None,
                                    stream=2 + a // piece, scale=scale)
        d_pts[a:b].copy_(torch.from_numpy(pts[a:b]))
    torch.cuda.synchronize()
    res["points"] = n
    res["points_gen_s"] = round(time.time() - t0, 1)
    log(f"{n} points generated and copied in {res['points_gen_s']}s")

    n_ids = len(bundle.ids)
    d_counts = torch.zeros(max(1, n_ids), dtype=torch.int64, device="cuda")
    d_stats = torch.zeros(6, dtype=torch.int64, device="cuda")
    d_first = torch.empty(n if want_ids else 1, dtype=torch.int32, device="cuda")
    stream = torch.cuda.ExternalStream(sess.stream)
    launch = n if (not exact and launch <= 0) else (launch if launch > 0 else 20_000_000)
    flat = d_pts.view(-1)

    def step():
        for a in range(0, n, launch):
            m = min(launch, n - a)
            sess.join_count_device(flat[2 * a:].data_ptr(), m, d_counts.data_ptr(), mode,
                                   d_stats_ptr=d_stats.data_ptr() if want_stats else 0,
                                   d_first_id_ptr=d_first[a:].data_ptr() if want_ids else 0)

    torch.cuda.synchronize()
    step()  # warm-up (also sizes the session's task buffers)
    step()
    sess.sync()
    d_counts.zero_()
    d_stats.zero_()
    torch.cuda.synchronize()
    l0 = sess.launches
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        e0.record()
        for _ in range(reps):
            step()
        e1.record()
    sess.sync()
    ms = e0.elapsed_time(e1) / reps
    counts = (d_counts.cpu().numpy() // reps).astype(np.uint64)
    stats = (d_stats.cpu().numpy() // reps).tolist()
    res.update({
        "mode": "exact" if exact else "approx", "ids": want_ids, "stats_collected": want_stats,
        "points_per_launch": launch, "kernel_launches_per_pass": (sess.launches - l0) // reps,
        "ms_per_pass": ms, "gpoints_per_s": n / ms / 1e6,
        "algorithmic_GBps": (20 if want_ids else 16) * n / ms / 1e6,
        "pairs_per_point": float(counts.sum()) / n,
        "stats": dict(zip(["probes", "pip_tests", "false_hits", "solely_true_hits", "refinement_entered",
                           "candidate_refs"], stats)) if want_stats else None,
    })
    log(f"device-resident join: {ms:.3f} ms per {n} points = {res['gpoints_per_s']:.1f} G points/s")

    def timed(sess_, label, ids, stats_):
        def one():
            for a in range(0, n, launch):
                m = min(launch, n - a)
                sess_.join_count_device(flat[2 * a:].data_ptr(), m, d_counts.data_ptr(), mode,
                                        d_stats_ptr=d_stats.data_ptr() if stats_ else 0,
                                        d_first_id_ptr=d_first[a:].data_ptr() if ids else 0)
        torch.cuda.synchronize()
        one()
        sess_.sync()
        st = torch.cuda.ExternalStream(sess_.stream)
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(st):
            a0.record()
            for _ in range(reps):
                one()
            a1.record()
        sess_.sync()
        t = a0.elapsed_time(a1) / reps
        log(f"variant {label}: {t:.3f} ms")
        return t

    if variants:  # where the time goes: ids / counts, then index variants built with explicit options (gj_options)
        v = {}
        v["ids+counts (no stats)"] = timed(sess, "ids+counts", want_ids, False)
        v["counts only"] = timed(sess, "counts only", False, False)
        for label, kw in variants:
            try:
                b2 = join.IndexBundle.from_arrays(arena, lut, roots, prefixes, pbits, rb.k_max, rb.approx,
                                                  rp.ids, rp.vtx_off, rp.latlng, device=0,
                                                  options=capi.Options(debug_plan=1, **kw))
            except Exception as ex:  # e.g. out of device memory for the second copy
                log(f"variant {label}: {ex}")
                continue
            s2 = b2.session()
            d_counts.zero_()
            d_stats.zero_()
            v[f"{label}: ids+counts+stats"] = timed(s2, label, want_ids, want_stats)
            torch.cuda.synchronize()
            res[f"{label}: counts equal"] = bool(np.array_equal(
                (d_counts.cpu().numpy() // (reps + 1)).astype(np.uint64), counts))
            v[f"{label}: counts only"] = timed(s2, f"{label}, counts only", False, False)
            s2.close()
            b2.close()
        res["variants_ms"] = v

    # ---- host-buffer call (pageable numpy points -> counts) ----
    if host_points:
        hp = min(host_points, n)
        sess.join_count(pts[:min(hp, 4_000_000)], mode)
        t0 = time.time()
        hc, _, _ = sess.join_count(pts[:hp], mode)
        dt = time.time() - t0
        res["host_call"] = {"points": hp, "seconds": dt, "gpoints_per_s": hp / dt / 1e9,
                            "call": "gj_join_count_host, pageable numpy points, counts out"}
        log(f"host-buffer join: {dt:.3f} s per {hp} points")
        if hp == n:
            res["host_counts_equal_device"] = bool(np.array_equal(hc.astype(np.uint64), counts))

    if check <= 0:
        res["peak_rss_gb"] = rss_gb()
        print(json.dumps(res), flush=True)
        sess.close()
        bundle.close()
        return res
    # ---- parity: the reference's own CPU join ----
    m = min(check, n)
    t0 = time.time()
    if exact:
        want = rb.join_exact_count_threads(pts[:m], threads)
    else:
        want = rb.join_count(pts[:m], threads)
    cpu_s = time.time() - t0
    if m == n:
        got = counts
    else:
        d_counts.zero_()
        torch.cuda.synchronize()
        for a in range(0, m, launch):
            sess.join_count_device(flat[2 * a:].data_ptr(), min(launch, m - a), d_counts.data_ptr(), mode)
        sess.sync()
        got = d_counts.cpu().numpy().astype(np.uint64)
    got_map = {int(bundle.ids[k]): int(got[k]) for k in np.nonzero(got)[0]}
    res["reference_counts_equal"] = bool(got_map == want)
    res["reference_check_points"] = m
    res["reference_cpu"] = {"threads": threads, "seconds": cpu_s, "mpoints_per_s": m / cpu_s / 1e6,
                            "call": "join_exact over 64 K chunks on threads" if exact else "join_count_per_polygon"}
    log(f"reference CPU join on {m} points: {cpu_s:.1f}s ({m / cpu_s / 1e6:.1f} M points/s, {threads} threads); "
        f"counts equal: {res['reference_counts_equal']}")
    mp = min(200_000, n)
    row_ptr, ids = sess.join_pairs(pts[:mp], mode)
    pi, pid, rst = rb.join_pairs(pts[:mp], exact)
    gpi = np.repeat(np.arange(mp, dtype=np.uint64), np.diff(row_ptr.astype(np.int64)))
    res["reference_pairs_equal"] = bool(np.array_equal(gpi, pi) and np.array_equal(ids, pid))
    if want_ids and not exact:  # first-id words of the device-resident pass == the host-buffer call's, and a point
        # has a first id exactly when the reference emits a pair for it
        first = d_first[:mp].cpu().numpy().view(np.uint32)
        _, f2, _ = sess.join_count(pts[:mp], mode, want_ids=True)
        has = np.diff(row_ptr.astype(np.int64)) > 0
        res["first_ids_device_equal_host"] = bool(np.array_equal(first, f2))
        res["first_id_present_iff_reference_pair"] = bool(np.array_equal(first != capi.GJ_NO_MATCH, has))
    if pairs_points:  # the materialised-pairs call (CSR through host buffers), the config's own output form
        mq = min(pairs_points, n)
        t0 = time.time()
        rp2, pid2 = sess.join_pairs(pts[:mq], mode)
        dt = time.time() - t0
        t0 = time.time()
        rp2, pid2 = sess.join_pairs(pts[:mq], mode)
        dt2 = time.time() - t0
        res["join_pairs_host"] = {"points": mq, "pairs": int(rp2[-1]), "seconds_first_call": dt, "seconds": dt2,
                                  "mpoints_per_s": mq / dt2 / 1e6, "mpairs_per_s": int(rp2[-1]) / dt2 / 1e6}
        log(f"join_pairs (CSR, host buffers): {dt2:.3f} s per {mq} points, {int(rp2[-1])} pairs")
        del rp2, pid2
    res["peak_rss_gb"] = rss_gb()
    print(json.dumps(res), flush=True)
    sess.close()
    bundle.close()
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", type=int, choices=[4, 5])
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--points", type=int, default=1 << 62)
    ap.add_argument("--launch", type=int, default=0, help="points per launch (exact mode default 20 M; approx: all)")
    ap.add_argument("--check", type=int, default=1 << 62, help="points joined by the reference on the CPU")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--threads", type=int, default=os.cpu_count() or 1)
    ap.add_argument("--no-ids", action="store_true")
    ap.add_argument("--no-stats", action="store_true")
    ap.add_argument("--host-points", type=int, default=1 << 62, help="points of the host-buffer call (0 = skip)")
    ap.add_argument("--pairs", type=int, default=0, help="also time gj_join_pairs_host + gj_pairs_copy on this many points")
    ap.add_argument("--save-index", default="", help="write the built index here (GJX1) for a later --load-index run")
    ap.add_argument("--load-index", default="", help="load the index from this GJX1 file when it exists")
    ap.add_argument("--variants", default="",
                    help="extra timings that attribute the time: ';'-separated index variants, each a comma-separated "
                         "list of gj_options fields, e.g. 'hist16=0;node_pal_max_mb=4096;tier_sub=1'")
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    r = run(a.config, a.scale, a.points, a.launch, a.check, a.reps, a.threads, not a.no_ids, not a.no_stats,
            a.host_points, a.pairs, a.save_index, a.load_index,
            [(v, {k: int(x) for k, x in (kv.split("=") for kv in v.split(","))}) for v in a.variants.split(";") if v])
    if a.out:
        Path(a.out).parent.mkdir(parents=True, exist_ok=True)
        Path(a.out).write_text(json.dumps(r, indent=1))


if __name__ == "__main__":
    main()
