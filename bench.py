#!/usr/bin/env python
"""Benchmark of the probe side of the adaptive geospatial join on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

A "step" is one pass of the hot path over one batch of synthetic points:
BASELINE.json configs[1] — 289-polygon jittered-Voronoi tessellation, 100 M
uniform float64 points per GPU, index built at 4 m precision (approx mode,
k_max 48) by the reference's build_index, output = first polygon id per
point + per-polygon counts.  Points shard by range over the GPUs with the
index replicated (weak scaling, no data-path collective; one NCCL all-reduce
sums the per-polygon counts after the timed region).

Prints ONE JSON line (rank 0).  ``value`` = points/s with points resident in
HBM; ``e2e`` = the same join through the host-buffer C-ABI call with H2D/D2H
inside the timed region; ``roofline`` = algorithmic bytes (20 B/point) over
the measured kernel time against the measured HBM copy bandwidth;
``cpu_baseline`` = the reference's own multithreaded CPU join on this box, whose
per-polygon counts must equal the GPU's (``counts_equal_reference``; a mismatch
exits non-zero); ``secondary`` (N = 1) = the other BASELINE configs — configs[2]
exact at full size, configs[3] / configs[4] on their cached density-matched
indexes — each timed the same way and compared per polygon with the reference.

``--gpus N`` with N > 1 and no torchrun environment starts the N ranks itself
(re-exec under ``torch.distributed.run``, NCCL's init log left on); it fails
loudly when the box has fewer than N GPUs or when WORLD_SIZE disagrees with N.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

from paper_1802_09488_b200 import synth  # noqa: E402

BYTES_PER_POINT = 20  # 16 B point read + 4 B polygon-id write
CONFIG = 2


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def workload_config(points_per_gpu: int, n_gpus: int) -> dict:
    return {
        "workload": "configs[1]: 289-polygon jittered-Voronoi tessellation (50-400 vtx), uniform float64 "
                    "points in a 0.45x0.55 deg box, approx join at 4 m precision (k_max 48), "
                    "output first polygon id per point + per-polygon counts",
        "points_per_gpu": points_per_gpu,
        "total_points": points_per_gpu * n_gpus,
        "mode": "approx",
        "sharding": f"points by range over {n_gpus} GPU(s), index replicated, no hot-path collective",
        "l2": "inputs larger than L2 (1.6 GB of points per step, streamed evict-first)",
    }


class ClockSampler:
    """nvidia-smi clocks / throttle reasons DURING the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.lines = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-lms", "100",
                 "-i", str(self.gpu)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._pump, daemon=True).start()
        except OSError:
            self.proc = None

    def _pump(self):
        for line in self.proc.stdout:
            self.lines.append((time.time(), line.strip()))

    def stop(self, t0: float, t1: float) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.15)
        self.proc.terminate()
        sm, mx, reasons = [], [], set()
        for t, line in self.lines:
            if t < t0 - 0.05 or t > t1 + 0.15:
                continue
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
            except ValueError:
                continue
            for name, val in zip(("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"),
                                 f[5:9]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "samples": len(sm), "reasons": sorted(reasons)}


def measured_peak():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            return float(json.loads(p.read_text())["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, burst copy)"
        except Exception:
            pass
    return 6650.0, "fallback (B200_PROFILING.md)"


def kernel_source_hash() -> str:
    """Content hash of the CUDA sources (works on the GPU box, which has no .git)."""
    import hashlib
    h = hashlib.sha256()
    for f in sorted((ROOT / "paper_1802_09488_b200" / "csrc").iterdir()):
        h.update(f.name.encode())
        h.update(f.read_bytes())
    return h.hexdigest()[:16]


def ncu_traffic():
    """profiles/roofline.json: the last ncu capture of K1 (tools/ncu_roofline.py), stamped with the hash of
    the kernel sources it was taken on — stale when they have changed since."""
    p = ROOT / "profiles" / "roofline.json"
    if p.exists():
        try:
            doc = json.loads(p.read_text())
            doc["ncu_stale"] = doc.get("kernel_source_hash") != kernel_source_hash()
            return doc
        except Exception:
            pass
    return {}


def make_points(n: int, rank: int, pinned_alloc=None):
    """Seeded uniform points for this rank's shard (global range [rank*n, (rank+1)*n))."""
    seed = synth.seed_for(CONFIG, 2) + 7919 * rank
    if pinned_alloc is None:
        return synth.uniform_points(n, seed)
    ptr = pinned_alloc(n * 16)
    if not ptr:
        raise RuntimeError("pinned allocation failed")
    buf = (ctypes.c_double * (2 * n)).from_address(ptr)
    arr = np.frombuffer(buf, dtype=np.float64).reshape(n, 2)
    synth.uniform_points(n, seed, out=arr)
    return arr


def bundle_path() -> Path:
    from tools import build_bundles
    t0 = time.time()
    p = build_bundles.ensure_workload_bundle(CONFIG, log=log)  # offline: reference build_index, cached GJX1
    log(f"[bench] index bundle {p.name} ready in {time.time() - t0:.1f}s")
    return p


# --------------------------------------------------------------------------------------
# reference arm / cpu baseline: the reference's own CPU join on the host cores
# --------------------------------------------------------------------------------------
def cpu_join_runner(path: Path, exact: bool = False):
    """Returns (kind, cores, fn(points) -> (seconds, pairs), counts_fn(points) -> ({polygon id: count}, seconds))
    for the CPU arm: the compiled reference when oracle/_ref is present, else the C oracle port.  ``exact``:
    the join mode (the reference's join_count_per_polygon takes it from the bundle, join.cpp:257; an exact join
    over an approx-built bundle — configs[4] — threads join_exact over 64 K-point chunks)."""
    from oracle import build as obuild
    cores = os.cpu_count() or 1
    if obuild.REF_LIB.exists() or obuild.reference_available():
        from oracle import ref
        b = ref.RefBundle.load(path)

        def counts(pts):
            t0 = time.perf_counter()
            m = b.join_exact_count_threads(pts, cores) if exact and b.approx else b.join_count(pts, cores)
            return m, time.perf_counter() - t0
        assert exact or b.approx
        return "reference", cores, (lambda pts: b.time_join_count(pts, cores)), counts
    from tests import golden_util
    ox = golden_util.oracle_index(golden_util.parse_gjx(path.read_bytes()))

    def run(pts):
        t0 = time.perf_counter()
        _, tot = ox.join_count(pts, approx=not exact, threads=cores)
        return time.perf_counter() - t0, tot

    def counts(pts):
        t0 = time.perf_counter()
        m, _ = ox.join_count(pts, approx=not exact, threads=cores)
        return m, time.perf_counter() - t0
    return "port", cores, run, counts


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    path = bundle_path()
    kind, cores, fn, _ = cpu_join_runner(path)
    n = min(args.points, args.ref_points)
    pts = make_points(n, 0)
    for _ in range(args.warmup):
        fn(pts[: max(1, n // 8)])
    times = []
    for _ in range(args.steps):
        secs, _ = fn(pts)
        times.append(secs)
    total = sum(times)
    value = n * args.steps / total
    sample = f"{n} of {args.points} points per step ({kind} join_count_per_polygon, {cores} threads)"
    out = {
        "impl": "reference", "metric": "joined_points_per_sec", "value": value, "unit": "points/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(args.points, args.gpus),
        "cpu_baseline": {"value": value, "unit": "points/s", "cores": cores, "kind": kind, "sample": sample},
        "e2e": {"value": value, "unit": "points/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)


# --------------------------------------------------------------------------------------
# our arm
# --------------------------------------------------------------------------------------
def counts_map(ids, counts) -> dict:
    c = np.asarray(counts).astype(np.uint64)
    return {int(ids[k]): int(c[k]) for k in np.nonzero(c[:len(ids)])[0]}


def time_device_join(torch, sess, d_pts, n, d_counts, d_first, mode, reps, warmup=2):
    """Mean CUDA-event time (ms) of ``reps`` device-resident joins on the session stream."""
    stream = torch.cuda.ExternalStream(sess.stream)

    def step():
        sess.join_count_device(d_pts.data_ptr(), n, d_counts.data_ptr(), mode,
                               d_first_id_ptr=d_first.data_ptr() if d_first is not None else 0)
    torch.cuda.synchronize()
    for _ in range(warmup):
        step()
    sess.sync()
    l0 = sess.launches
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        e0.record()
        for _ in range(reps):
            step()
        e1.record()
    sess.sync()
    return e0.elapsed_time(e1) / reps, (sess.launches - l0) // reps


# (config, density scale of the cached index, points, gj_options fields, label)
SECONDARY = [
    (3, 1.0, 100_000_000, {},
     "configs[2]: exact join, trained index, 289 polygons, 100 M mixture points, ~1 % on edges / vertices (FULL size)"),
    (4, 0.04, 40_000_000, {"dir16_level_max": 17, "hist16": 1, "smem_pad": 78700},
     "configs[3] regime on its density-matched 4 % index (1 600 polygons at 1 m, k_max 56; shared-memory tier capped "
     "at the level the full-size box gets, the 16-bit flushed histogram the full config's 40 000 ids force, shared "
     "memory padded to the 154 KB the full config's 80 KB histogram makes it; the join kernel runs its direct form "
     "with the sparse refinement of the tier's link cells, as at full size); the full 40 000-polygon / 1 B-point "
     "run is tools/fullsize.py 4 (profiles/fullsize_r02_cfg4_direct_form_final.json)"),
    (5, 0.03, 10_000_000, {},
     "configs[4] regime on its density-matched 3 % index (300 overlapping stars, every probe a lookup-table "
     "record, exact); the full 10 000-star / 500 M-point run is tools/fullsize.py 5 (profiles/fullsize_r02_cfg5.json)"),
]


def run_secondary(torch, capi, join, peak, reps=5):
    """The other BASELINE configs, each: device-resident join (first ids + counts) timed with CUDA events, and
    the per-polygon counts of the host-buffer call compared with the reference's CPU join on the same points."""
    from tools import build_bundles
    out = []
    for config, scale, n, opt, label in SECONDARY:
        t_all = time.time()
        name = build_bundles.workload_name(config, scale)
        if not build_bundles.have_bundle(name):
            out.append({"config": config, "workload": label, "unavailable": f"no cached index {name}"})
            continue
        spec = synth.SPECS[config]
        path = build_bundles.bundle_file(name)
        bundle = join.IndexBundle.load(path, device=torch.cuda.current_device(),
                                       options=capi.Options(**opt) if opt else None)
        sess = bundle.session()
        polys = synth.polygons_for(config, scale) if spec.boundary_fraction > 0 else None
        pts = synth.points_for(config, n, polys, scale=scale)
        exact = spec.exact
        mode = capi.GJ_MODE_EXACT if exact else capi.GJ_MODE_APPROX
        d_pts = torch.from_numpy(pts).cuda()
        d_counts = torch.zeros(max(1, len(bundle.ids)), dtype=torch.int64, device="cuda")
        d_first = torch.empty(n, dtype=torch.int32, device="cuda")
        ms, launches = time_device_join(torch, sess, d_pts, n, d_counts, d_first, mode, reps)
        del d_pts, d_first
        # parity: the host-buffer call against the reference's CPU join, polygon by polygon
        st = join.JoinStats()
        counts, _, _ = sess.join_count(pts, mode, stats=st)
        kind, cores, _, cpu_counts = cpu_join_runner(path, exact)
        want, cpu_s = cpu_counts(pts)
        equal = counts_map(bundle.ids, counts) == want
        pairs = int(counts.sum())
        if config == 5:   # 16 B point + 4 B id + the lookup-table record [t, ids, c, ids] every probe reads
            all_refs, _, _ = sess.join_count(pts, capi.GJ_MODE_APPROX)  # approx mode emits every reference
            a_bytes = 20.0 + 4.0 * (2.0 + float(all_refs.sum()) / max(1, n))
            a_note = "16 B point + 4 B first id + 4 B x (2 + references per point) of lookup-table record"
        elif exact:       # + 12 B written and read again per candidate task (point, slot, ordinal)
            a_bytes = 20.0 + 12.0 * st.pip_tests / max(1, n)
            a_note = "16 B point + 4 B first id + 12 B per candidate task (SURVEY.md 8d)"
        else:
            a_bytes = 20.0
            a_note = "16 B point + 4 B first id"
        achieved = a_bytes * n / (ms * 1e-3) / 1e9
        csr = None
        if config == 5:  # configs[4]'s own output form: every covering polygon per point, as CSR, left in HBM
            d_pts = torch.from_numpy(pts).cuda()
            d_rows = torch.empty(n + 1, dtype=torch.int64, device="cuda")
            d_ids = torch.empty(pairs, dtype=torch.int32, device="cuda")
            torch.cuda.synchronize()
            sess.join_pairs_device(d_pts.data_ptr(), n, mode, d_rows.data_ptr(), d_ids.data_ptr(), pairs)  # warm-up
            t0 = time.perf_counter()
            total = sess.join_pairs_device(d_pts.data_ptr(), n, mode, d_rows.data_ptr(), d_ids.data_ptr(), pairs)
            csr_s = time.perf_counter() - t0  # synchronous call: returns when row offsets and ids are in HBM
            m = min(n, 200_000)
            pairs_equal = None
            if kind == "reference":
                from oracle import ref
                rpi, rpid, _ = ref.RefBundle.load(path).join_pairs(pts[:m], exact)
                rows = d_rows[:m + 1].cpu().numpy().astype(np.int64)
                gpi = np.repeat(np.arange(m, dtype=np.uint64), np.diff(rows))
                pairs_equal = bool(np.array_equal(gpi, rpi) and
                                   np.array_equal(d_ids[:rows[-1]].cpu().numpy().view(np.uint32), rpid))
            csr = {"call": "gj_join_pairs_device (points, row offsets and polygon ids in HBM)", "ms": 1e3 * csr_s,
                   "pairs": int(total), "pairs_per_s": total / csr_s,
                   "ordered_pairs_equal_reference_on_prefix": pairs_equal, "prefix": m}
            del d_pts, d_rows, d_ids
        out.append({
            "config": config, "workload": label, "index": name, "mode": "exact" if exact else "approx",
            "points": n, "ms": ms, "points_per_s": n / (ms * 1e-3), "kernel_launches_per_step": launches,
            "pairs_per_point": pairs / n, "pip_tests_per_point": st.pip_tests / n,
            "algorithmic_bytes_per_point": a_bytes, "algorithmic_bytes_note": a_note,
            "achieved_GBps": achieved, "frac": achieved / peak,
            "counts_equal_reference": bool(equal), "csr": csr,
            "cpu_baseline": {"value": n / cpu_s, "unit": "points/s", "cores": cores, "kind": kind,
                             "sample": f"all {n} points, per-polygon counts, {cpu_s:.2f}s"},
            "options": opt, "k1_direct_form": int(bundle.info.k1_direct), "link_records": int(bundle.info.link_records),
            "seconds_total": round(time.time() - t_all, 1),
        })
        log(f"[bench] secondary config {config}: {ms:.3f} ms per {n} points, frac {achieved / peak:.3f}, "
            f"counts equal reference: {equal} ({time.time() - t_all:.1f}s)")
        sess.close()
        bundle.close()
        del pts
    return out


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_1802_09488_b200 import capi, join, sharding

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE is {world}: launch one rank per GPU "
                         f"(python -m torch.distributed.run --nproc-per-node {args.gpus} bench.py --gpus {args.gpus} ...)")
    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device: the GPU path has no CPU fallback")
    if torch.cuda.device_count() <= local:
        raise SystemExit(f"bench.py: rank {rank} wants cuda:{local} but the box has {torch.cuda.device_count()} GPU(s)")
    torch.cuda.set_device(local)
    # under a launcher (torchrun sets RANK / MASTER_*) the NCCL group is created even for one rank, so that the
    # rendezvous, the barriers and the all-reduces below run through the same code whatever N is
    use_dist = world > 1 or ("RANK" in os.environ and "MASTER_PORT" in os.environ)
    if use_dist:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        # NCCL's communicator / transport lines (NVLS, P2P) stay on, on stderr: stdout carries the one JSON line
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        # (NCCL logs to stdout: fd 1 points at stderr while the communicator comes up and runs its first collective)
        sys.stdout.flush()
        saved_stdout = os.dup(1)
        os.dup2(2, 1)
        try:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
            dist.barrier()
            torch.cuda.synchronize()
        finally:
            os.dup2(saved_stdout, 1)
            os.close(saved_stdout)
        log(f"[bench] rank {rank}: NCCL process group of {dist.get_world_size()} rank(s) up")

    def barrier():
        if use_dist:
            dist.barrier()
        torch.cuda.synchronize()

    n = args.points
    path = bundle_path() if rank == 0 else None
    if use_dist:
        dist.barrier()
        from tools import build_bundles
        path = build_bundles.bundle_file(build_bundles.workload_name(CONFIG))
    L = capi.lib()
    bundle = join.IndexBundle.load(path, device=local)  # replicate: every rank loads into its own HBM
    sess = bundle.session()
    info = bundle.info
    log(f"[bench] rank {rank}/{world} on cuda:{local}: index {info.node_count} nodes, {info.device_bytes / 1e6:.0f} MB HBM, "
        f"shared-memory tier level {info.dir16_level} ({info.dir16_width}x{info.dir16_height}), "
        f"L2 tier level {info.dir2_level} ({info.dir2_width}x{info.dir2_height}), dict {info.dir_dict_len}")

    t0 = time.time()
    host_pts = make_points(n, rank, pinned_alloc=L.gj_host_alloc)
    log(f"[bench] rank {rank}: {n} points generated in {time.time() - t0:.1f}s")
    d_pts = torch.empty((n, 2), dtype=torch.float64, device="cuda")
    d_pts.copy_(torch.from_numpy(host_pts))
    n_ids = len(bundle.ids)
    d_counts = torch.zeros(max(1, n_ids), dtype=torch.int64, device="cuda")
    d_first = torch.empty(n, dtype=torch.int32, device="cuda")
    torch.cuda.synchronize()

    stream = torch.cuda.ExternalStream(sess.stream, device=torch.device("cuda", local))

    def step():
        sess.join_count_device(d_pts.data_ptr(), n, d_counts.data_ptr(), capi.GJ_MODE_APPROX,
                               d_first_id_ptr=d_first.data_ptr())

    for _ in range(args.warmup):
        step()
    sess.sync()
    d_counts.zero_()
    barrier()

    sampler = ClockSampler(local)
    if rank == 0:
        sampler.start()
        time.sleep(0.25)
    launches0 = sess.launches
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    barrier()
    wall0 = time.time()
    with torch.cuda.stream(stream):
        ev[0].record()
        for k in range(args.steps):
            step()
            ev[k + 1].record()
    sess.sync()
    barrier()
    wall1 = time.time()
    gpu_launches = sess.launches - launches0
    total_ms = ev[0].elapsed_time(ev[-1])
    step_ms = [ev[k].elapsed_time(ev[k + 1]) for k in range(args.steps)]
    t = torch.tensor([total_ms], dtype=torch.float64, device="cuda")
    if use_dist:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms_max = float(t.item())

    # counts: the only cross-GPU exchange (one NCCL all-reduce), after the timed region
    local_counts = d_counts.clone()
    counts_steps = sharding.allreduce_counts(d_counts.clone())

    # ---- end to end through the host-buffer C-ABI call (pinned host memory) ----
    e2e_steps = max(1, min(args.steps, args.e2e_steps))
    first_host_ptr = L.gj_host_alloc(n * 4)
    first_host = np.frombuffer((ctypes.c_uint32 * n).from_address(first_host_ptr), dtype=np.uint32)
    h_counts = np.zeros(max(1, n_ids), np.uint64)
    ovf_cap = max(1 << 20, n // 16)
    ovf_pt = np.empty(ovf_cap, np.uint64)
    ovf_id = np.empty(ovf_cap, np.uint32)

    def e2e_step():
        ovf = capi.Overflow(ovf_pt.ctypes.data, ovf_id.ctypes.data, ovf_cap, 0)
        bad = ctypes.c_uint64(0)
        rc = L.gj_join_count_host(sess._h, host_pts.ctypes.data, n, rank * n, capi.GJ_MODE_APPROX,
                                  h_counts.ctypes.data, None, first_host_ptr, ctypes.byref(ovf),
                                  ctypes.byref(bad))
        if rc != 0:
            raise RuntimeError(f"gj_join_count_host failed: {rc} {L.gj_last_error().decode()}")
        return int(ovf.count)

    e2e_step()  # warm-up (allocates the staging buffers)
    h_counts[:] = 0
    barrier()
    te0 = time.perf_counter()
    n_ovf = 0
    for _ in range(e2e_steps):
        n_ovf = e2e_step()
    torch.cuda.synchronize()
    te = time.perf_counter() - te0
    tt = torch.tensor([te], dtype=torch.float64, device="cuda")
    if use_dist:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    e2e_s = float(tt.item())

    # ---- self-check: the device-resident and the host-buffer path agree on this rank's shard ----
    per_step_dev = (local_counts.cpu().numpy().astype(np.uint64))[:n_ids]
    if not np.array_equal(per_step_dev, (h_counts[:n_ids] // e2e_steps) * args.steps):
        raise SystemExit(f"bench.py: rank {rank}: device-resident and host-buffer counts differ")
    if not np.array_equal(first_host, d_first.cpu().numpy().view(np.uint32)):
        raise SystemExit(f"bench.py: rank {rank}: device-resident and host-buffer first ids differ")

    if rank != 0:
        dist.barrier()
        dist.destroy_process_group()
        return

    clocks = sampler.stop(wall0, wall1)
    points_total = n * world * args.steps
    value = points_total / (total_ms_max * 1e-3)
    kernel_ms = statistics.mean(step_ms)  # one K1 launch per step in approx mode
    peak, peak_src = measured_peak()
    achieved = BYTES_PER_POINT * n / (kernel_ms * 1e-3) / 1e9
    prof = ncu_traffic()
    roofline = {
        "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
        "traffic": prof.get("traffic_bytes_per_launch"),
        "kernel": "gj::join_kernel<ids=true, stats=false>", "kernel_ms": kernel_ms,
        "algorithmic_bytes_per_point": BYTES_PER_POINT, "points_per_launch": n, "peak_source": peak_src,
        "l2_hit_rate_pct": prof.get("lts__t_sector_hit_rate_pct"),
        "sectors_per_request": prof.get("l1tex_sectors_per_request_global_ld"),
        "ncu_stale": prof.get("ncu_stale", True),
        "ncu": {k: v for k, v in prof.items() if k not in ("traffic_bytes_per_launch", "ncu_stale")} or None,
    }

    # ---- CPU baseline: the reference's multithreaded join on this box's cores, and the parity gate ----
    cpu = None
    counts_equal = None
    if world == 1 and not args.no_cpu_baseline:
        kind, cores, fn, cpu_counts = cpu_join_runner(path)
        m = min(n, args.ref_points)
        fn(host_pts[: m // 8])
        secs, pairs = fn(host_pts[:m])
        cpu = {"value": m / secs, "unit": "points/s", "cores": cores, "kind": kind,
               "sample": f"first {m} of {n} points, one join_count_per_polygon call, {cores} threads, {secs:.2f}s"}
        # the CPU join of the sample must give the GPU's per-polygon counts, polygon by polygon
        want, _ = cpu_counts(host_pts[:m])
        if m == n:
            got = counts_map(bundle.ids, h_counts[:n_ids] // e2e_steps)
        else:
            chk = np.zeros(max(1, n_ids), np.uint64)
            bad = ctypes.c_uint64(0)
            rc = L.gj_join_count_host(sess._h, host_pts.ctypes.data, m, 0, capi.GJ_MODE_APPROX,
                                      chk.ctypes.data, None, None, None, ctypes.byref(bad))
            if rc != 0:
                raise SystemExit(f"bench.py: gj_join_count_host failed: {rc} {L.gj_last_error().decode()}")
            got = counts_map(bundle.ids, chk)
        counts_equal = got == want and sum(want.values()) == int(pairs)
        log(f"[bench] per-polygon counts equal the CPU {kind} join on {m} points: {counts_equal}")

    # ---- the other configs (N = 1): configs[2] exact at full size, configs[3]/[4] on density-matched indexes ----
    secondary = None
    if world == 1 and not args.no_secondary:
        del d_pts, d_first
        L.gj_host_free(first_host_ptr)
        first_host = None
        torch.cuda.empty_cache()
        secondary = run_secondary(torch, capi, join, peak)

    out = {
        "metric": "joined_points_per_sec", "value": value, "unit": "points/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms_max / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": workload_config(n, world), "clocks": clocks,
        "e2e": {"value": n * world * e2e_steps / e2e_s, "unit": "points/s",
                "h2d_bytes_per_step": 16 * n, "d2h_bytes_per_step": 4 * n + 8 * n_ids + 12 * n_ovf,
                "steps": e2e_steps, "ms_per_step": 1e3 * e2e_s / e2e_steps,
                "call": "gj_join_count_host (pinned host points in, first ids + counts + overflow out)"},
        "gpu_launches": int(gpu_launches),
        "roofline": roofline, "cpu_baseline": cpu, "counts_equal_reference": counts_equal,
        "pairs_per_step": int(counts_steps.sum().item()) // args.steps,
        "secondary": secondary,
    }
    print(json.dumps(out), flush=True)
    if use_dist:
        dist.barrier()
        dist.destroy_process_group()
    bad_secondary = [x["config"] for x in (secondary or []) if x.get("counts_equal_reference") is False or
                     (x.get("csr") or {}).get("ordered_pairs_equal_reference_on_prefix") is False]
    if counts_equal is False or bad_secondary:
        raise SystemExit(f"bench.py: GPU per-polygon counts differ from the reference CPU join "
                         f"(headline: {counts_equal}, secondary configs failing: {bad_secondary})")


def launch_ranks(args, argv) -> int:
    """``--gpus N`` outside torchrun: start the N ranks here, one per GPU, over NCCL."""
    import socket

    import torch
    have = torch.cuda.device_count() if torch.cuda.is_available() else 0
    if have < args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but this box has {have} CUDA device(s); "
                         "the GPU path has no CPU fallback and does not oversubscribe devices")
    with socket.socket() as sck:
        sck.bind(("127.0.0.1", 0))
        port = sck.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")  # from process start; the ranks keep whatever NCCL prints off stdout (run_ours)
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(Path(__file__).resolve()), *argv]
    log(f"[bench] starting {args.gpus} ranks: {' '.join(cmd)}")
    return subprocess.call(cmd, env=env)


def main(argv=None):
    argv = list(sys.argv[1:] if argv is None else argv)
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--points", type=int, default=synth.SPECS[CONFIG].n_points, help="points per GPU and step")
    ap.add_argument("--ref-points", type=int, default=100_000_000, help="CPU-arm sample size per step")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-secondary", action="store_true", help="skip the other BASELINE configs (N = 1 only anyway)")
    ap.add_argument("--spawn", action="store_true",
                    help="start the ranks through torch.distributed.run even for --gpus 1 (what --gpus N > 1 does by itself)")
    args = ap.parse_args(argv)
    if args.gpus < 1:
        raise SystemExit("bench.py: --gpus must be >= 1")
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup
    if args.impl == "reference":
        run_reference(args)
    elif (args.gpus > 1 or args.spawn) and "WORLD_SIZE" not in os.environ:
        raise SystemExit(launch_ranks(args, [a for a in argv if a != "--spawn"]))
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
