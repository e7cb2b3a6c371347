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
``cpu_baseline`` = the reference's own multithreaded CPU join on this box.
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


def ncu_traffic():
    p = ROOT / "profiles" / "roofline.json"
    if p.exists():
        try:
            return json.loads(p.read_text())
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
def cpu_join_runner(path: Path):
    """Returns (kind, cores, fn(points) -> (seconds, pairs)) for the CPU arm:
    the compiled reference when oracle/_ref is present, else the C oracle port."""
    from oracle import build as obuild
    cores = os.cpu_count() or 1
    if obuild.REF_LIB.exists() or obuild.reference_available():
        from oracle import ref
        b = ref.RefBundle.load(path)
        return "reference", cores, lambda pts: b.time_join_count(pts, cores)
    from oracle import oracle
    from tests import golden_util
    ox = golden_util.oracle_index(golden_util.parse_gjx(path.read_bytes()))

    def run(pts):
        t0 = time.perf_counter()
        _, tot = ox.join_count(pts, approx=True, threads=cores)
        return time.perf_counter() - t0, tot
    return "port", cores, run


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    path = bundle_path()
    kind, cores, fn = cpu_join_runner(path)
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
def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_1802_09488_b200 import capi, join

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if not torch.cuda.is_available():
        raise RuntimeError("bench.py needs a CUDA device: the GPU path has no CPU fallback")
    torch.cuda.set_device(local)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    n = args.points
    path = bundle_path() if rank == 0 else None
    if world > 1:
        dist.barrier()
        from tools import build_bundles
        path = build_bundles.bundle_file(build_bundles.workload_name(CONFIG))
    L = capi.lib()
    bundle = join.IndexBundle.load(path, device=local)  # replicate: every rank loads into its own HBM
    sess = bundle.session()
    info = bundle.info
    log(f"[bench] rank {rank}: index {info.node_count} nodes, {info.device_bytes / 1e6:.0f} MB HBM, "
        f"directory tier 1 level {info.dir_level} ({info.dir_width}x{info.dir_height}, shared memory), "
        f"tier 2 level {info.dir2_level} ({info.dir2_width}x{info.dir2_height}, L2), dict {info.dir_dict_len}")

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
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms_max = float(t.item())

    # counts: the only cross-GPU exchange, after the timed region
    counts_steps = d_counts.clone()
    if world > 1:
        dist.all_reduce(counts_steps, op=dist.ReduceOp.SUM)

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
    if world > 1:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    e2e_s = float(tt.item())

    # ---- self-check: device-resident, e2e and a CPU-oracle sample agree ----
    per_step_dev = (d_counts.cpu().numpy().astype(np.uint64))[:n_ids]
    assert np.array_equal(per_step_dev, (h_counts[:n_ids] // e2e_steps) * args.steps), "device vs e2e counts differ"
    assert np.array_equal(first_host, d_first.cpu().numpy().view(np.uint32)), "device vs e2e ids differ"

    if rank != 0:
        if world > 1:
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
        "ncu": {k: v for k, v in prof.items() if k != "traffic_bytes_per_launch"} or None,
    }

    # ---- CPU baseline: the reference's multithreaded join on this box's cores ----
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        try:
            kind, cores, fn = cpu_join_runner(path)
            m = min(n, args.ref_points)
            fn(host_pts[: m // 8])
            secs, pairs = fn(host_pts[:m])
            cpu = {"value": m / secs, "unit": "points/s", "cores": cores, "kind": kind,
                   "sample": f"first {m} of {n} points, one join_count_per_polygon call, {cores} threads, {secs:.2f}s"}
            # the CPU join of the sample must give the GPU's counts
            chk = np.zeros(max(1, n_ids), np.uint64)
            bad = ctypes.c_uint64(0)
            rc = L.gj_join_count_host(sess._h, host_pts.ctypes.data, m, 0, capi.GJ_MODE_APPROX,
                                      chk.ctypes.data, None, None, None, ctypes.byref(bad))
            assert rc == 0 and int(chk.sum()) == int(pairs), "GPU vs CPU pair totals differ on the sample"
        except Exception as exc:  # the baseline is reported, never required
            log(f"[bench] cpu baseline unavailable: {exc}")

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
        "roofline": roofline, "cpu_baseline": cpu,
        "pairs_per_step": int(counts_steps.sum().item()) // args.steps,
    }
    print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--points", type=int, default=synth.SPECS[CONFIG].n_points, help="points per GPU and step")
    ap.add_argument("--ref-points", type=int, default=100_000_000, help="CPU-arm sample size per step")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
