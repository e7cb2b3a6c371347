"""Tuning harness for K1 (join_kernel): builds variants of the library with -D
switches and times the device-resident join of BASELINE config 2 for each.

    python tools/k1_sweep.py build      # here (CPU): cross-compile all variants
    python tools/k1_sweep.py run [N]    # on the GPU box: time them

Variants whose name starts with ``exp_`` drop work (wrong results) and exist
only to attribute time to phases."""
from __future__ import annotations

import ctypes
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_1802_09488_b200 import _build  # noqa: E402

OUT = ROOT / "tools" / "_variants"
VARIANTS = {
    "base": [],
    "pf0": ["GJ_PF_DIST=0"],
    "pf2": ["GJ_PF_DIST=2"],
    "ppt3": ["GJ_PPT=3"],
    "ppt5": ["GJ_PPT=5"],
    "ppt6": ["GJ_PPT=6"],
    "exp_phase1_only": ["GJ_EXP_PHASE1_ONLY"],
    "exp_no_phase3": ["GJ_EXP_NO_PHASE3"],
    "exp_no_arena": ["GJ_EXP_NO_ARENA"],
    "exp_no_tb": ["GJ_EXP_NO_TB", "GJ_EXP_NO_PHASE3"],
}


def build_all():
    OUT.mkdir(exist_ok=True)
    for name, defs in VARIANTS.items():
        t0 = time.time()
        _build.build(defines=defs, out=OUT / f"lib_{name}.so")
        print(f"built {name} in {time.time() - t0:.1f}s")


def run_all(n_points: int, config: int = 2, scale: float = 1.0, opt: dict | None = None, want_ids: bool = True,
            only=None):
    import numpy as np
    import torch

    from paper_1802_09488_b200 import capi, join, synth
    from tools import build_bundles

    path = build_bundles.bundle_file(build_bundles.workload_name(config, scale))
    pts = synth.points_for(config, n_points, None, scale=scale)
    d_pts = torch.from_numpy(pts).cuda()
    results = {}
    ref_counts = None
    # ground truth for a 20 M prefix from the CPU oracle (test infrastructure)
    from oracle import oracle as _oracle
    from tests import golden_util
    n_chk = min(n_points, 20_000_000)
    ox = golden_util.oracle_index(golden_util.parse_gjx(path.read_bytes()))
    truth_map, _ = ox.join_count(pts[:n_chk], approx=True, threads=16)
    extra = sorted(p.stem[4:] for p in OUT.glob("lib_*.so") if p.stem[4:] not in VARIANTS)  # hand-built A/B libraries
    for name in list(VARIANTS) + extra:
        lib = OUT / f"lib_{name}.so"
        if not lib.exists() or (only and name not in only):
            continue
        capi._LIB = None
        _build.LIB = lib
        capi._build.LIB = lib
        bundle = join.IndexBundle.load(path, device=0, options=capi.Options(**opt) if opt else None)
        sess = bundle.session()
        d_counts = torch.zeros(len(bundle.ids), dtype=torch.int64, device="cuda")
        d_first = torch.empty(n_points, dtype=torch.int32, device="cuda")
        stream = torch.cuda.ExternalStream(sess.stream)

        def step():
            sess.join_count_device(d_pts.data_ptr(), n_points, d_counts.data_ptr(), capi.GJ_MODE_APPROX,
                                   d_first_id_ptr=d_first.data_ptr() if want_ids else 0)
        truth = np.zeros(len(bundle.ids), np.int64)
        for k, v in truth_map.items():
            truth[np.searchsorted(bundle.ids, k)] = v
        sess.join_count_device(d_pts.data_ptr(), n_chk, d_counts.data_ptr(), capi.GJ_MODE_APPROX,
                               d_first_id_ptr=d_first.data_ptr(), sync=True)
        chk = d_counts.cpu().numpy()
        truth_ok = bool(np.array_equal(chk, truth))
        if not truth_ok:
            print(f"   {name}: prefix counts differ from the oracle: sum {chk.sum()} vs {truth.sum()}, "
                  f"{(chk != truth).sum()} slots", flush=True)
        d_counts.zero_()
        torch.cuda.synchronize()  # the session launches on its own stream
        for _ in range(3):
            step()
        sess.sync()
        d_counts.zero_()
        torch.cuda.synchronize()  # the session launches on its own stream
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 10
        with torch.cuda.stream(stream):
            e0.record()
            for _ in range(reps):
                step()
            e1.record()
        sess.sync()
        ms = e0.elapsed_time(e1) / reps
        counts = d_counts.cpu().numpy() // reps
        ok = None
        if not name.startswith("exp_"):
            if ref_counts is None:
                ref_counts = counts
            ok = bool(np.array_equal(counts, ref_counts))
        results[name] = {"ms": ms, "gpts": n_points / ms / 1e6, "counts_ok": ok, "oracle_ok": truth_ok}
        print(f"{name:28s} {ms:8.4f} ms  {n_points / ms / 1e6:8.1f} Gpts/s  counts_ok={ok} oracle_ok={truth_ok}",
              flush=True)
        sess.close()
        bundle.close()
    (ROOT / "gpurun_out").mkdir(exist_ok=True)
    tag = f"cfg{config}" + ("" if want_ids else "_noids")
    (ROOT / "gpurun_out" / f"k1_sweep_{tag}.json").write_text(json.dumps(results, indent=1))


if __name__ == "__main__":
    if sys.argv[1] == "build":
        build_all()
    else:
        import argparse
        ap = argparse.ArgumentParser()
        ap.add_argument("cmd")
        ap.add_argument("points", nargs="?", type=int, default=100_000_000)
        ap.add_argument("--config", type=int, default=2)
        ap.add_argument("--scale", type=float, default=1.0)
        ap.add_argument("--opt", default="", help="comma-separated gj_options fields")
        ap.add_argument("--no-ids", action="store_true")
        ap.add_argument("--only", default="", help="comma-separated variant names")
        a = ap.parse_args()
        run_all(a.points, a.config, a.scale, {k: int(v) for k, v in (kv.split("=") for kv in a.opt.split(",") if kv)},
                not a.no_ids, set(a.only.split(",")) if a.only else None)
