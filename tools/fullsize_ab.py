"""A/B of library builds on a FULL-SIZE index file left in /tmp by ``tools/fullsize.py --save-index`` (the GPU box
keeps /tmp for a few minutes between calls, which saves the 13-20 minute reference build):

    python tools/fullsize_ab.py /tmp/cfg5_full.gjx 5 --points 100000000 --launch 20000000 --libs base,ld_alloc

The file is read by the product's own GJX1 loader; every library of tools/_variants/ named in --libs (plus "main" =
the shipped one) times the device-resident join over the same seeded points; counts must agree between them."""
from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    import numpy as np
    import torch

    from paper_1802_09488_b200 import _build, capi, join, synth

    ap = argparse.ArgumentParser()
    ap.add_argument("gjx")
    ap.add_argument("config", type=int)
    ap.add_argument("--points", type=int, default=100_000_000)
    ap.add_argument("--launch", type=int, default=20_000_000)
    ap.add_argument("--libs", default="main")
    ap.add_argument("--opt", default="")
    ap.add_argument("--no-ids", action="store_true")
    ap.add_argument("--stats", action="store_true")
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    if not Path(a.gjx).exists():
        print(f"{a.gjx} is gone (fresh box): rebuild with tools/fullsize.py --save-index", flush=True)
        return 3
    spec = synth.SPECS[a.config]
    n = a.points
    pts = synth.points_for(a.config, n, None)
    d_pts = torch.from_numpy(pts).cuda()
    flat = d_pts.view(-1)
    mode = capi.GJ_MODE_EXACT if spec.exact else capi.GJ_MODE_APPROX
    opt = {k: int(v) for k, v in (kv.split("=") for kv in a.opt.split(",") if kv)}
    main_lib = _build.LIB
    out, first_counts = {}, None
    for entry in a.libs.split(","):  # "main", "base", or "main:stage_lut=0+hist16=0" (library : its own options)
        name, _, own = entry.partition(":")
        opt_here = dict(opt, **{k: int(v) for k, v in (kv.split("=") for kv in own.split("+") if kv)})
        lib = main_lib if name == "main" else ROOT / "tools" / "_variants" / f"lib_{name}.so"
        capi._LIB = None
        _build.LIB = lib
        capi._build.LIB = lib
        t0 = time.time()
        bundle = join.IndexBundle.load(a.gjx, device=0, options=capi.Options(**opt_here) if opt_here else None)
        load_s = time.time() - t0
        sess = bundle.session()
        d_counts = torch.zeros(len(bundle.ids), dtype=torch.int64, device="cuda")
        d_stats = torch.zeros(6, dtype=torch.int64, device="cuda")
        d_first = torch.empty(n, dtype=torch.int32, device="cuda")
        stream = torch.cuda.ExternalStream(sess.stream)

        def step():
            for b in range(0, n, a.launch):
                m = min(a.launch, n - b)
                sess.join_count_device(flat[2 * b:].data_ptr(), m, d_counts.data_ptr(), mode,
                                       d_stats_ptr=d_stats.data_ptr() if a.stats else 0,
                                       d_first_id_ptr=0 if a.no_ids else d_first[b:].data_ptr())
        torch.cuda.synchronize()
        step()
        sess.sync()
        d_counts.zero_()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            e0.record()
            for _ in range(a.reps):
                step()
            e1.record()
        sess.sync()
        ms = e0.elapsed_time(e1) / a.reps
        counts = d_counts.cpu().numpy() // a.reps
        if first_counts is None:
            first_counts = counts
        out[entry] = {"ms": ms, "ms_per_20M": ms * 20e6 / n, "gpoints_per_s": n / ms / 1e6, "index_load_s": load_s,
                     "counts_equal_first": bool(np.array_equal(counts, first_counts)), "pairs_per_point": float(counts.sum()) / n}
        print(entry, out[entry], flush=True)
        sess.close()
        bundle.close()
        del d_counts, d_first
        torch.cuda.empty_cache()
    (ROOT / "gpurun_out").mkdir(exist_ok=True)
    (ROOT / "gpurun_out" / f"fullsize_ab_cfg{a.config}.json").write_text(json.dumps(out, indent=1))
    return 0


if __name__ == "__main__":
    sys.exit(main())
