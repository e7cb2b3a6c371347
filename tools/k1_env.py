"""Time K1 (device-resident join of BASELINE config 2) under explicit index
options (gj_options), e.g.
    python tools/k1_env.py "" dir16_max_entries=34000 node_pal_max_mb=0,smem_pad=30000

Each argument is a comma-separated list of field=value settings the index is
loaded with; results are checked against each other (counts, first ids)."""
from __future__ import annotations

import json
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    import numpy as np
    import torch

    from paper_1802_09488_b200 import capi, join, synth
    from tools import build_bundles

    n = int(os.environ.get("K1_POINTS", 100_000_000))
    path = build_bundles.ensure_workload_bundle(2, 1.0)
    pts = synth.uniform_points(n, synth.seed_for(2, 2))
    d_pts = torch.from_numpy(pts).cuda()
    first = None
    out = {}
    for arg in sys.argv[1:] or [""]:
        sets = {k: int(v) for k, v in (kv.split("=", 1) for kv in arg.split(",") if kv)}
        bundle = join.IndexBundle.load(path, device=0, options=capi.Options(**sets))
        sess = bundle.session()
        d_counts = torch.zeros(len(bundle.ids), dtype=torch.int64, device="cuda")
        d_first = torch.empty(n, dtype=torch.int32, device="cuda")
        stream = torch.cuda.ExternalStream(sess.stream)
        step = lambda: sess.join_count_device(d_pts.data_ptr(), n, d_counts.data_ptr(), capi.GJ_MODE_APPROX,
                                              d_first_id_ptr=d_first.data_ptr())
        for _ in range(5):
            step()
        sess.sync()
        d_counts.zero_()
        torch.cuda.synchronize()  # the session launches on its own stream
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            e0.record()
            for _ in range(20):
                step()
            e1.record()
        sess.sync()
        ms = e0.elapsed_time(e1) / 20
        counts = d_counts.cpu().numpy() // 20
        ids = d_first.cpu().numpy()
        if first is None:
            first = (counts, ids)
        same = bool(np.array_equal(counts, first[0]) and np.array_equal(ids, first[1]))
        out[arg] = {"ms": ms, "dir16_level": bundle.info.dir16_level, "same_as_first": same}
        print(arg or "(default)", out[arg], flush=True)
        sess.close()
        bundle.close()
    (ROOT / "gpurun_out").mkdir(exist_ok=True)
    (ROOT / "gpurun_out" / "k1_env.json").write_text(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
