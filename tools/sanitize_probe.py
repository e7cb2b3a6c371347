"""A small, complete pass over the kernels for compute-sanitizer (tools/sanitize.sh): one fixture, one set of
gj_options; entries, the streaming join (both modes, first ids + overflow + stats, host-buffer and device-resident),
the CSR calls and a two-replica group — each checked against the fixture, so a tool run that "passes" also computed
the right thing.

    compute-sanitizer --tool racecheck python tools/sanitize_probe.py cfg5_stars_scaled stage_lut=1,hist16=1
"""
from __future__ import annotations

import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    import numpy as np
    import torch

    from paper_1802_09488_b200 import capi, join
    from tests import golden_util

    name = sys.argv[1] if len(sys.argv) > 1 else "cfg3_tess16_exact_trained"
    opt = {k: int(v) for k, v in (kv.split("=") for kv in (sys.argv[2] if len(sys.argv) > 2 else "").split(",") if kv)}
    fx = golden_util.load(name)
    pts = np.ascontiguousarray(fx["points"])
    n = len(pts)
    b = join.IndexBundle.load(golden_util.bundle_file(name), device=0, options=capi.Options(**opt))
    s = b.session()
    assert np.array_equal(s.probe_points(pts), fx["entries"])
    d_pts = torch.from_numpy(pts).cuda()
    for kind, mode in (("exact", capi.GJ_MODE_EXACT), ("approx", capi.GJ_MODE_APPROX)):
        epi, epid = golden_util.pairs_of(fx, kind)
        want = np.bincount(np.searchsorted(b.ids, epid), minlength=len(b.ids)).astype(np.uint64)
        st = join.JoinStats()
        counts, first, (ovf_pt, ovf_id) = s.join_count(pts, mode, stats=st, want_ids=True)
        assert np.array_equal(counts, want) and st.as_tuple() == tuple(int(v) for v in fx[f"{kind}_stats"])
        c2, _, _ = s.join_count(pts, mode)
        assert np.array_equal(c2, want)
        d_counts = torch.zeros(max(1, len(b.ids)), dtype=torch.int64, device="cuda")
        d_first = torch.empty(n, dtype=torch.int32, device="cuda")
        torch.cuda.synchronize()
        s.join_count_device(d_pts.data_ptr(), n, d_counts.data_ptr(), mode, d_first_id_ptr=d_first.data_ptr(), sync=True)
        assert np.array_equal(d_counts.cpu().numpy()[:len(want)].astype(np.uint64), want)
        row_ptr, ids = s.join_pairs(pts, mode)
        assert np.array_equal(ids, epid)
        rp = np.empty(n + 1, np.uint64)
        out = np.empty(len(epid), np.uint32)
        assert s.join_pairs_into(pts, mode, rp, out) == len(epid) and np.array_equal(out, epid) and np.array_equal(rp, row_ptr)
    fleet = join.IndexGroup.load(golden_util.bundle_file(name), [0, 0], options=capi.Options(**opt))
    want = {int(k): int(v) for k, v in zip(fx["count_ids"], fx["count_values"])}
    assert join.join_count_per_polygon(fleet, pts, 2) == want
    fleet.close()
    print(f"sanitize probe ok: {name} {opt} {n} points, {s.launches} launches")
    s.close()
    b.close()


if __name__ == "__main__":
    main()
