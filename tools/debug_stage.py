import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import numpy as np, torch
from paper_1802_09488_b200 import _build, capi, join, synth
from tools import build_bundles
path = build_bundles.bundle_file(build_bundles.workload_name(2))
n = 20_000_000
pts = synth.uniform_points(n, synth.seed_for(2, 2))
d_pts = torch.from_numpy(pts).cuda()
res = {}
for name in ("nostage", "base"):
    lib = ROOT / "tools" / "_variants" / f"lib_{name}.so"
    capi._LIB = None; _build.LIB = lib; capi._build.LIB = lib
    b = join.IndexBundle.load(path, device=0); s = b.session()
    d_counts = torch.zeros(len(b.ids), dtype=torch.int64, device="cuda")
    outs = []
    for rep in range(3):
        d_first = torch.full((n,), -7, dtype=torch.int32, device="cuda")
        s.join_count_device(d_pts.data_ptr(), n, d_counts.data_ptr(), capi.GJ_MODE_APPROX, d_first_id_ptr=d_first.data_ptr(), sync=True)
        outs.append(d_first.cpu().numpy())
    res[name] = outs
    s.close(); b.close()
ref = res["nostage"][0]
print("nostage self-consistent:", all(np.array_equal(ref, o) for o in res["nostage"]))
for k, o in enumerate(res["base"]):
    bad = np.nonzero(o != ref)[0]
    print(f"base run {k}: {len(bad)} differing points")
    if len(bad):
        print("  idx[:20]", bad[:20])
        print("  tile", (bad // 4096)[:20], " tile%148", ((bad // 4096) % 148)[:20])
        print("  in-tile offset", (bad % 4096)[:20])
        print("  warp", ((bad % 4096) // 128)[:20], "slot j", (((bad % 4096) % 128) // 32)[:20], "lane", (bad % 32)[:20])
        print("  values got", o[bad[:10]], "want", ref[bad[:10]])
        # does the wrong value equal the right answer of the point one 'ring period' earlier?
        period = 148 * 4096
        prev = bad - period
        ok = prev >= 0
        print("  equals answer of same slot in previous tile of this CTA:", np.mean(o[bad[ok]] == ref[prev[ok]]))
