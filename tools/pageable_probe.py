import sys, time
sys.path.insert(0, '.')
import numpy as np
from paper_1802_09488_b200 import capi, join, synth
from tools import build_bundles
bundle = join.IndexBundle.load(build_bundles.ensure_workload_bundle(2), device=0)
s = bundle.session()
pts = synth.points_for(2, 100_000_000, None)
s.join_count(pts[:1_000_000], capi.GJ_MODE_APPROX, want_ids=True)
for want in (False, True):
    for _ in range(2):
        t0 = time.time(); c, f, o = s.join_count(pts, capi.GJ_MODE_APPROX, want_ids=want); dt = time.time() - t0
        print(f"pageable join_count want_ids={want}: {dt*1e3:.1f} ms, {len(pts)/dt/1e9:.2f} G points/s", flush=True)
