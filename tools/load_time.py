import sys, time
sys.path.insert(0, '.')
from paper_1802_09488_b200 import join
from tools import build_bundles
for cfg, scale in ((2, 1.0), (3, 1.0), (4, 0.04), (5, 0.03)):
    p = build_bundles.ensure_workload_bundle(cfg, scale)
    for _ in range(2):
        t0 = time.time(); b = join.IndexBundle.load(p, device=0); dt = time.time() - t0
        print(f"config {cfg}: load {dt:.2f} s, {b.info.node_count} nodes, {b.info.device_bytes/1e6:.0f} MB on device", flush=True)
        b.close()
