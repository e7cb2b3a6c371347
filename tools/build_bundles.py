"""OFFLINE index build — outside the GPU hot path and outside every timed region.

The index (polygon coverings, super covering, Adaptive Cell Trie, training)
is built by the UNMODIFIED reference library's ``build_index``
(proj/src/join.cpp:152-235) — SURVEY.md §2.1 marks the builder "out of scope,
reference code reused".  This tool calls it through ``oracle/_ref`` (the
compiled reference), saves the result with the reference's own
``IndexBundle::save`` (GJX1 format, join.cpp:316-339) and caches it
zlib-compressed under ``.cache/`` (git-ignored, travels to the GPU box).  The
product then reads the GJX1 file with its own loader (``gj_index_load_file``).
"""
from __future__ import annotations

import os
import sys
import tempfile
import time
import zlib
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

from paper_1802_09488_b200 import synth  # noqa: E402

CACHE = ROOT / ".cache"
# inflated copies live outside the repo so they are not shipped to the GPU box
SCRATCH = Path(tempfile.gettempdir()) / f"gj_bundles_{os.getuid()}"


def bundle_paths(name: str):
    return SCRATCH / f"{name}.gjx", CACHE / f"{name}.gjx.z"


def have_bundle(name: str) -> bool:
    return bundle_paths(name)[1].exists()


def bundle_file(name: str) -> Path:
    """Path of the uncompressed GJX1 file, inflating the cached copy if needed."""
    raw, z = bundle_paths(name)
    if not raw.exists():
        if not z.exists():
            raise FileNotFoundError(f"no cached index {name}; run tools/build_bundles.py")
        SCRATCH.mkdir(exist_ok=True)
        tmp = raw.with_suffix(f".tmp{os.getpid()}")
        tmp.write_bytes(zlib.decompress(z.read_bytes()))
        tmp.rename(raw)
    return raw


def build_bundle(name: str, polys: synth.PolygonSet, spec: synth.WorkloadSpec,
                 training_points=None, log=print) -> Path:
    from oracle import ref  # the reference's build_index, offline

    CACHE.mkdir(exist_ok=True)
    SCRATCH.mkdir(exist_ok=True)
    raw, z = bundle_paths(name)
    cfg = ref.default_config(mode_approx=int(spec.build_approx), precision_m=spec.precision_m,
                             k_max=spec.k_max, memory_budget_bytes=spec.budget_bytes,
                             training_point_limit=max(1, spec.training_points))
    t0 = time.time()
    b = ref.RefBundle.build(ref.Polygons(polys.ids, polys.vtx_off, polys.latlng), cfg, training_points)
    i = b.info
    log(f"[build_bundles] {name}: {time.time() - t0:.1f}s mode={'approx' if i.mode_approx else 'exact'} "
        f"achieved={i.precision_achieved} bound={i.achieved_precision_m:.3f}m nodes={i.node_count} "
        f"lut={i.lut_len} mem={i.memory_bytes / 1e6:.1f}MB")
    if spec.build_approx and not i.mode_approx:
        raise RuntimeError(f"{name}: approximate build fell back to exact (SURVEY.md trap 11)")
    b.save(raw)
    z.write_bytes(zlib.compress(raw.read_bytes(), 6))
    return raw


def workload_name(config: int, scale: float = 1.0) -> str:
    spec = synth.SPECS[config]
    return spec.name if scale == 1.0 else f"{spec.name}_s{scale:g}"


def ensure_workload_bundle(config: int, scale: float = 1.0, log=print) -> Path:
    """GJX1 file for a BASELINE config (cached)."""
    name = workload_name(config, scale)
    if have_bundle(name):
        return bundle_file(name)
    spec = synth.SPECS[config]
    polys = synth.polygons_for(config, scale)
    training = None
    if spec.training_points:
        training = synth.points_for(config, int(spec.training_points * min(1.0, scale * 4)), stream=1, scale=scale)
    return build_bundle(name, polys, spec, training, log)


if __name__ == "__main__":
    configs = [int(a) for a in sys.argv[1:]] or [2]
    for c in configs:
        print(ensure_workload_bundle(c))
