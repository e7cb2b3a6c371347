"""Builds ``paper_1802_09488_b200/libgeojoin_b200.so`` in-tree with nvcc for
sm_100a.  The library is plain CUDA runtime + C ABI (include/geojoin_b200.h);
it does not link against torch."""
from __future__ import annotations

import os
import shutil
import subprocess
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
LIB = PKG / "libgeojoin_b200.so"
SOURCES = ["gj_index.cu", "gj_api.cu"]


def _headers():
    """Every header the two translation units can include: all of csrc/ and include/."""
    return sorted(p for d in (CSRC, PKG.parent / "include") for p in d.iterdir()
                  if p.suffix in (".cuh", ".hpp", ".h"))


NVCC_FLAGS = [
    "-std=c++17", "-O3", "-lineinfo",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-fmad=false",            # the reference build is FMA-free; results are rounding-sensitive
    "-prec-div=true", "-prec-sqrt=true", "-ftz=false",
    "-Xcompiler", "-fPIC,-fvisibility=hidden,-O2",
    "-shared", "-cudart", "static",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def up_to_date() -> bool:
    if not LIB.exists():
        return False
    t = LIB.stat().st_mtime
    deps = [CSRC / f for f in SOURCES] + _headers() + [Path(__file__)]
    return all(d.stat().st_mtime <= t for d in deps)


def build(force: bool = False, verbose: bool = False, defines=(), out: Path | None = None) -> Path:
    """Default: the product library.  ``defines``/``out`` build tuning variants
    (tools/k1_sweep.py) next to it."""
    target = out or LIB
    if out is None and not force and up_to_date():
        return LIB
    cmd = [nvcc(), *NVCC_FLAGS, *(["-Xptxas", "-v"] if verbose else []), *[f"-D{d}" for d in defines],
           "-o", str(target), *[str(CSRC / f) for f in SOURCES]]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError("nvcc failed:\n" + res.stdout + res.stderr)
    if verbose:
        print(res.stderr)
    return target


if __name__ == "__main__":
    import sys
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
