"""TEST INFRASTRUCTURE — builds the two CPU checkers.  Not product code.

1. ``oracle/libgeojoin_oracle.so``  — the plain-C restatement of the hot path
   (``oracle/geojoin_oracle.c``).  Always buildable (gcc only).
2. ``oracle/_ref/libgeojoin_ref.so`` — the UNMODIFIED reference library,
   compiled from the sources where they lie under ``/root/reference/proj/src``
   (nothing is copied into this repo) plus ``oracle/ref_shim.cpp`` (our C ABI
   over it).  Only possible where ``/root/reference`` exists (the build
   container); the built ``.so`` is git-ignored but travels to the GPU box.

Reference flags: the reference's CMake Release build is ``-O3`` with no
``-march`` (proj/CMakeLists.txt:8-10), i.e. FMA-free; only
``act_probe_avx2.cpp`` gets ``-mavx2`` (proj/src/CMakeLists.txt:19-25).  We
add ``-ffp-contract=off`` so the guarantee does not depend on the host's
default ``-march``.  The reference's own build system (cmake + vendor/) is NOT
run: ``geojson.cpp``, the CLI and the doctest suites need git-ignored
third-party headers and are not on the hot path.
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

HERE = Path(__file__).resolve().parent
REF_ROOT = Path(os.environ.get("GEOJOIN_REFERENCE_ROOT", "/root/reference")) / "proj"
REF_DIR = HERE / "_ref"
REF_LIB = REF_DIR / "libgeojoin_ref.so"
ORACLE_LIB = HERE / "libgeojoin_oracle.so"

REF_TUS = [
    "cell_id.cpp",
    "geometry.cpp",
    "super_covering.cpp",
    "act.cpp",
    "act_probe_scalar.cpp",
    "act_probe_avx2.cpp",
    "join.cpp",
    "csv.cpp",
]
REF_FLAGS = ["-std=gnu++20", "-O3", "-fPIC", "-ffp-contract=off", "-DNDEBUG"]


def _run(cmd: list[str]) -> None:
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"command failed: {' '.join(cmd)}\n{res.stdout}\n{res.stderr}")


def _newer(target: Path, sources: list[Path]) -> bool:
    if not target.exists():
        return False
    t = target.stat().st_mtime
    return all(s.exists() and s.stat().st_mtime <= t for s in sources)


def build_oracle(force: bool = False) -> Path:
    src = [HERE / "geojoin_oracle.c", HERE / "geojoin_oracle.h"]
    if not force and _newer(ORACLE_LIB, src):
        return ORACLE_LIB
    _run(["gcc", "-std=c11", "-O2", "-fPIC", "-shared", "-ffp-contract=off",
          "-Wall", "-Wextra", "-pthread", "-o", str(ORACLE_LIB), str(src[0]), "-lm"])
    return ORACLE_LIB


def reference_available() -> bool:
    return (REF_ROOT / "src" / "join.cpp").exists()


def build_ref(force: bool = False) -> Path | None:
    """Compile the reference where it lies; returns None when it is absent."""
    if not reference_available():
        return REF_LIB if REF_LIB.exists() else None
    srcs = [REF_ROOT / "src" / f for f in REF_TUS] + [HERE / "ref_shim.cpp"]
    if not force and _newer(REF_LIB, srcs):
        return REF_LIB
    REF_DIR.mkdir(exist_ok=True)
    inc = ["-I", str(REF_ROOT / "include")]

    def compile_one(src: Path) -> Path:
        obj = REF_DIR / (src.stem + ".o")
        flags = list(REF_FLAGS)
        if src.name == "act_probe_avx2.cpp":
            flags.append("-mavx2")
        _run(["g++", *flags, *inc, "-c", str(src), "-o", str(obj)])
        return obj

    with ThreadPoolExecutor(max_workers=8) as ex:
        objs = list(ex.map(compile_one, srcs))
    _run(["g++", "-shared", "-o", str(REF_LIB), *map(str, objs), "-lpthread"])
    for o in objs:
        o.unlink()
    return REF_LIB


def build_dropin_test(force: bool = False) -> Path | None:
    """tests/cpp/dropin_test: the reference's headers + library and
    include/geojoin_gpu.hpp + libgeojoin_b200.so in one C++ program."""
    root = HERE.parent
    src = root / "tests" / "cpp" / "dropin_test.cpp"
    out = root / "tests" / "cpp" / "dropin_test"
    gpu_lib = root / "paper_1802_09488_b200" / "libgeojoin_b200.so"
    if not reference_available() or not gpu_lib.exists() or build_ref() is None:
        return out if out.exists() else None
    deps = [src, root / "include" / "geojoin_gpu.hpp", root / "include" / "geojoin_b200.h", REF_LIB, gpu_lib]
    if not force and _newer(out, deps):
        return out
    _run(["g++", "-std=gnu++20", "-O2", "-ffp-contract=off", "-I", str(REF_ROOT / "include"),
          "-I", str(root / "include"), str(src), "-o", str(out),
          "-L", str(REF_DIR), "-lgeojoin_ref", "-L", str(gpu_lib.parent), "-lgeojoin_b200",
          "-Wl,-rpath,$ORIGIN/../../oracle/_ref:$ORIGIN/../../paper_1802_09488_b200", "-lpthread"])
    return out


if __name__ == "__main__":
    force = "--force" in sys.argv
    print("oracle:", build_oracle(force))
    print("ref   :", build_ref(force))
    print("dropin:", build_dropin_test(force))
