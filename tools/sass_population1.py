"""SASS of K1's population-1 loop body (one full tile of a warp: 4 points per lane) from the built library:

    python tools/sass_population1.py > profiles/sass_rNN_k1_population1.txt

Instantiation join_kernel<kIds=true, kStats=false, kDense=true, kLate=false, kStage=false, kDirect=false> — the kernel bench.py times.  The
excerpt runs from the L2 prefetch + the four 16-byte evict-first point loads to the fourth queue append, i.e. the
straight-line code every point passes through (grid coordinates in two DFMAs, 16-bit tier lookup, histogram
increment, first-id store, ballot/popc queue append); what follows it in the kernel (queue drains, populations 2
and 3) runs only for the points this code leaves open."""
from __future__ import annotations

import re
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
LIB = ROOT / "paper_1802_09488_b200" / "libgeojoin_b200.so"
KERNEL = "_ZN2gj11join_kernelILb1ELb0ELb1ELb0ELb0ELb0EEEvNS_8DevIndexENS_10JoinParamsE"


def main():
    sass = subprocess.run(["cuobjdump", "-sass", str(LIB)], capture_output=True, text=True, check=True).stdout.splitlines()
    start = next(i for i, l in enumerate(sass) if "Function : " + KERNEL in l)
    end = next((i for i in range(start + 1, len(sass)) if "Function : " in sass[i]), len(sass))
    body = [l for l in sass[start:end] if re.search(r"/\*[0-9a-f]{4,}\*/\s+\S", l) and not re.match(r"\s+/\* 0x", l)]
    ins = [re.sub(r"\s*/\* 0x[0-9a-f]+ \*/\s*$", "", l).rstrip() for l in body]
    first_load = next(i for i, l in enumerate(ins) if "LDG.E.EF.128" in l)
    begin = max(i for i in range(first_load) if "CCTL.E.PF2" in ins[i])
    appends = [i for i in range(first_load, len(ins)) if "STS.64" in ins[i]][:4]
    stop = appends[-1] + 1
    excerpt = ins[begin:stop]
    n = len(excerpt)
    print(f"# {KERNEL}")
    print(f"# whole kernel: {len(ins)} SASS instructions; population 1 (below): {n} instructions per lane for 4 points "
          f"= {n / 4:.1f} per point")
    ops = {}
    for l in excerpt:
        m = re.search(r"\*/\s+(?:@!?U?P\d\s+)?([A-Z0-9_.]+)", l)
        if m:
            op = m.group(1).split(".")[0]
            ops[op] = ops.get(op, 0) + 1
    print("# opcode mix: " + ", ".join(f"{k} {v}" for k, v in sorted(ops.items(), key=lambda kv: -kv[1])))
    print("\n".join(excerpt))


if __name__ == "__main__":
    sys.exit(main())
