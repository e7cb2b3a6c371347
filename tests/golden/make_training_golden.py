"""Generates tests/golden/training_candidates.npz from the UNMODIFIED reference
(oracle/_ref): for every join fixture, the indices of the fixture points for
which Act::train's `any_candidate` test (src/act.cpp:414-440) is true, computed
with the reference's own Act::probe / for_each_reference on the fixture's own
GJX1 bundle.  Run in the build container only (needs /root/reference):

    python tests/golden/make_training_golden.py
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle import ref  # noqa: E402
from tests import golden_util  # noqa: E402


def main():
    out = {}
    for name in golden_util.names():
        fx = golden_util.load(name)
        if "entries" not in fx:
            continue
        b = ref.RefBundle.load(golden_util.bundle_file(name))
        idx = b.training_candidates(fx["points"])
        # the same reference run pins the count: JoinStats::refinement_entered of the probe pass
        assert len(idx) == int(fx["probe_stats"][4]), (name, len(idx), fx["probe_stats"])
        out[name] = idx.astype(np.uint32)
        print(f"{name}: {len(idx)} of {len(fx['points'])} points hit candidate cells")
    path = golden_util.GOLDEN / "training_candidates.npz"
    np.savez_compressed(path, **out)
    print(f"{path.name}: {path.stat().st_size / 1024:.0f} KB")


if __name__ == "__main__":
    main()
