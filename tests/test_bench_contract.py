"""The reference arm of bench.py runs on CPU: check its one-line JSON contract
here (keys, units, the cpu_baseline / e2e objects), on a small sample."""
import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


def test_reference_arm_prints_one_contract_line():
    from tools import build_bundles
    if not build_bundles.have_bundle(build_bundles.workload_name(2)):
        pytest.skip("no cached config-2 index (tools/build_bundles.py needs the reference)")
    res = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--gpus", "1", "--steps", "2",
                          "--warmup", "1", "--points", "400000", "--ref-points", "400000"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert res.returncode == 0, res.stderr[-2000:]
    lines = [l for l in res.stdout.splitlines() if l.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["metric"] == "joined_points_per_sec" and d["unit"] == "points/s"
    assert d["n_gpus"] == 1 and d["steps"] == 2 and d["warmup"] == 1 and d["higher_is_better"] is True
    assert d["value"] > 0 and d["ms_per_step"] > 0 and d["vs_baseline"] is None and d["scaling"] == "weak"
    assert d["dtype"] == "f64" and d["data"] == "synthetic" and "workload" in d["config"]
    cb = d["cpu_baseline"]
    assert cb["kind"] in ("reference", "port") and cb["cores"] >= 1 and cb["value"] == d["value"] and cb["sample"]
    assert d["e2e"] == {"value": d["value"], "unit": "points/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


def test_reference_arm_other_ranks_exit_quietly():
    import os
    env = dict(os.environ, RANK="1", WORLD_SIZE="2", LOCAL_RANK="1")
    res = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--gpus", "2", "--steps", "1",
                          "--warmup", "0"], capture_output=True, text=True, timeout=120, cwd=ROOT, env=env)
    assert res.returncode == 0 and res.stdout.strip() == ""


def test_own_arm_fails_loudly_without_enough_gpus():
    """``--gpus N`` never degrades to fewer ranks: outside torchrun it starts N ranks itself and refuses when the
    box has fewer than N devices; under a launcher whose WORLD_SIZE disagrees with N it refuses as well."""
    import os
    import torch
    have = torch.cuda.device_count() if torch.cuda.is_available() else 0
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    want = have + 1 if have else 2
    res = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", str(want), "--steps", "1", "--warmup", "3"],
                         capture_output=True, text=True, timeout=300, cwd=ROOT, env=env)
    assert res.returncode != 0 and res.stdout.strip() == ""
    assert f"--gpus {want}" in res.stderr and "CUDA device" in res.stderr
    res = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--steps", "1", "--warmup", "3"],
                         capture_output=True, text=True, timeout=300, cwd=ROOT,
                         env=dict(env, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0"))
    assert res.returncode != 0 and res.stdout.strip() == "" and "WORLD_SIZE is 1" in res.stderr


@pytest.mark.gpu
def test_own_arm_prints_one_contract_line():
    from tools import build_bundles
    if not build_bundles.have_bundle(build_bundles.workload_name(2)):
        pytest.skip("no cached config-2 index")
    res = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "1", "--steps", "4", "--warmup", "3",
                          "--points", "4000000", "--ref-points", "4000000", "--e2e-steps", "2", "--no-secondary"],
                         capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert res.returncode == 0, res.stderr[-2000:]
    lines = [l for l in res.stdout.splitlines() if l.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert "impl" not in d and d["metric"] == "joined_points_per_sec" and d["unit"] == "points/s"
    assert d["n_gpus"] == 1 and d["steps"] == 4 and d["warmup"] == 3 and d["higher_is_better"] is True
    assert d["value"] > 0 and d["ms_per_step"] > 0 and d["vs_baseline"] is None and d["scaling"] == "weak"
    assert d["dtype"] == "f64" and d["data"] == "synthetic" and "workload" in d["config"]
    assert d["gpu_launches"] == 4  # one join_kernel launch per step
    assert set(d["clocks"]) >= {"sm_mhz", "sm_max_mhz", "reasons"}
    e = d["e2e"]
    assert e["value"] > 0 and e["unit"] == "points/s" and e["h2d_bytes_per_step"] == 16 * 4000000
    assert e["d2h_bytes_per_step"] >= 4 * 4000000
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0 < r["frac"] < 1.2 and r["peak"] > 1000
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9 and "traffic" in r
    assert "ncu_stale" in r and "sectors_per_request" in r and "l2_hit_rate_pct" in r
    cb = d["cpu_baseline"]
    assert cb["kind"] in ("reference", "port") and cb["cores"] >= 1 and cb["value"] > 0 and cb["sample"]
    assert d["counts_equal_reference"] is True and d["secondary"] is None


@pytest.mark.gpu
def test_own_arm_through_its_own_launcher_and_nccl():
    """``--spawn`` takes the route ``--gpus N > 1`` takes by itself — re-exec under torch.distributed.run, NCCL
    process group, barriers, max-over-ranks timing, the counts all-reduce — with the one rank a one-GPU box allows."""
    from tools import build_bundles
    if not build_bundles.have_bundle(build_bundles.workload_name(2)):
        pytest.skip("no cached config-2 index")
    res = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "1", "--spawn", "--steps", "3", "--warmup", "3",
                          "--points", "3000000", "--ref-points", "3000000", "--e2e-steps", "1", "--no-secondary"],
                         capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert res.returncode == 0, res.stderr[-3000:]
    lines = [l for l in res.stdout.splitlines() if l.strip()]
    assert len(lines) == 1, res.stdout[-2000:]  # stdout carries the JSON line and nothing else
    d = json.loads(lines[0])
    assert d["n_gpus"] == 1 and d["gpu_launches"] == 3 and d["counts_equal_reference"] is True
    assert "torch.distributed.run" in res.stderr and "NCCL process group of 1 rank(s) up" in res.stderr
