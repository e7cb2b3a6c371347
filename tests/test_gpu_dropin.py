"""Runs the compiled C++ drop-in test (tests/cpp/dropin_test.cpp): the
reference library and geojoin::gpu (include/geojoin_gpu.hpp) side by side on
the same IndexBundle, through the reference's own C++ types."""
import subprocess
from pathlib import Path

import pytest

BIN = Path(__file__).resolve().parent / "cpp" / "dropin_test"


@pytest.mark.gpu
def test_cpp_dropin_against_reference_library():
    if not BIN.exists():
        pytest.skip("tests/cpp/dropin_test not built (needs /root/reference at build time)")
    res = subprocess.run([str(BIN)], capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stdout + res.stderr
    assert "DROPIN OK" in res.stdout
