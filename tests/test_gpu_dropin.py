"""The C++ drop-in shim (include/dmtk_gpu.hpp) driven by a C++ program that
uses the reference's own types (tests/cpp/drop_in_test.cpp), checked against
the unmodified reference library."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "drop_in_test")


@pytest.mark.gpu
def test_cpp_drop_in_driver():
    if not os.path.exists(BIN):
        pytest.skip("tests/cpp/drop_in_test not built (needs /root/reference headers at build time)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout[-2000:])
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert "0 failed" in r.stdout
