"""Acceptance check 4 of the reference (proj/tests/acceptance.cpp:304-369: no
algorithm ever writes X) on the device: tests/readonly_check.py runs every
flavor on a tensor mapped read-only with the CUDA virtual-memory API, in its
own process (a write would fault and poison that process's context)."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

pytestmark = pytest.mark.gpu


def test_every_flavor_reads_a_read_only_tensor():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "readonly_check.py")], capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert "readonly ok" in r.stdout
