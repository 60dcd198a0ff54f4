"""CPU: the C-ABI library loads, exports every entry point include/dmtk_gpu.h
declares, and -- with no GPU -- fails loudly instead of falling back to CPU
code. Plus the host-side pieces that need no device (validation order and
messages, choose_order, shape checks)."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "dmtk_gpu.h")
LIB = os.path.join(ROOT, "paper_1708_08976_b200", "libdmtk_gpu.so")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(dmtk_gpu_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    assert os.path.exists(LIB), "run __graft_entry__.build() first"
    lib = ctypes.CDLL(LIB)
    syms = declared_symbols()
    assert len(syms) >= 18
    for s in syms:
        assert hasattr(lib, s), s
    from paper_1708_08976_b200 import _lib
    assert set(syms) == set(_lib.EXPORTED)


def test_library_is_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out.replace("sm_100a", ""))


def test_no_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    import paper_1708_08976_b200 as dg
    assert dg.device_count() == 0
    with pytest.raises(dg.DeviceError, match="no CPU fallback"):
        dg.krp([np.ones((2, 2)), np.ones((3, 2))])
    t = dg.DenseTensor((2, 2, 2), np.ones(8))
    with pytest.raises(dg.DeviceError):
        dg.mttkrp(dg.MttkrpRequest(t, [np.ones((2, 1))] * 3, 0))


def test_host_validation_without_device():
    import paper_1708_08976_b200 as dg
    from paper_1708_08976_b200 import TwoStepOrder as O
    assert dg.choose_order((20, 30, 40), 1) == O.right  # test_mttkrp.cpp:153-158
    assert dg.choose_order((40, 30, 20), 1) == O.left
    assert dg.choose_order((5, 3, 5), 1) == O.right
    assert dg.choose_order((2, 3, 4, 5), 2) == O.left
    with pytest.raises(dg.InvalidArgument, match="extent of mode 1 must be >= 1"):
        dg.choose_order((3, 0, 2), 0)
    with pytest.raises(dg.ShapeOverflow):
        dg.choose_order((1 << 40, 1 << 40), 0)
    with pytest.raises(dg.InvalidArgument):
        dg.mttkrp(dg.MttkrpRequest(None, [], 0))
    with pytest.raises(dg.InvalidArgument, match="krp: input 1 has 3 columns, expected 2"):
        dg.krp([np.ones((2, 2)), np.ones((2, 3))])
    with pytest.raises(dg.InvalidArgument, match="empty input list"):
        dg.krp([])


def test_cpp_shim_header_compiles():
    """include/dmtk_gpu.hpp against the reference headers (syntax-only)."""
    if not os.path.isdir("/root/reference/proj/include"):
        pytest.skip("reference headers absent")
    src = '#include "dmtk_gpu.hpp"\nint main(){return 0;}\n'
    r = subprocess.run(["g++", "-std=c++20", "-fsyntax-only", "-x", "c++", "-", "-I", os.path.join(ROOT, "include"),
                        "-I", "/root/reference/proj/include"], input=src, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
