"""Host-side check (no GPU) of the jump-ahead behind the on-device gen_tensor
(csrc/mt_gen.cu): the window a generator CTA starts from, formed from the first
raw words of mt19937_64(seed) and x^(311+start) mod phi, must temper to the
reference stream's draws start .. start+311 (bench.cpp:22-24, 88-97; the C
oracle's restatement is pinned against the reference in test_oracle.py).
"""
import ctypes as C

import numpy as np
import pytest

from paper_1708_08976_b200 import _lib


def _temper(y):
    y = y.copy()
    y ^= (y >> np.uint64(29)) & np.uint64(0x5555555555555555)
    y ^= (y << np.uint64(17)) & np.uint64(0x71D67FFFEDA60000)
    y ^= (y << np.uint64(37)) & np.uint64(0xFFF7EEE000000000)
    y ^= y >> np.uint64(43)
    return (y >> np.uint64(11)).astype(np.float64) * 2.0**-53


@pytest.mark.parametrize("seed", [0, 23, 2**64 - 1])
@pytest.mark.parametrize("start", [0, 1, 155, 156, 311, 312, 100003, 1351352])
def test_jump_window_matches_stream(oracle, seed, start):
    w = np.empty(312, dtype=np.uint64)
    assert _lib.lib.dmtk_gpu_mt64_jump(seed, start, w.ctypes.data_as(C.POINTER(C.c_uint64))) == 0
    want = oracle.uniform(seed, start + 312)[start:]
    assert np.array_equal(_temper(w), want)


def test_jump_rejects_negative_start():
    w = np.empty(312, dtype=np.uint64)
    assert _lib.lib.dmtk_gpu_mt64_jump(1, -1, w.ctypes.data_as(C.POINTER(C.c_uint64))) == -1
