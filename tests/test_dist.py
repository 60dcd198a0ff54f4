"""CPU: the seeded value distributions of BASELINE configs 3-5 (SURVEY.md 8d,
BASELINE.md 3) in the test-side restatement (oracle/oracle.c orc_gen_dist).

The uniforms underneath are the reference's gen_tensor stream (bench.cpp:88-97,
pinned by gen.npz); the transforms are the published Box-Muller and tanh
formulas, checked here against numpy (libm) to 1e-12, and frozen bitwise by
tests/golden/dist.npz (make_dist_golden.py). tests/test_gpu_generate.py checks
the device generator against this restatement bitwise.
"""
import os

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def box_muller_np(u):
    u0, u1 = u[0::2], u[1::2]
    r = np.sqrt(-2.0 * np.log(1.0 - u0))
    z = np.empty_like(u)
    z[0::2] = r * np.cos(2 * np.pi * u1)
    z[1::2] = r * np.sin(2 * np.pi * u1)
    return z


def test_signed_is_exact_affine_of_reference_stream(oracle):
    g = np.load(os.path.join(GOLD, "gen.npz"))
    u = g["gen_tensor_3x4x5_s17"]  # the reference library's gen_tensor bytes
    assert np.array_equal(oracle.gen_dist((3, 4, 5), 17, "signed"), 2.0 * u - 1.0)


@pytest.mark.parametrize("dims", [(9, 8, 7), (5, 3), (7,)])
def test_normal_is_box_muller(oracle, dims):
    n = int(np.prod(dims))
    u = oracle.uniform(12, n + (n & 1))
    want = box_muller_np(u)[:n]
    got = oracle.gen_dist(dims, 12, "normal")
    assert np.max(np.abs(got - want)) <= 1e-12


def test_normal_statistics(oracle):
    z = oracle.gen_dist((1000, 1000), 3, "normal")
    assert abs(z.mean()) < 5e-3 and abs(z.var() - 1.0) < 5e-3
    assert np.all(np.isfinite(z))


def test_symslice_structure(oracle):
    dims = (6, 6, 4, 3)
    x = oracle.gen_dist(dims, 14, "symslice").reshape(3, 4, 6, 6)  # (q2, q1, j, i)
    assert np.array_equal(x, np.swapaxes(x, 2, 3))
    assert np.all(x[:, :, range(6), range(6)] == 1.0)
    # off-diagonals: tanh(0.3 z_m), m = q P + j (j - 1) / 2 + i for i < j
    I, P, R = 6, 15, 12
    u = oracle.uniform(14, P * R + ((P * R) & 1))
    z = box_muller_np(u)
    flat = x.reshape(R, I, I)
    for q in range(R):
        for j in range(I):
            for i in range(j):
                want = np.tanh(0.3 * z[q * P + j * (j - 1) // 2 + i])
                assert abs(flat[q, j, i] - want) <= 1e-12


def test_factors_follow_gen_factors_streams(oracle):
    g = np.load(os.path.join(GOLD, "gen.npz"))
    got = oracle.gen_factors_dist((3, 4, 5), 5, 23, "signed")
    for k, m in enumerate(got):
        assert np.array_equal(m, 2.0 * g[f"gen_factors_3x4x5_r5_s23_{k}"] - 1.0)


def test_frozen_bytes(oracle):
    g = np.load(os.path.join(GOLD, "dist.npz"))
    for key in g.files:
        dist, shape, seed = key.split("_")
        dims = tuple(int(v) for v in shape.split("x"))
        for threads in (1, 3):
            assert np.array_equal(oracle.gen_dist(dims, int(seed[1:]), dist, threads=threads), g[key]), key
