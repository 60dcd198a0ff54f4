"""CPU: pin the C oracle (oracle/oracle.c) before trusting it.

1. against the reference's own known-answer tests (restated from
   proj/tests/test_krp.cpp, test_mttkrp.cpp, test_cpals.cpp, test_linalg.cpp);
2. against golden vectors produced by the unmodified reference library
   (tests/golden/*.npz, made by tests/golden/make_golden.py from oracle/_ref);
3. against the reference library itself when oracle/_ref is built.
"""
import os

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def rel(a, b):
    r = np.linalg.norm(b)
    return np.linalg.norm(a - b) / r if r else np.linalg.norm(a - b)


def test_generators_match_golden(oracle):
    g = np.load(os.path.join(GOLD, "gen.npz"))
    assert np.array_equal(oracle.gen_tensor((3, 4, 5), 17), g["gen_tensor_3x4x5_s17"])
    for k, m in enumerate(oracle.gen_factors((3, 4, 5), 5, 23)):
        assert np.array_equal(m, g[f"gen_factors_3x4x5_r5_s23_{k}"])
    f, lam = oracle.kruskal_random((4, 5, 6), 3, 99)
    for k, m in enumerate(f):
        assert np.array_equal(m, g[f"kruskal_4x5x6_r3_s99_{k}"])
    assert np.all(lam == 1.0)


def test_python_mt19937_matches_oracle(oracle):
    from paper_1708_08976_b200._mt19937 import mt19937_64
    m = mt19937_64(99)
    vals = np.array([(m.next() >> 11) * 2.0 ** -53 for _ in range(50)])
    assert np.array_equal(vals, oracle.uniform(99, 50))


def test_krp_known_answers(oracle):
    a, b, c = np.array([[1.0, 2.0]]), np.array([[3.0, 4.0]]), np.array([[5.0, 6.0]])
    assert oracle.krp([a, b, c]).tolist() == [[15.0, 48.0]]  # test_krp.cpp:41-49
    k = oracle.krp([np.array([[1.0], [2.0]]), np.array([[3.0], [4.0]])])
    assert k[:, 0].tolist() == [3.0, 4.0, 6.0, 8.0]  # test_krp.cpp:51-61


def test_krp_matches_golden_bitwise(oracle):
    g = np.load(os.path.join(GOLD, "krp.npz"))
    keys = sorted({k.rsplit("_", 1)[0] for k in g.files if k.endswith("_out")})
    assert keys
    for key in keys:
        dims = g[f"{key}_dims"]
        ins = [g[f"{key}_in{z}"] for z in range(len(dims))]
        assert np.array_equal(oracle.krp(ins), g[f"{key}_out"]), key


def test_mttkrp_known_answers(oracle):
    dims = (2, 2, 2)  # test_mttkrp.cpp:68-88
    for mode in range(3):
        m = oracle.mttkrp(np.ones(8), dims, [np.ones((2, 1))] * 3, mode)
        assert m.tolist() == [[4.0], [4.0]]
    f = [np.zeros((2, 2)), np.array([[1, 0], [0, 1], [0, 0]], float), np.ones((2, 2))]
    assert oracle.mttkrp(np.arange(12.0), (2, 3, 2), f, 0).tolist() == [[6.0, 10.0], [8.0, 12.0]]


def test_mttkrp_matches_golden(oracle):
    g = np.load(os.path.join(GOLD, "mttkrp.npz"))
    si = 0
    while f"s{si}_dims" in g.files:
        dims = tuple(int(d) for d in g[f"s{si}_dims"])
        x = g[f"s{si}_x"]
        assert np.array_equal(x, oracle.gen_tensor(dims, 17))
        for rank in (1, 2, 5):
            fs = [g[f"s{si}_r{rank}_f{k}"] for k in range(len(dims))]
            for mode in range(len(dims)):
                got = oracle.mttkrp(x, dims, fs, mode)
                assert rel(got, g[f"s{si}_r{rank}_m{mode}_loops"]) <= 1e-15
                assert rel(got, g[f"s{si}_r{rank}_m{mode}_auto"]) <= 1e-12
        si += 1
    assert si >= 8


def test_cp_als_matches_golden(oracle):
    g = np.load(os.path.join(GOLD, "cpals.npz"))
    ci = 0
    while f"c{ci}_dims" in g.files:
        dims = tuple(int(d) for d in g[f"c{ci}_dims"])
        rank, iters, seed = (int(v) for v in g[f"c{ci}_meta"])
        if np.prod(dims) * rank * iters * len(dims) > 5e7:  # keep the CPU suite quick
            ci += 1
            continue
        x = oracle.gen_tensor(dims, 31)
        _, lam, fits, zero = oracle.cp_als(x, dims, rank, iters, 0.0, seed)
        assert not zero
        assert np.max(np.abs(fits - g[f"c{ci}_fits"])) <= 1e-9, ci
        assert abs(oracle.tensor_norm(x) - g[f"c{ci}_norm"][0]) <= 1e-12 * g[f"c{ci}_norm"][0]
        ci += 1


def test_normalize_and_solve_known_answers(oracle):
    u, lam = oracle.normalize_mode(np.array([[3.0, 0.0], [4.0, 0.0]]))  # test_cpals.cpp:60-70
    assert lam.tolist() == [5.0, 0.0]
    assert np.allclose(u[:, 0], [0.6, 0.8]) and np.all(u[:, 1] == 0.0)
    u, chol = oracle.solve_psd(np.eye(3), np.arange(6.0).reshape(2, 3))
    assert chol and np.array_equal(u, np.arange(6.0).reshape(2, 3))
    _, chol = oracle.solve_psd(np.ones((3, 3)), np.ones((1, 3)))
    assert not chol  # singular -> Jacobi pseudo-inverse (linalg.cpp:358-386)


def test_oracle_against_reference_library(oracle, ref):
    dims = (7, 6, 5, 4)
    x = ref.gen_tensor(dims, 3)
    f = ref.gen_factors(dims, 6, 4)
    for mode in range(4):
        assert rel(oracle.mttkrp(x, dims, f, mode), ref.mttkrp(x, dims, f, mode, "one_step", threads=2)) <= 1e-12
    h_o = oracle.gram_hadamard(f, 1)
    h_r = ref.gram_hadamard(f, 1)
    assert rel(h_o, h_r) <= 1e-14
    m = oracle.uniform(5, 6 * 6).reshape(6, 6)
    assert rel(oracle.solve_psd(h_r, m)[0], ref.solve_psd(h_r, m)) <= 1e-10
