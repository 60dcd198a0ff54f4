"""GPU parity for the Khatri-Rao product and CP-ALS through the C ABI.

KRP: bitwise equality with the Kronecker oracle (reference test_krp.cpp:69-91,
krp.hpp:19-32) and the reference's KrpStats counts (test_krp.cpp:108-155).
CP-ALS: reference test_cpals.cpp cases, plus fits within 1e-9 of the
reference after the same number of iterations (BASELINE.json north_star).
"""
import os
import numpy as np
import pytest

import paper_1708_08976_b200 as dg
from paper_1708_08976_b200 import AlsConfig, MttkrpAlgo as A

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def inputs(oracle, dims, cols, seed):
    return [oracle.uniform(seed + z * 1000, d * cols).reshape(d, cols) for z, d in enumerate(dims)]


@pytest.mark.parametrize("dims", [(6,), (3, 4), (2, 3, 4), (3, 2, 2, 3), (2, 2, 3, 2, 2), (4, 1, 3), (1, 1, 5),
                                  (200, 200, 2), (5, 4, 3, 2)])
@pytest.mark.parametrize("cols", [1, 3, 16, 25])
def test_krp_bitwise(oracle, dims, cols):
    ins = inputs(oracle, dims, cols, 42)
    want = oracle.krp(ins)
    assert np.array_equal(dg.krp(ins), want)
    assert np.array_equal(dg.krp_naive(ins), want)


def test_krp_known_answers():
    a, b, c = np.array([[1.0, 2.0]]), np.array([[3.0, 4.0]]), np.array([[5.0, 6.0]])
    assert dg.krp([a, b, c]).tolist() == [[15.0, 48.0]]
    k = dg.krp([np.array([[1.0], [2.0]]), np.array([[3.0], [4.0]])])
    assert k[:, 0].tolist() == [3.0, 4.0, 6.0, 8.0]
    single = np.arange(15, dtype=float).reshape(5, 3)
    assert np.array_equal(dg.krp([single]), single)


def test_krp_stats_match_reference(ref, oracle):
    for dims in [(2, 2, 2), (2, 2, 2, 2), (3, 4, 5), (5, 4, 3, 2), (2, 3, 2, 3, 2), (4, 4, 4, 4), (3, 2)]:
        ins = inputs(oracle, dims, 3, 11)
        s1, s2 = dg.KrpStats(), dg.KrpStats()
        dg.krp(ins, 1, s1)
        dg.krp_naive(ins, 1, s2)
        _, want_reuse = ref.krp(ins, threads=1)
        _, want_naive = ref.krp(ins, threads=1, naive=True)
        assert s1.hadamard_products == want_reuse, dims
        assert s2.hadamard_products == want_naive, dims


def test_krp_validation():
    with pytest.raises(dg.InvalidArgument):
        dg.krp([])
    with pytest.raises(dg.InvalidArgument):
        dg.krp([np.ones((2, 2)), np.ones((2, 3))])
    with pytest.raises(dg.InvalidArgument):
        dg.krp([np.ones((2, 2)), None])


def test_krp_config1_product(oracle):
    """BASELINE config 1's 3-matrix KRP: 200x16 (.) 200x16 (.) 200x16 -> 8e6 x 16."""
    ins = oracle.gen_factors((200, 200, 200), 16, 2)
    got = dg.krp(ins)
    # spot-check bitwise on rows through the oracle's small products
    sub = oracle.krp([ins[0][:3], ins[1], ins[2]])
    assert np.array_equal(got[:sub.shape[0]], sub)
    r = 7_654_321
    d0, d1, d2 = r // 40000, (r // 200) % 200, r % 200
    assert np.array_equal(got[r], (ins[0][d0] * ins[1][d1]) * ins[2][d2])


def cp(x, dims, rank, iters, seed, tol=0.0, algo=A.automatic, tree=False):
    t = dg.DenseTensor(dims, x)
    return dg.cp_als(t, AlsConfig(rank=rank, max_iters=iters, tol=tol, seed=seed, algo=algo, dimension_tree=tree))


@pytest.mark.parametrize("dims,rank,iters", [((6, 5, 4), 3, 6), ((7, 6, 5), 3, 8), ((8, 9, 10), 4, 40),
                                             ((12, 10, 8, 6), 5, 10), ((40, 40, 12, 8), 20, 25),
                                             # ranks above 22: two Gram / inverse entries per thread of the
                                             # two-launch factor update; 4000 rows: several row blocks per CTA
                                             ((30, 28, 26), 32, 8), ((4000, 6, 5), 27, 6), ((33, 9, 7, 5), 23, 8)])
def test_cp_als_fits_match_reference(ref, oracle, dims, rank, iters):
    x = oracle.gen_tensor(dims, 31)
    got = cp(x, dims, rank, iters, 7)
    want = ref.cp_als(x, dims, rank, iters, tol=0.0, seed=7)
    f_got = np.array([r.fit.fit for r in got.trace.iters])
    assert len(f_got) == len(want["fits"])
    assert np.max(np.abs(f_got - want["fits"])) <= 1e-9
    assert abs(got.trace.tensor_norm - want["norm_x"]) <= 1e-12 * want["norm_x"]
    for u in got.model.factors:  # final factors column-normalised (test_cpals.cpp:157-167)
        assert np.allclose(np.linalg.norm(u, axis=0), 1.0, rtol=1e-12, atol=0)
    assert np.all(got.model.lambda_ >= 0)


@pytest.mark.parametrize("dims,rank,iters", [((6, 5, 4), 3, 6), ((8, 9, 10), 4, 40), ((12, 10, 8, 6), 5, 10),
                                             ((40, 40, 12, 8), 20, 25), ((5, 4, 3, 2, 6), 4, 12),
                                             ((9, 3, 4, 2, 2, 5), 6, 10)])
def test_cp_als_dimension_tree_matches_reference(ref, oracle, dims, rank, iters):
    """Dimension-tree sweep (two tensor passes per iteration):
    the same updates as the reference's per-mode sweep, fits within 1e-9."""
    x = oracle.gen_tensor(dims, 31)
    got = cp(x, dims, rank, iters, 7, tree=True)
    want = ref.cp_als(x, dims, rank, iters, tol=0.0, seed=7)
    f_got = np.array([r.fit.fit for r in got.trace.iters])
    assert len(f_got) == len(want["fits"])
    assert np.max(np.abs(f_got - want["fits"])) <= 1e-9
    for u in got.model.factors:
        assert np.allclose(np.linalg.norm(u, axis=0), 1.0, rtol=1e-12, atol=0)
    again = cp(x, dims, rank, iters, 7, tree=True)  # deterministic
    assert [r.fit.fit for r in again.trace.iters] == list(f_got)


def test_cp_als_four_launch_update_chain_matches_reference(ref, oracle):
    """DMTK_GPU_ALS_FUSED=0 (read once per process, hence the subprocess): the
    solve / apply / normalise / Gram chain gives the reference's fits too."""
    import subprocess
    import sys
    code = (
        "import sys, numpy as np; sys.path[:0] = [%r, %r]\n"
        "import paper_1708_08976_b200 as dg\n"
        "from oracle_bindings import Oracle, Ref\n"
        "o, r = Oracle(), Ref()\n"
        "for dims, rank, iters in (((12, 10, 8, 6), 5, 10), ((30, 28, 26), 32, 6)):\n"
        "    x = o.gen_tensor(dims, 31)\n"
        "    got = dg.cp_als(dg.DenseTensor(dims, x), dg.AlsConfig(rank=rank, max_iters=iters, tol=0.0, seed=7))\n"
        "    want = r.cp_als(x, dims, rank, iters, tol=0.0, seed=7)\n"
        "    f = np.array([it.fit.fit for it in got.trace.iters])\n"
        "    assert np.max(np.abs(f - want['fits'])) <= 1e-9, (dims, f, want['fits'])\n"
        "print('ok')\n" % (ROOT, os.path.join(ROOT, "tests")))
    env = dict(os.environ, DMTK_GPU_ALS_FUSED="0")
    res = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert res.returncode == 0 and "ok" in res.stdout, res.stderr[-3000:]


def test_cp_als_monotone_and_deterministic(oracle):
    dims = (8, 9, 10)
    x = oracle.gen_tensor(dims, 77)
    a = cp(x, dims, 4, 40, 13)
    b = cp(x, dims, 4, 40, 13)
    fa = [r.fit.fit for r in a.trace.iters]
    assert len(fa) == 40
    assert all(fa[i] >= fa[i - 1] - 1e-10 for i in range(1, 40))
    assert fa == [r.fit.fit for r in b.trace.iters]
    for u, v in zip(a.model.factors, b.model.factors):
        assert np.array_equal(u, v)


def test_cp_als_rank1_recovery(oracle):
    dims = (8, 7, 6)
    f, lam = oracle.kruskal_random(dims, 1, 3)
    x = oracle.reconstruct(f, lam)
    res = cp(x, dims, 1, 30, 5)
    assert res.trace.iters[-1].fit.fit >= 1 - 1e-6


def test_cp_als_tolerance_stop_and_zero_tensor(oracle):
    dims = (5, 5, 5)
    x = oracle.gen_tensor(dims, 9)
    assert len(cp(x, dims, 2, 50, 3, tol=1.0).trace.iters) == 2
    assert len(cp(x, dims, 2, 12, 3, tol=0.0).trace.iters) == 12
    z = cp(np.zeros(64), (4, 4, 4), 2, 10, 1)
    assert z.trace.zero_tensor and z.trace.iters == [] and z.trace.tensor_norm == 0.0
    assert all(np.all(u == 0) for u in z.model.factors) and np.all(z.model.lambda_ == 0)


def test_cp_als_algorithms_agree(oracle):
    dims = (6, 7, 8)
    x = oracle.gen_tensor(dims, 50)
    fits = [cp(x, dims, 3, 8, 4, algo=a).trace.iters[-1].fit.fit for a in (A.automatic, A.baseline, A.one_step)]
    assert abs(fits[1] - fits[0]) <= 1e-8 and abs(fits[2] - fits[0]) <= 1e-8
    with pytest.raises(dg.InvalidArgument):
        cp(x, dims, 3, 8, 4, algo=A.two_step)


def test_cp_als_validation(oracle):
    x = oracle.gen_tensor((3, 3), 1)
    for bad in (AlsConfig(rank=0), AlsConfig(rank=2, max_iters=-1), AlsConfig(rank=2, threads=0)):
        with pytest.raises(dg.InvalidArgument):
            dg.cp_als(dg.DenseTensor((3, 3), x), bad)


def test_fit_matches_reference(ref, oracle):
    dims = (6, 5, 4)
    x = oracle.gen_tensor(dims, 31)
    f, lam = oracle.kruskal_random(dims, 3, 7)
    lam = np.array([2.0, 0.5, 1.0])
    got = dg.fit(dg.DenseTensor(dims, x), dg.KruskalModel(f, lam))
    want = ref.fit(x, dims, f, lam)
    assert abs(got.fit - want["fit"]) <= 1e-10 and got.defined
    with pytest.raises(dg.InvalidArgument):
        dg.fit(dg.DenseTensor(dims, x), dg.KruskalModel(f[:2], lam))


def test_gram_hadamard_and_solve(ref, oracle):
    f, _ = oracle.kruskal_random((9, 8, 7), 5, 1)
    for skip in (-1, 0, 1, 2):
        assert np.allclose(dg.gram_hadamard(f, skip), ref.gram_hadamard(f, skip), rtol=1e-13, atol=0)
    h = ref.gram_hadamard(f, 1)
    m = oracle.uniform(3, 8 * 5).reshape(8, 5)
    assert np.allclose(dg.solve_psd(h, m), ref.solve_psd(h, m), rtol=1e-9, atol=1e-12)
    # singular H -> Jacobi pseudo-inverse path (test_linalg.cpp:239-298)
    hs = np.ones((3, 3))
    ms = np.array([[3.0, 3.0, 3.0], [1.0, 2.0, 3.0]])
    assert np.allclose(dg.solve_psd(hs, ms), ref.solve_psd(hs, ms), rtol=1e-9, atol=1e-12)


def test_tensor_norm(oracle, ref):
    dims = (30, 20, 11)
    x = oracle.gen_tensor(dims, 2)
    assert abs(dg.tensor_norm(dg.DenseTensor(dims, x)) - ref.tensor_norm(x, dims)) <= 1e-13 * ref.tensor_norm(x, dims)


@pytest.mark.parametrize("rows,C", [((37, 11, 6), 6), ((200, 200, 9), 16), ((5, 7), 25), ((64, 3, 64, 2), 3)])
def test_krp_device_bitwise(rows, C):
    """Device-resident KRP (16-byte vector path on aligned torch buffers) is
    bitwise the host-API KRP (and hence the reference, test_krp.cpp:69-81)."""
    import torch
    g = torch.Generator(device="cuda").manual_seed(11)
    ins = [torch.rand((r, C), dtype=torch.float64, device="cuda", generator=g) for r in rows]
    total = int(np.prod(rows))
    out = torch.empty((total, C), dtype=torch.float64, device="cuda")
    scr = torch.empty((2 * max(1, int(np.prod(rows[:-1]))), C), dtype=torch.float64, device="cuda")
    dg.krp_device([t.data_ptr() for t in ins], list(rows), C, out.data_ptr(), scr.data_ptr(),
                  torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    host = dg.krp([t.cpu().numpy() for t in ins])
    assert np.array_equal(out.cpu().numpy(), host)


def _sym_tensor(oracle, dims, seed):
    """U[0,1) tensor symmetrised in modes 0 and 1 (natural order, mode 0 fastest)."""
    x = oracle.gen_tensor(dims, seed).reshape(dims[::-1])
    x = x + np.swapaxes(x, -1, -2)  # X(i, j, ...) + X(j, i, ...)
    return np.ascontiguousarray(x).reshape(-1)


@pytest.mark.parametrize("dims,rank,iters", [((8, 8, 5, 3), 3, 10), ((12, 12, 7, 5), 5, 12), ((9, 9, 4, 3, 2), 4, 8),
                                             ((7, 7, 10), 3, 15), ((40, 40, 12, 8), 20, 25), ((101, 101, 6), 4, 5)])
def test_cp_als_symmetric_packed_matches_reference(ref, oracle, dims, rank, iters):
    """Tensors symmetric in modes 0/1 packed to their upper triangles (SURVEY
    8f-4): the packed dimension-tree sweep reads about half the bytes; its fits
    agree with the reference's CP-ALS on the full tensor within 1e-9."""
    x = _sym_tensor(oracle, dims, 41)
    t = dg.DenseTensor(dims, x)
    tp = t.pack_symmetric01()
    got = dg.cp_als(tp, AlsConfig(rank=rank, max_iters=iters, tol=0.0, seed=7))
    want = ref.cp_als(x, dims, rank, iters, tol=0.0, seed=7)
    f_got = np.array([r.fit.fit for r in got.trace.iters])
    assert len(f_got) == len(want["fits"])
    assert np.max(np.abs(f_got - want["fits"])) <= 1e-9
    assert abs(got.trace.tensor_norm - want["norm_x"]) <= 1e-12 * want["norm_x"]
    assert abs(dg.tensor_norm(tp) - want["norm_x"]) <= 1e-12 * want["norm_x"]
    for u in got.model.factors:
        assert np.allclose(np.linalg.norm(u, axis=0), 1.0, rtol=1e-12, atol=0)


def test_pack_symmetric_validation(oracle):
    dims = (6, 6, 4)
    x = oracle.gen_tensor(dims, 3)  # not symmetric
    with pytest.raises(dg.InvalidArgument):
        dg.DenseTensor(dims, x).pack_symmetric01()
    with pytest.raises(dg.InvalidArgument):
        dg.DenseTensor((6, 5, 4), oracle.gen_tensor((6, 5, 4), 3)).pack_symmetric01()
    tp = dg.DenseTensor(dims, _sym_tensor(oracle, dims, 3)).pack_symmetric01()
    f = oracle.gen_factors(dims, 2, 1)
    with pytest.raises(dg.InvalidArgument):  # packed handles only run cp_als / tensor_norm
        dg.mttkrp(dg.MttkrpRequest(tp, f, 0))


# ----------------------------------------------------------- ranks above 64
@pytest.mark.parametrize("dims,rank", [((90, 85, 80), 72), ((70, 66, 8, 9), 100)])
def test_cp_als_rank_above_64_matches_reference(ref, oracle, dims, rank):
    """The reference takes any rank >= 1 (cp_als.cpp:175-177): ranks above 64
    run the per-mode sweep with the global-memory factor update (als_wide.cu:
    left-looking Cholesky + row substitution, the Jacobi fallback)."""
    x = oracle.gen_tensor(dims, 31)
    got = cp(x, dims, rank, 6, 7)
    want = ref.cp_als(x, dims, rank, 6, tol=0.0, seed=7)
    f_got = np.array([r.fit.fit for r in got.trace.iters])
    assert np.max(np.abs(f_got - want["fits"])) <= 1e-9
    for u, v in zip(got.model.factors, want["factors"]):
        assert np.linalg.norm(u - v) <= 1e-6 * np.linalg.norm(v)
    t = dg.DenseTensor(dims, x)
    fr = dg.fit(t, got.model)
    rf = ref.fit(x, dims, got.model.factors, got.model.lambda_)
    assert abs(fr.fit - rf["fit"]) <= 1e-9
    with pytest.raises(dg.InvalidArgument):
        dg.cp_als(t, AlsConfig(rank=rank, max_iters=2, tol=0.0, seed=7, dimension_tree=True))


def test_gram_hadamard_and_solve_rank_above_64(ref, oracle):
    f = oracle.gen_factors((120, 110, 100), 96, 5)
    h = dg.gram_hadamard(f, 1)
    want = ref.gram_hadamard(f, 1)
    assert np.linalg.norm(h - want) <= 1e-13 * np.linalg.norm(want)
    m = oracle.gen_factors((300,), 96, 6)[0]
    u = dg.solve_psd(h, m)
    assert np.linalg.norm(u - ref.solve_psd(h, m)) <= 1e-8 * np.linalg.norm(u)
    # a singular system (rank-deficient Gram): the Jacobi pseudo-inverse path
    g = oracle.gen_factors((40,), 80, 7)[0]
    hs = g.T @ g
    us = dg.solve_psd(hs, m[:, :80].copy())
    ws = ref.solve_psd(hs, m[:, :80].copy())
    assert np.linalg.norm(us - ws) <= 1e-6 * np.linalg.norm(ws)


@pytest.mark.timeout(300)
def test_loopback_sharded_rank_above_64(oracle, ref):
    from paper_1708_08976_b200.distributed import loopback_cp_als
    dims, rank = (70, 66, 9, 10), 80
    x = oracle.gen_tensor(dims, 3)
    t = dg.DenseTensor(dims, x)
    res, _ = loopback_cp_als(t, 3, AlsConfig(rank=rank, max_iters=4, tol=0.0, seed=2))
    want = ref.cp_als(x, dims, rank, 4, tol=0.0, seed=2)
    assert np.max(np.abs(np.array(res[0].fits) - want["fits"])) <= 1e-9


@pytest.mark.parametrize("dims,rank,tree", [((2, 2, 2), 5, False), ((3, 2, 4), 7, False), ((2, 3, 2, 2), 6, False),
                                            ((2, 3, 2, 2), 6, True)])
def test_cp_als_singular_systems_match_reference(ref, oracle, dims, rank, tree):
    """Ranks above what the tiny extents support make every H = Hadamard of
    Grams singular (a 2-row factor's Gram has rank 2): each ALS update takes
    the Jacobi pseudo-inverse, which the Gauss-Jordan solve CTA now computes
    itself (no separate fallback launches). Such ranks exceed the tensor's
    rank; near an exact fit, fit = 1 - sqrt(res^2) / ||X|| turns
    rounding-level differences of res^2 (~1e-16) into ~1e-8, so the bound on
    the fits is 1e-7."""
    x = oracle.gen_tensor(dims, 5)
    res = cp(x, dims, rank, 6, 11, tree=tree)
    got = np.array([it.fit.fit for it in res.trace.iters])
    rf = ref.cp_als(x, dims, rank, 6, tol=0.0, seed=11)
    assert np.max(np.abs(got - rf["fits"])) <= 1e-7, (got, rf["fits"])
