"""GPU parity for MTTKRP through the C ABI (libdmtk_gpu.so) against the C
oracle (oracle/oracle.c, restating reference oracle.cpp:38-70) and the
reference library itself (oracle/_ref).

Mirrors reference tests/test_mttkrp.cpp case by case; tolerance is the
reference's: relative Frobenius error <= 1e-12 (test_mttkrp.cpp:134,
bench.cpp:20).
"""
import os

import numpy as np
import pytest

import paper_1708_08976_b200 as dg
from paper_1708_08976_b200 import MttkrpAlgo as A
from paper_1708_08976_b200 import TwoStepOrder as O

pytestmark = pytest.mark.gpu
TOL = 1e-12


def rel(got, want):
    d = np.linalg.norm(got - want)
    r = np.linalg.norm(want)
    return d if r == 0 else d / r


def run(x, dims, factors, mode, algo=A.automatic, order=O.automatic, threads=1):
    t = dg.DenseTensor(dims, x)
    return dg.mttkrp(dg.MttkrpRequest(t, factors, mode, algo, order, threads))


def algos_for(mode, n):
    out = [(A.baseline, O.automatic), (A.one_step, O.automatic), (A.automatic, O.automatic)]
    if 0 < mode < n - 1:
        out += [(A.two_step, O.left), (A.two_step, O.right), (A.two_step, O.automatic)]
    return out


# test_mttkrp.cpp:68-88
def test_all_ones_cube():
    dims = (2, 2, 2)
    x = np.ones(8)
    f = [np.ones((2, 1)) for _ in range(3)]
    for mode in range(3):
        for algo, order in algos_for(mode, 3):
            m = run(x, dims, f, mode, algo, order).m
            assert m[0, 0] == 4.0 and m[1, 0] == 4.0


# test_mttkrp.cpp:90-97
def test_zero_factor_zeroes_result(oracle):
    dims = (3, 4, 5)
    x = oracle.gen_tensor(dims, 5)
    f = oracle.kruskal_random(dims, 3, 6)[0]
    f[2][:] = 0.0
    m = run(x, dims, f, 0, A.one_step).m
    assert np.all(m == 0.0)


# test_mttkrp.cpp:99-118 (frozen 2x3x2 offsets tensor)
def test_frozen_small_case():
    dims = (2, 3, 2)
    x = np.arange(12, dtype=np.float64)
    f = [np.zeros((2, 2)), np.array([[1, 0], [0, 1], [0, 0]], dtype=float), np.ones((2, 2))]
    for algo in (A.baseline, A.one_step):
        m = run(x, dims, f, 0, algo).m
        assert m.tolist() == [[6.0, 10.0], [8.0, 12.0]]


REF_SHAPES = [(3, 4, 5), (2, 3, 4, 2), (2, 2, 2, 2, 2), (4, 1, 3), (6, 7), (9,)]


# test_mttkrp.cpp:120-151: every algorithm agrees with the exhaustive sum
@pytest.mark.parametrize("dims", REF_SHAPES)
@pytest.mark.parametrize("rank", [1, 2, 5])
def test_reference_sweep(oracle, dims, rank):
    x = oracle.gen_tensor(dims, 17)
    f = oracle.kruskal_random(dims, rank, 23)[0]
    for mode in range(len(dims)):
        want = oracle.mttkrp(x, dims, f, mode)
        for algo, order in algos_for(mode, len(dims)):
            for threads in (1, 4):
                got = run(x, dims, f, mode, algo, order, threads).m
                assert rel(got, want) <= TOL, (dims, rank, mode, algo, order)


# shapes that take the TMA + DMMA streaming path (even strides), ragged tiles,
# every rank class of the kernel (C % 8 tails 0/1/2/4 and padded ones)
TC_SHAPES = [(10, 12, 14), (16, 18, 20), (130, 66, 34), (30, 20, 10, 8), (8, 6, 4, 6, 8), (2, 250, 4), (64, 2, 96),
             (6, 10, 4, 2, 2, 4)]


@pytest.mark.parametrize("dims", TC_SHAPES)
@pytest.mark.parametrize("rank", [1, 3, 8, 16, 20, 25, 29, 32, 50, 64])
def test_tc_path_parity(oracle, dims, rank):
    x = oracle.uniform(1234 + rank, int(np.prod(dims))) * 2.0 - 1.0
    f = [m * 2.0 - 1.0 for m in oracle.gen_factors(dims, rank, 99)]
    for mode in range(len(dims)):
        want = oracle.mttkrp(x, dims, f, mode)
        for algo, order in algos_for(mode, len(dims)):
            got = run(x, dims, f, mode, algo, order).m
            assert rel(got, want) <= TOL, (dims, rank, mode, algo, order, rel(got, want))


def test_large_rank_generic_path(oracle):
    dims = (6, 8, 10)
    x = oracle.gen_tensor(dims, 3)
    f = oracle.gen_factors(dims, 70, 4)
    for mode in range(3):
        want = oracle.mttkrp(x, dims, f, mode)
        for algo, order in algos_for(mode, 3):
            assert rel(run(x, dims, f, mode, algo, order).m, want) <= TOL


# test_mttkrp.cpp:153-158
def test_choose_order():
    assert dg.choose_order((20, 30, 40), 1) == O.right
    assert dg.choose_order((40, 30, 20), 1) == O.left
    assert dg.choose_order((5, 3, 5), 1) == O.right
    assert dg.choose_order((2, 3, 4, 5), 2) == O.left


# test_mttkrp.cpp:160-173
def test_two_step_refuses_boundary(oracle):
    dims = (3, 4, 5)
    x = oracle.gen_tensor(dims, 2)
    f = oracle.kruskal_random(dims, 2, 3)[0]
    for mode in (0, 2):
        with pytest.raises(dg.InvalidArgument, match="boundary"):
            run(x, dims, f, mode, A.two_step)
    want = oracle.mttkrp(x, dims, f, 0)
    assert rel(run(x, dims, f, 0, A.automatic).m, want) <= TOL


# test_mttkrp.cpp:191-218: vectors and matrices
def test_vector_and_matrix(oracle):
    xv = oracle.gen_tensor((7,), 4)
    fv = oracle.kruskal_random((7,), 3, 5)[0]
    for algo in (A.baseline, A.one_step):
        m = run(xv, (7,), fv, 0, algo).m
        assert np.allclose(m, np.repeat(xv[:, None], 3, axis=1), rtol=1e-14, atol=0)
    xm = oracle.gen_tensor((3, 4), 6)
    fm = oracle.kruskal_random((3, 4), 2, 7)[0]
    for mode in range(2):
        want = oracle.mttkrp(xm, (3, 4), fm, mode)
        for algo in (A.baseline, A.one_step):
            assert rel(run(xm, (3, 4), fm, mode, algo).m, want) <= TOL


# test_mttkrp.cpp:220-243 + determinism of the deterministic slot reduction
def test_bitwise_repeatable(oracle):
    dims = (6, 5, 4, 3)
    x = oracle.gen_tensor(dims, 44)
    f = oracle.kruskal_random(dims, 4, 45)[0]
    t = dg.DenseTensor(dims, x)
    for mode in range(4):
        for algo, order in algos_for(mode, 4):
            a = dg.mttkrp(dg.MttkrpRequest(t, f, mode, algo, order, 1)).m
            b = dg.mttkrp(dg.MttkrpRequest(t, f, mode, algo, order, 8)).m
            assert np.array_equal(a, b)


# test_mttkrp.cpp:245-274
def test_timing_categories(oracle):
    dims = (5, 6, 7)
    x = oracle.gen_tensor(dims, 3)
    f = oracle.kruskal_random(dims, 3, 4)[0]
    base = run(x, dims, f, 1, A.baseline).time
    assert base["krp_partial"] == 0.0 and base["matvec"] == 0.0 and base["reduce"] == 0.0
    assert base["reorder"] > 0.0 and base["krp_full"] > 0.0
    assert run(x, dims, f, 0, A.baseline).time["reorder"] == 0.0
    one = run(x, dims, f, 1, A.one_step).time
    assert one["matvec"] == 0.0 and one["reorder"] == 0.0 and one["krp_full"] == 0.0
    assert one["krp_partial"] > 0.0
    two = run(x, dims, f, 1, A.two_step).time
    assert two["krp_full"] == 0.0 and two["reduce"] == 0.0 and two["reorder"] == 0.0
    assert two["matvec"] > 0.0
    assert one["total"] > 0.0 and base["total"] >= 0.0


# test_mttkrp.cpp:276-306
def test_requests_are_validated(oracle):
    dims = (3, 4)
    x = oracle.gen_tensor(dims, 1)
    f = oracle.kruskal_random(dims, 2, 2)[0]
    with pytest.raises(dg.InvalidArgument):
        dg.mttkrp(dg.MttkrpRequest(None, f, 0, A.one_step))
    with pytest.raises(dg.OutOfRange):
        run(x, dims, f, 2, A.one_step)
    with pytest.raises(dg.InvalidArgument, match="factors for an order-2"):
        run(x, dims, f[:1], 0, A.one_step)
    with pytest.raises(dg.InvalidArgument, match="rows, mode extent"):
        run(x, dims, [f[0], np.zeros((5, 2))], 0, A.one_step)
    with pytest.raises(dg.InvalidArgument, match="has rank 3, expected 2"):
        run(x, dims, [f[0], np.zeros((4, 3))], 0, A.one_step)
    with pytest.raises(dg.InvalidArgument, match="threads"):
        run(x, dims, f, 0, A.one_step, threads=0)


# test_mttkrp.cpp:308-325
def test_fault_hook_perturbs_one_entry(oracle, monkeypatch):
    dims = (3, 4, 5)
    x = oracle.gen_tensor(dims, 12)
    f = oracle.kruskal_random(dims, 2, 13)[0]
    clean = run(x, dims, f, 0, A.one_step).m
    monkeypatch.setenv("DMTK_INJECT_FAULT", "1")
    faulty = run(x, dims, f, 0, A.one_step).m
    monkeypatch.delenv("DMTK_INJECT_FAULT")
    assert faulty[0, 0] != clean[0, 0]
    mask = np.ones_like(clean, dtype=bool)
    mask[0, 0] = False
    assert np.array_equal(faulty[mask], clean[mask])


def test_matches_reference_library(oracle, ref):
    """Same bytes through the unmodified reference (oracle/_ref) and the GPU."""
    dims = (24, 18, 12, 10)
    x = ref.gen_tensor(dims, 7)
    f = ref.gen_factors(dims, 25, 8)
    for mode in range(4):
        for algo, order in algos_for(mode, 4):
            want = ref.mttkrp(x, dims, f, mode, algo.name, order.name, threads=4)
            got = run(x, dims, f, mode, algo, order).m
            assert rel(got, want) <= TOL


def test_device_resident_entry_point(oracle):
    import torch
    dims = (40, 30, 20)
    x = oracle.gen_tensor(dims, 1)
    f = oracle.gen_factors(dims, 16, 2)
    xd = torch.from_numpy(x).cuda()
    fd = [torch.from_numpy(m).cuda() for m in f]
    t = dg.DenseTensor.from_device(dims, xd.data_ptr(), owner=xd)
    for mode in range(3):
        out = torch.empty((dims[mode], 16), dtype=torch.float64, device="cuda")
        dg.mttkrp_device(t, [m.data_ptr() for m in fd], 16, mode, A.automatic, O.automatic, out.data_ptr(),
                         torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        assert rel(out.cpu().numpy(), oracle.mttkrp(x, dims, f, mode)) <= TOL


@pytest.mark.slow
def test_config1_200cube(oracle):
    """BASELINE config 1: 200^3 U[0,1), C=16, every mode, 1-step and 2-step."""
    dims = (200, 200, 200)
    x = oracle.gen_tensor(dims, 1)
    f = oracle.gen_factors(dims, 16, 2)
    t = dg.DenseTensor(dims, x)
    for mode in range(3):
        want = oracle.mttkrp(x, dims, f, mode)
        for algo, order in algos_for(mode, 3):
            got = dg.mttkrp(dg.MttkrpRequest(t, f, mode, algo, order)).m
            assert rel(got, want) <= TOL, (mode, algo, order, rel(got, want))
