"""The production sharded CP-ALS (dmtk_gpu_cp_als_sharded) on one B200.

* NCCL communicator in a real process group at world size 1 (one GPU per
  gpurun box): every exchange point runs as an NCCL all-reduce inside the
  per-mode CUDA graphs;
* loopback communicators (dmtk_gpu_comm_loopback): P = 2, 3, 8 virtual ranks
  of one device, each in its own host thread, the tensor cut into uneven
  last-mode slabs -- the multi-rank exchanges of the same code path (partials,
  the sharded last factor's norms and Gram, the fit's inner product, ||X||^2,
  the tree's left partial and right-half multi-TTVs, the packed Q), checked
  against the single-GPU cp_als and the reference. The reference's analogue is
  its thread-count invariance (test_mttkrp.cpp:220-243, test_krp.cpp:83-91).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist

from paper_1708_08976_b200.distributed import loopback_cp_als, shard_bounds

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.fixture(scope="module")
def group():
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_port())
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    yield
    dist.destroy_process_group()


@pytest.mark.parametrize("dims,C", [((6, 5, 7), 4), ((9, 3, 4, 5), 3), ((40, 40, 12, 8), 20)])
@pytest.mark.parametrize("exchange", ["xrank", "nccl"])
def test_device_sharded_cp_als_world1(group, oracle, dims, C, exchange):
    """dmtk_gpu_cp_als_sharded with a library-owned NCCL communicator (world 1
    here): every exchange point (MTTKRP partials, the last factor's column
    norms and Gram, the fit's inner product, ||X||^2) runs inside the per-mode
    CUDA graphs, as the fused peer-memory exchange kernel (the real, one-rank
    launch of csrc/xrank.cu: the partials' slot reduction is the exchange) or
    as an NCCL all-reduce (DMTK_GPU_XRANK=0); with one rank the result must
    equal the single-GPU cp_als and the reference."""
    import paper_1708_08976_b200 as dg
    from paper_1708_08976_b200.distributed import DeviceComm, dist_cp_als_device

    x = oracle.gen_tensor(dims, 5)
    t = dg.DenseTensor(dims, x)
    if exchange == "nccl":
        os.environ["DMTK_GPU_XRANK"] = "0"
    try:
        comm = DeviceComm(0)
    finally:
        os.environ.pop("DMTK_GPU_XRANK", None)
    assert comm.fused == (exchange == "xrank")
    cfg = dg.AlsConfig(rank=C, max_iters=8, tol=0.0, seed=11)
    res = dist_cp_als_device(t, comm, dims[-1], 0, cfg)
    one = dg.cp_als(t, cfg)
    want = [it.fit.fit for it in one.trace.iters]
    assert len(res.fits) == len(want) == 8
    assert np.max(np.abs(np.array(res.fits) - np.array(want))) <= 1e-12
    for a, b in zip(res.factors, one.model.factors):
        assert np.linalg.norm(a - b) <= 1e-12 * np.linalg.norm(b)
    _, _, ref_fits, _ = oracle.cp_als(x, dims, C, 8, 0.0, 11)
    assert np.max(np.abs(np.array(res.fits) - ref_fits)) <= 1e-9
    comm.close()


def test_device_sharded_cp_als_validation(group, oracle):
    import paper_1708_08976_b200 as dg
    from paper_1708_08976_b200.distributed import DeviceComm, dist_cp_als_device

    dims = (6, 5, 7)
    t = dg.DenseTensor(dims, oracle.gen_tensor(dims, 5))
    comm = DeviceComm(0)
    with pytest.raises(RuntimeError, match="outside the global extent"):
        dist_cp_als_device(t, comm, 7, 3, dg.AlsConfig(rank=2, max_iters=2, tol=0.0))
    comm.close()


def _sym_slab(dg, oracle):
    dims = (4, 4, 3, 6)
    x = oracle.gen_tensor(dims, 9).reshape(dims[::-1])
    x = x + np.swapaxes(x, -1, -2)  # symmetric in modes 0 and 1
    return dg.DenseTensor(dims, np.ascontiguousarray(x).reshape(-1)).pack_symmetric01()


@pytest.mark.parametrize("dims,C", [((9, 3, 4, 5), 3), ((40, 40, 12, 8), 20), ((6, 5, 7, 4, 3), 4)])
def test_device_sharded_cp_als_dimension_tree_world1(group, oracle, dims, C):
    """The dimension-tree sweep over last-mode shards (left partial all-reduced,
    right-half multi-TTVs of the non-last modes all-reduced, the last factor's
    rows local): with one rank, equal to the single-GPU tree and within 1e-9 of
    the reference's per-mode fits."""
    import paper_1708_08976_b200 as dg
    from paper_1708_08976_b200.distributed import DeviceComm, dist_cp_als_device

    x = oracle.gen_tensor(dims, 5)
    t = dg.DenseTensor(dims, x)
    comm = DeviceComm(0)
    cfg = dg.AlsConfig(rank=C, max_iters=6, tol=0.0, seed=11, dimension_tree=True)
    res = dist_cp_als_device(t, comm, dims[-1], 0, cfg)
    one = dg.cp_als(t, cfg)
    want = [it.fit.fit for it in one.trace.iters]
    assert np.max(np.abs(np.array(res.fits) - np.array(want))) <= 1e-12
    _, _, ref_fits, _ = oracle.cp_als(x, dims, C, 6, 0.0, 11)
    assert np.max(np.abs(np.array(res.fits) - ref_fits)) <= 1e-9
    comm.close()


def test_device_sharded_cp_als_symmetric_packed_world1(group, oracle):
    """A packed symmetric slab (modes 0/1): Q over the pair index all-reduced,
    the right half as in the tree; with one rank equal to the single-GPU
    packed sweep."""
    import paper_1708_08976_b200 as dg
    from paper_1708_08976_b200.distributed import DeviceComm, dist_cp_als_device

    tp = _sym_slab(dg, oracle)
    comm = DeviceComm(0)
    cfg = dg.AlsConfig(rank=3, max_iters=6, tol=0.0, seed=11)
    res = dist_cp_als_device(tp, comm, 6, 0, cfg)
    one = dg.cp_als(tp, cfg)
    want = [it.fit.fit for it in one.trace.iters]
    assert np.max(np.abs(np.array(res.fits) - np.array(want))) <= 1e-12
    comm.close()


def _assemble(results):
    return np.concatenate([r.factors[-1] for r in results], axis=0)


@pytest.mark.timeout(300)
@pytest.mark.parametrize("dims,C,P", [((6, 5, 7), 4, 2), ((6, 5, 7), 4, 3), ((9, 3, 4, 5), 3, 2),
                                      ((9, 3, 4, 5), 3, 3), ((20, 18, 17), 9, 8), ((40, 40, 12, 8), 20, 3),
                                      ((40, 40, 12, 8), 20, 8), ((12, 10, 9, 6, 11), 5, 3)])
@pytest.mark.parametrize("tree", [False, True])
def test_loopback_sharded_cp_als(oracle, ref, dims, C, P, tree):
    """P ranks (uneven splits: 7/2, 7/3, 17/8, 11/3) of the production sharded
    sweep equal the single-GPU sweep (fits 1e-12, factors 1e-10) and the
    reference's cp_als (fits 1e-9)."""
    import paper_1708_08976_b200 as dg
    x = oracle.gen_tensor(dims, 5)
    t = dg.DenseTensor(dims, x)
    iters = 6
    cfg = dg.AlsConfig(rank=C, max_iters=iters, tol=0.0, seed=11, dimension_tree=tree)
    res, last = loopback_cp_als(t, P, cfg)
    one = dg.cp_als(t, cfg)
    want = np.array([it.fit.fit for it in one.trace.iters])
    for r in res:
        assert len(r.fits) == iters
        assert np.max(np.abs(np.array(r.fits) - want)) <= 1e-12
        assert abs(r.tensor_norm - one.trace.tensor_norm) <= 1e-12 * one.trace.tensor_norm
        for a, b in zip(r.factors[:-1], one.model.factors[:-1]):  # replicated factors
            assert np.linalg.norm(a - b) <= 1e-10 * np.linalg.norm(b)
        assert np.array_equal(r.factors[0], res[0].factors[0])  # identical on every rank
    assert np.linalg.norm(last - one.model.factors[-1]) <= 1e-10 * np.linalg.norm(one.model.factors[-1])
    rf = ref.cp_als(x, dims, C, iters, tol=0.0, seed=11)
    assert np.max(np.abs(np.array(res[0].fits) - rf["fits"])) <= 1e-9


@pytest.mark.timeout(300)
@pytest.mark.parametrize("P", [2, 3])
def test_loopback_sharded_cp_als_symmetric_packed(oracle, ref, P):
    """Each rank packs its slab's symmetric slices; Q over the pair index is
    summed over the ranks; fits equal the single-GPU packed sweep and the
    reference's CP-ALS on the full tensor."""
    import paper_1708_08976_b200 as dg
    dims = (6, 6, 4, 7)
    x = oracle.gen_tensor(dims, 9).reshape(dims[::-1])
    x = np.ascontiguousarray(x + np.swapaxes(x, -1, -2)).reshape(-1)
    t = dg.DenseTensor(dims, x)
    cfg = dg.AlsConfig(rank=3, max_iters=6, tol=0.0, seed=11)
    res, last = loopback_cp_als(t, P, cfg, packed=True)
    tp = t.pack_symmetric01()
    one = dg.cp_als(tp, cfg)
    want = np.array([it.fit.fit for it in one.trace.iters])
    for r in res:
        assert np.max(np.abs(np.array(r.fits) - want)) <= 1e-12
    rf = ref.cp_als(x, dims, 3, 6, tol=0.0, seed=11)
    assert np.max(np.abs(np.array(res[0].fits) - rf["fits"])) <= 1e-9


def test_sharded_mttkrp_partials_sum_to_full(oracle):
    """The bench's sharded MTTKRP: per-slab results of modes < N-1 summed over
    the slabs (the all-reduce) and the last mode's rows concatenated equal the
    full tensor's MTTKRP (1e-12)."""
    import paper_1708_08976_b200 as dg
    dims, C, P = (30, 20, 17), 9, 3
    x = oracle.gen_tensor(dims, 3)
    f = oracle.gen_factors(dims, C, 4)
    t = dg.DenseTensor(dims, x)
    for m in range(3):
        want = oracle.mttkrp(x, dims, f, m)
        parts = []
        for r in range(P):
            lo, hi = shard_bounds(dims[-1], P, r)
            s = t.slab(lo, hi)
            assert np.array_equal(s.download(), x[lo * 600:hi * 600])
            parts.append(dg.mttkrp(dg.MttkrpRequest(s, f[:-1] + [f[-1][lo:hi]], m)).m)
            s.release()
        got = np.concatenate(parts) if m == 2 else sum(parts)
        assert np.linalg.norm(got - want) <= 1e-12 * np.linalg.norm(want)


def test_slab_validation(oracle):
    import paper_1708_08976_b200 as dg
    t = dg.DenseTensor((4, 5, 6), oracle.gen_tensor((4, 5, 6), 1))
    with pytest.raises(dg.OutOfRange):
        t.slab(4, 7)
    with pytest.raises(dg.OutOfRange):
        t.slab(3, 3)


def _run_ranks(P, fn):
    import threading
    errs = [None] * P

    def go(r):
        try:
            fn(r)
        except Exception as e:  # surfaced below
            errs[r] = e

    ts = [threading.Thread(target=go, args=(r,)) for r in range(P)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    for e in errs:
        if e is not None:
            raise e


@pytest.mark.timeout(300)
@pytest.mark.parametrize("P", [1, 2, 3, 8, 16])
def test_loopback_fused_exchange_allreduce(P):
    """The fused peer-memory exchange (csrc/xrank.cu) through
    dmtk_gpu_comm_allreduce on P loopback ranks (all ranks in one cooperative
    launch): every rank gets the rank-order sum, bitwise equal to the left fold
    b_0 + b_1 + ... + b_{P-1} on the host and the same on every rank; sizes from
    1 to above the receive capacity (chunked), each exchanged three times in a
    row (epoch parity reuse of the receive rows)."""
    from paper_1708_08976_b200.distributed import loopback_comms
    comms = loopback_comms(P)
    try:
        assert all(c.fused for c in comms)
        sizes = [1, 7, 1000, 20000, (1 << 18) + 5]
        g = torch.Generator().manual_seed(P)
        host = [[torch.randn(n, dtype=torch.float64, generator=g) for n in sizes] for _ in range(P)]
        dev = [[h.cuda() for h in row] for row in host]
        torch.cuda.synchronize()
        rounds = 3

        def work(r):
            for _ in range(rounds):
                for b in dev[r]:
                    comms[r].allreduce(b.data_ptr(), b.numel())

        _run_ranks(P, work)
        torch.cuda.synchronize()
        for i, n in enumerate(sizes):
            want = [host[r][i].numpy().copy() for r in range(P)]
            for _ in range(rounds):
                acc = want[0].copy()
                for r in range(1, P):
                    acc = acc + want[r]
                want = [acc] * P
            for r in range(P):
                got = dev[r][i].cpu().numpy()
                assert np.array_equal(got, want[0]), (P, n, r)
    finally:
        for c in comms:
            c.close()


@pytest.mark.timeout(300)
@pytest.mark.parametrize("dims,C,P,tree", [((40, 40, 12, 8), 20, 3, False), ((20, 18, 17), 9, 8, False),
                                           ((9, 3, 4, 5), 3, 2, True), ((40, 40, 12, 8), 20, 8, True)])
def test_loopback_fused_vs_event_exchange(oracle, dims, C, P, tree):
    """The sharded CP-ALS with the fused exchange (each non-last mode's slot
    reduction sums the ranks' partials in the same kernel) against the
    stream-event all-reduce path (DMTK_GPU_XRANK=0): fits within 1e-12 and
    factors within 1e-12; the fused factors are bitwise identical on every
    rank and bitwise repeatable on a second run over the same communicators
    (the exchange epochs carry over)."""
    import paper_1708_08976_b200 as dg
    from paper_1708_08976_b200.distributed import loopback_comms
    x = oracle.gen_tensor(dims, 5)
    t = dg.DenseTensor(dims, x)
    cfg = dg.AlsConfig(rank=C, max_iters=5, tol=0.0, seed=11, dimension_tree=tree)
    comms = loopback_comms(P)
    try:
        assert all(c.fused for c in comms)
        res, last = loopback_cp_als(t, P, cfg, comms=comms)
        res2, last2 = loopback_cp_als(t, P, cfg, comms=comms)
    finally:
        for c in comms:
            c.close()
    os.environ["DMTK_GPU_XRANK"] = "0"
    try:
        ev = loopback_comms(P)
        assert not any(c.fused for c in ev)
        for c in ev:
            c.close()
        ref_res, ref_last = loopback_cp_als(t, P, cfg)
    finally:
        del os.environ["DMTK_GPU_XRANK"]
    for r in range(P):
        assert np.max(np.abs(np.array(res[r].fits) - np.array(ref_res[r].fits))) <= 1e-12
        for a, b in zip(res[r].factors[:-1], ref_res[r].factors[:-1]):
            assert np.linalg.norm(a - b) <= 1e-12 * np.linalg.norm(b)
        for a, b in zip(res[r].factors, res[0].factors[:-1]):
            assert np.array_equal(a, b)
        for a, b in zip(res[r].factors, res2[r].factors):
            assert np.array_equal(a, b)
        assert res[r].fits == res2[r].fits
    assert np.linalg.norm(last - ref_last) <= 1e-12 * np.linalg.norm(ref_last)
    assert np.array_equal(last, last2)


@pytest.mark.timeout(300)
@pytest.mark.parametrize("dims,C,P", [((30, 20, 17), 9, 3), ((12, 10, 9, 8), 25, 2), ((40, 40, 12, 8), 20, 8),
                                      ((200, 200, 200), 16, 3)])
def test_loopback_mttkrp_sharded(oracle, dims, C, P):
    """dmtk_gpu_mttkrp_sharded on P loopback ranks (the fused peer-memory
    exchange: each non-last mode's slot reduction sums the ranks' partials):
    modes < N-1 give the full MTTKRP on every rank, bitwise the same on all
    ranks and within 1e-12 of the single-device result; the last mode gives
    each rank its rows. Every mode twice in a row (exchange epochs)."""
    import paper_1708_08976_b200 as dg
    from paper_1708_08976_b200.distributed import loopback_comms
    x = oracle.gen_tensor(dims, 3)
    f = oracle.gen_factors(dims, C, 4)
    t = dg.DenseTensor(dims, x)
    N = len(dims)
    want = [dg.mttkrp(dg.MttkrpRequest(t, f, m)).m for m in range(N)]
    comms = loopback_comms(P)
    slabs, outs, facs = [], [], []
    try:
        for r in range(P):
            lo, hi = shard_bounds(dims[-1], P, r)
            slabs.append(t.slab(lo, hi))
            fr = [torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in f[:-1]]
            fr.append(torch.from_numpy(np.ascontiguousarray(f[-1][lo:hi])).cuda())
            facs.append(fr)
            outs.append([torch.zeros((dims[m] if m < N - 1 else hi - lo, C), dtype=torch.float64, device="cuda")
                         for m in range(N)])
        torch.cuda.synchronize()

        def work(r):
            for _ in range(2):
                for m in range(N):
                    comms[r].mttkrp(slabs[r], [a.data_ptr() for a in facs[r]], C, m, outs[r][m].data_ptr())
            torch.cuda.synchronize()

        _run_ranks(P, work)
        torch.cuda.synchronize()
        for m in range(N - 1):
            got0 = outs[0][m].cpu().numpy()
            assert np.linalg.norm(got0 - want[m]) <= 1e-12 * np.linalg.norm(want[m]), m
            for r in range(1, P):
                assert np.array_equal(outs[r][m].cpu().numpy(), got0), (m, r)
        last = np.concatenate([outs[r][N - 1].cpu().numpy() for r in range(P)], axis=0)
        assert np.linalg.norm(last - want[N - 1]) <= 1e-12 * np.linalg.norm(want[N - 1])
    finally:
        for s in slabs:
            s.release()
        for c in comms:
            c.close()


@pytest.mark.parametrize("dims,C", [((30, 20, 17), 9), ((7, 6, 5, 9), 4), ((31, 8, 11), 3)])
def test_slab_is_its_own_extent(oracle, dims, C):
    """A slab holds only its own last-mode rows: the device-resident MTTKRP of
    every mode writes exactly its result rows (a guard band after an
    exactly-sized output stays untouched) and equals the MTTKRP of the slab's
    bytes uploaded as a tensor of its own."""
    import paper_1708_08976_b200 as dg
    from paper_1708_08976_b200 import MttkrpAlgo as A, TwoStepOrder as O
    x = oracle.gen_tensor(dims, 3)
    f = oracle.gen_factors(dims, C, 4)
    t = dg.DenseTensor(dims, x)
    N = len(dims)
    plane = int(np.prod(dims[:-1]))
    for lo, hi in [(0, 2), (2, dims[-1]), (1, dims[-1] - 1)]:
        s = t.slab(lo, hi)
        sd = tuple(dims[:-1]) + (hi - lo,)
        own = dg.DenseTensor(sd, x[lo * plane:hi * plane].copy())
        fr = f[:-1] + [f[-1][lo:hi]]
        dev = [torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in fr]
        for m in range(N):
            rows = sd[m]
            buf = torch.full((rows * C + 64,), 7.25, dtype=torch.float64, device="cuda")
            torch.cuda.synchronize()
            dg.mttkrp_device(s, [a.data_ptr() for a in dev], C, m, A.automatic, O.automatic, buf.data_ptr(), 0)
            torch.cuda.synchronize()
            got = buf.cpu().numpy()
            assert np.all(got[rows * C:] == 7.25), (lo, hi, m)  # nothing past the result
            want = dg.mttkrp(dg.MttkrpRequest(own, fr, m)).m
            assert np.linalg.norm(got[:rows * C].reshape(rows, C) - want) <= 1e-12 * np.linalg.norm(want)
        s.release()
        own.release()


@pytest.mark.parametrize("exchange", ["xrank", "nccl"])
def test_device_mttkrp_sharded_world1(group, oracle, exchange):
    """bench.py's N > 1 MTTKRP path (dmtk_gpu_mttkrp_sharded through a
    library-owned NCCL communicator) at world 1: the fused exchange kernel's
    real one-rank launch, or the NCCL all-reduce; equal to the single-device
    MTTKRP (1e-12) for every mode, twice in a row."""
    import paper_1708_08976_b200 as dg
    from paper_1708_08976_b200.distributed import DeviceComm
    dims, C = (60, 40, 30), 12
    x = oracle.gen_tensor(dims, 3)
    f = oracle.gen_factors(dims, C, 4)
    t = dg.DenseTensor(dims, x)
    if exchange == "nccl":
        os.environ["DMTK_GPU_XRANK"] = "0"
    try:
        comm = DeviceComm(0)
    finally:
        os.environ.pop("DMTK_GPU_XRANK", None)
    assert comm.fused == (exchange == "xrank")
    dev = [torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in f]
    s = torch.cuda.Stream()
    for _ in range(2):
        for m in range(3):
            out = torch.zeros((dims[m], C), dtype=torch.float64, device="cuda")
            torch.cuda.synchronize()
            comm.mttkrp(t, [a.data_ptr() for a in dev], C, m, out.data_ptr(), s.cuda_stream)
            torch.cuda.synchronize()
            want = dg.mttkrp(dg.MttkrpRequest(t, f, m)).m
            assert np.linalg.norm(out.cpu().numpy() - want) <= 1e-12 * np.linalg.norm(want)
    comm.close()
