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
def test_device_sharded_cp_als_world1(group, oracle, dims, C):
    """dmtk_gpu_cp_als_sharded with a library-owned NCCL communicator (world 1
    here): every exchange point (MTTKRP partials, the last factor's column
    norms and Gram, the fit's inner product, ||X||^2) runs as an NCCL
    all-reduce inside the per-mode CUDA graphs; with one rank the result must
    equal the single-GPU cp_als and the reference."""
    import paper_1708_08976_b200 as dg
    from paper_1708_08976_b200.distributed import DeviceComm, dist_cp_als_device

    x = oracle.gen_tensor(dims, 5)
    t = dg.DenseTensor(dims, x)
    comm = DeviceComm(0)
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
