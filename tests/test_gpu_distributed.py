"""The sharded driver (paper_1708_08976_b200.distributed) with the B200
backend (GpuBackend, the C ABI) in a real process group: world_size 1 here
(one GPU per gpurun box), so the GPU backend, the shard plumbing and the
collectives' code paths run on the device; the multi-rank exchanges are
covered by tests/test_distributed_gloo.py on CPU."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist

from paper_1708_08976_b200.distributed import GpuBackend, dist_cp_als, dist_mttkrp, shard_slab

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


@pytest.mark.parametrize("dims,C", [((6, 5, 7), 4), ((9, 3, 4, 5), 3), ((20, 18, 16), 9)])
def test_gpu_backend_sharded_mttkrp_and_als(group, oracle, dims, C):
    x = oracle.gen_tensor(dims, 5)
    f = oracle.gen_factors(dims, C, 6)
    slab = np.ascontiguousarray(shard_slab(x, dims, 1, 0))
    be = GpuBackend(0)
    dev = torch.device("cuda", 0)
    for m in range(len(dims)):
        got = dist_mttkrp(be, slab, dims, f, m, dev)
        want = oracle.mttkrp(x, dims, f, m)
        assert np.linalg.norm(got - want) <= 1e-12 * np.linalg.norm(want)
    res = dist_cp_als(be, slab, dims, 3, 6, 0.0, 11, dev)
    _, _, want_fits, _ = oracle.cp_als(x, dims, 3, 6, 0.0, 11)
    assert np.max(np.abs(np.array(res.fits) - want_fits)) <= 1e-9


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
