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
