"""Multi-rank host logic of the sharded path (paper_1708_08976_b200.distributed)
on CPU: world_size 2 over gloo, the per-rank compute replaced by the C oracle
so the sharding, the uneven splits and every collective are exercised without
a GPU (the B200 run uses the same driver with GpuBackend over NCCL)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1708_08976_b200.distributed import Backend, dist_cp_als, dist_mttkrp, shard_bounds, shard_slab


class OracleBackend(Backend):
    def __init__(self):
        from oracle_bindings import Oracle
        self.o = Oracle()

    def mttkrp(self, slab, slab_dims, factors, mode):
        return self.o.mttkrp(slab, slab_dims, factors, mode)

    def gram(self, u):
        return self.o.gram_hadamard([u], -1)

    def solve(self, h, m):
        return self.o.solve_psd(h, m)[0]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, dims, C, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from oracle_bindings import Oracle
        o = Oracle()
        x = o.gen_tensor(dims, 5)
        f = o.gen_factors(dims, C, 6)
        slab = np.ascontiguousarray(shard_slab(x, dims, world, rank))
        be = OracleBackend()
        dev = torch.device("cpu")
        ms = [dist_mttkrp(be, slab, dims, f, m, dev) for m in range(len(dims))]
        res = dist_cp_als(be, slab, dims, 3, 6, 0.0, 11, dev)
        if rank == 0:
            q.put(("ok", [m for m in ms], res.fits, [u for u in res.factors], res.tensor_norm))
        dist.destroy_process_group()
    except Exception as e:  # surface worker failures to the test
        q.put(("err", repr(e)))


@pytest.mark.parametrize("dims,C", [((6, 5, 7), 4), ((4, 3, 2, 5), 3)])
def test_two_rank_sharded_mttkrp_and_als(oracle, dims, C):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, dims, C, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
    assert out[0] == "ok", out
    _, ms, fits, factors, norm = out
    x = oracle.gen_tensor(dims, 5)
    f = oracle.gen_factors(dims, C, 6)
    for m in range(len(dims)):
        want = oracle.mttkrp(x, dims, f, m)
        assert np.linalg.norm(ms[m] - want) / np.linalg.norm(want) <= 1e-12
    _, _, want_fits, _ = oracle.cp_als(x, dims, 3, 6, 0.0, 11)
    assert np.max(np.abs(np.array(fits) - want_fits)) <= 1e-9
    assert abs(norm - oracle.tensor_norm(x)) <= 1e-12 * norm
    for u in factors:
        assert np.allclose(np.linalg.norm(u, axis=0), 1.0, rtol=1e-12)


def test_shard_bounds_uneven():
    for extent, world in [(180, 8), (100, 8), (80, 8), (5, 2), (3, 4)]:
        spans = [shard_bounds(extent, world, r) for r in range(world)]
        assert spans[0][0] == 0 and spans[-1][1] == extent
        assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
        sizes = [h - lo for lo, h in spans]
        assert max(sizes) - min(sizes) <= 1
