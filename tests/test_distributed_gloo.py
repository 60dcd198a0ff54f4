"""Multi-rank HOST logic of the sharded path (paper_1708_08976_b200.distributed)
on CPU: world_size 2 over gloo, no GPU.

The device exchanges themselves (dmtk_gpu_cp_als_sharded at P = 2, 3, 8) are
tested on one B200 through loopback communicators
(tests/test_gpu_distributed.py). Here, with two real processes:
* the uneven last-mode split, the slab views and the all-gather of uneven row
  shards that returns the full last factor;
* the communicator bootstrap: rank 0's 128-byte id reaches every rank through
  torch.distributed, each joins with its own rank / world / device;
* the per-rank arguments of the sharded CP-ALS call (global extent, the rank's
  first last-mode row, the config) and the unpacking of its outputs, with the
  C library replaced by a recording stand-in.
"""
import ctypes as C
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1708_08976_b200.distributed import shard_bounds, shard_slab


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class FakeLib:
    """Records the C-ABI calls the Python driver makes (no device)."""

    def __init__(self, rank):
        self.rank = rank
        self.calls = []

    def dmtk_gpu_comm_unique_id(self, buf):
        for k in range(128):
            buf[k] = (k * 7 + 3) % 256
        return 0

    def dmtk_gpu_comm_init(self, buf, rank, world, device, out):
        self.calls.append(("init", bytes(buf), rank, world, device))
        out._obj.value = 1000 + rank
        return 0

    def dmtk_gpu_comm_free(self, h):
        return 0

    def dmtk_gpu_cp_als_sharded(self, t, comm, last_extent, last_lo, cfg, f, lam, fits, secs, msecs, k, zero, norm):
        c = cfg._obj
        self.calls.append(("als", t, comm.value, last_extent, last_lo, c.rank, c.max_iters, c.dimtree))
        n = c.max_iters
        for i in range(n):
            fits[i] = 0.5 + 0.01 * i
            secs[i] = 1e-3
        for e in range(self.ftot):  # the concatenated factors: their flat index
            f[e] = float(e)
        k._obj.value = n
        norm[0] = 3.0
        return 0

    def dmtk_gpu_last_error(self):
        return b"fake"


class FakeTensor:
    def __init__(self, dims):
        self.dims = tuple(dims)

    def handle(self):
        return 77


def _worker(rank, world, port, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_1708_08976_b200 import api
        from paper_1708_08976_b200.distributed import DeviceComm, dist_cp_als_device, gather_rows

        # slabs of an uneven split and the all-gather of uneven row shards
        dims, Cr = (4, 3, 7), 5
        x = np.arange(np.prod(dims), dtype=np.float64)
        slab = shard_slab(x, dims, world, rank)
        lo, hi = shard_bounds(dims[-1], world, rank)
        assert slab.size == (hi - lo) * 12 and slab[0] == lo * 12
        full_last = np.arange(dims[-1] * Cr, dtype=np.float64).reshape(dims[-1], Cr)
        gathered = gather_rows(full_last[lo:hi], dims[-1], world)

        # communicator bootstrap and the sharded call's arguments
        lib = FakeLib(rank)
        comm = DeviceComm(device=rank, lib=lib)
        t = FakeTensor(dims[:-1] + (hi - lo,))
        lib.ftot = sum(t.dims) * Cr
        res = dist_cp_als_device(t, comm, dims[-1], lo, api.AlsConfig(rank=Cr, max_iters=4, tol=0.0, seed=3,
                                                                      dimension_tree=True), lib=lib)
        q.put(("ok", rank, gathered, lib.calls, [f.shape for f in res.factors], res.fits, res.tensor_norm,
               res.factors[-1][0, 0]))
        dist.destroy_process_group()
    except Exception as e:  # surface worker failures to the test
        import traceback
        q.put(("err", rank, traceback.format_exc()))


def test_two_rank_host_logic():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    outs = sorted([q.get(timeout=240) for _ in range(2)], key=lambda o: o[1])
    for p in procs:
        p.join(timeout=60)
    for o in outs:
        assert o[0] == "ok", o
    dims, Cr = (4, 3, 7), 5
    full_last = np.arange(dims[-1] * Cr, dtype=np.float64).reshape(dims[-1], Cr)
    ids = set()
    for _, rank, gathered, calls, shapes, fits, norm, f_last00 in outs:
        assert np.array_equal(gathered, full_last)
        init = [c for c in calls if c[0] == "init"][0]
        ids.add(init[1])
        assert init[2:] == (rank, 2, rank)  # rank, world, device
        als = [c for c in calls if c[0] == "als"][0]
        lo, hi = shard_bounds(7, 2, rank)
        assert als[2] == 1000 + rank and als[3] == 7 and als[4] == lo
        assert als[5:] == (Cr, 4, 1)
        assert shapes == [(4, Cr), (3, Cr), (hi - lo, Cr)]
        assert fits == pytest.approx([0.5, 0.51, 0.52, 0.53]) and norm == 3.0
        assert f_last00 == float((4 + 3) * Cr)  # the last factor starts after modes 0..N-2
    assert len(ids) == 1  # every rank joined with rank 0's id


def test_shard_bounds_uneven():
    for extent, world in [(180, 8), (100, 8), (80, 8), (5, 2), (3, 4)]:
        spans = [shard_bounds(extent, world, r) for r in range(world)]
        assert spans[0][0] == 0 and spans[-1][1] == extent
        assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
        sizes = [h - lo for lo, h in spans]
        assert max(sizes) - min(sizes) <= 1
