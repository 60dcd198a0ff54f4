"""Multi-GPU MTTKRP / CP-ALS: the tensor sharded along its last (slowest) mode.

One process per GPU (torch.distributed for the plumbing, NCCL for the data).
Rank r owns the contiguous last-mode range [lo_r, hi_r) -- in the natural
layout that is one contiguous slab, itself a valid N-way tensor
(SURVEY.md §8e). Per mode n of an MTTKRP:

  n <  N-1   every rank computes the I_n x C partial over its slab; one
             all-reduce (sum) makes M identical everywhere.
  n == N-1   rows are disjoint: rank r holds M[lo_r:hi_r]; no exchange.

CP-ALS (dmtk_gpu_cp_als_sharded) keeps U_0..U_{N-2} replicated and U_{N-1}
row-sharded: the Gram of U_{N-1}, its column norms and the fit's inner product
are all-reduced (C x C, C and 1 doubles) inside the per-mode CUDA graphs; the
other solves run redundantly and bit-identically on every rank because their
inputs are identical (reference cp_als.cpp:122-158).

Communicators:
  DeviceComm      the production NCCL communicator (one process per GPU).
  loopback_comms  P virtual ranks on ONE device (dmtk_gpu_comm_loopback), each
                  driven by its own host thread: the same sharded code path,
                  so the multi-rank exchanges are tested on a single B200.
"""
from __future__ import annotations

import threading
from dataclasses import dataclass
from typing import List, Sequence

import numpy as np


def shard_bounds(extent: int, world: int, rank: int):
    """Balanced contiguous split of the last mode (first extent % world shards
    one longer), so 180/8 and 100/8 split evenly within one row."""
    q, r = divmod(extent, world)
    lo = rank * q + min(rank, r)
    return lo, lo + q + (1 if rank < r else 0)


def shard_slab(x_full: np.ndarray, dims: Sequence[int], world: int, rank: int) -> np.ndarray:
    """Rank's contiguous slab of a naturally ordered host tensor (a view)."""
    lo, hi = shard_bounds(dims[-1], world, rank)
    plane = int(np.prod(dims[:-1], dtype=np.int64))
    return x_full[lo * plane:hi * plane]


def gather_rows(local: np.ndarray, extent: int, world: int):
    """All-gather of uneven last-mode row shards (the sharded last factor /
    last-mode MTTKRP) over the default torch.distributed group, padded to the
    largest shard; returns the full extent x C matrix on every rank."""
    import torch
    import torch.distributed as dist
    dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend() == "nccl" else torch.device("cpu")
    cols = local.shape[1]
    width = -(-extent // world)
    buf = torch.zeros((width, cols), dtype=torch.float64, device=dev)
    buf[:local.shape[0]] = torch.from_numpy(np.ascontiguousarray(local)).to(dev)
    out = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(out, buf)
    rows = []
    for r in range(world):
        lo, hi = shard_bounds(extent, world, r)
        rows.append(out[r][:hi - lo].cpu().numpy())
    return np.concatenate(rows, axis=0)


def _check(lib, rc):
    if rc != 0:
        raise RuntimeError(lib.dmtk_gpu_last_error().decode())


def _lib():
    from . import _lib as L
    return L


# ------------------------------------------------------------ communicators
class _CommOps:
    """Exchange queries shared by both communicator kinds."""

    @property
    def fused(self) -> bool:
        """True when the exchanges run over peer memory (csrc/xrank.cu)."""
        C = self._C
        r, w, f = C.c_int(), C.c_int(), C.c_int()
        _check(self._lib, self._lib.dmtk_gpu_comm_info(self.handle, C.byref(r), C.byref(w), C.byref(f)))
        return bool(f.value)

    def mttkrp(self, slab, device_factor_ptrs, rank: int, mode: int, device_out_ptr: int, stream: int = 0,
               algo: int = 3, order: int = 0):
        """dmtk_gpu_mttkrp_sharded: this rank's slab; modes < N-1 return the
        full result summed over the ranks (fused into the MTTKRP's slot
        reduction with the peer exchange), the last mode this rank's rows.
        algo/order: MttkrpAlgo / TwoStepOrder values (default automatic)."""
        C = self._C
        arr = (C.c_void_p * len(device_factor_ptrs))(*[C.c_void_p(p) for p in device_factor_ptrs])
        _check(self._lib, self._lib.dmtk_gpu_mttkrp_sharded(self.handle, slab.handle(), arr, int(rank), int(mode),
                                                            int(algo), int(order), C.c_void_p(device_out_ptr),
                                                            C.c_void_p(stream or None)))

    def allreduce(self, device_ptr: int, n: int, stream: int = 0):
        """In-place sum of n doubles at device_ptr over the ranks
        (dmtk_gpu_comm_allreduce); rank-order sum with the peer exchange."""
        _check(self._lib, self._lib.dmtk_gpu_comm_allreduce(self.handle, self._C.c_void_p(device_ptr), int(n),
                                                            self._C.c_void_p(stream or None)))


class DeviceComm(_CommOps):
    """An NCCL communicator owned by the library (dmtk_gpu_comm_*): rank 0
    makes the 128-byte id, torch.distributed broadcasts it, every rank joins
    on its device. The library then all-reduces on its own stream, inside the
    CP-ALS per-mode CUDA graphs."""

    def __init__(self, device: int = 0, lib=None):
        import ctypes as C
        import torch.distributed as dist
        self._lib = lib or _lib().lib
        self._C = C
        world, rank = dist.get_world_size(), dist.get_rank()
        buf = (C.c_ubyte * 128)()
        if rank == 0:
            _check(self._lib, self._lib.dmtk_gpu_comm_unique_id(buf))
        obj = [bytes(buf)]
        dist.broadcast_object_list(obj, src=0)
        buf = (C.c_ubyte * 128).from_buffer_copy(obj[0])
        self.handle = C.c_void_p()
        _check(self._lib, self._lib.dmtk_gpu_comm_init(buf, rank, world, device, C.byref(self.handle)))
        self.rank, self.world, self.device = rank, world, device

    def close(self):
        if self.handle:
            self._lib.dmtk_gpu_comm_free(self.handle)
            self.handle = self._C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:  # pragma: no cover - interpreter shutdown
            pass


class LoopbackComm(_CommOps):
    """Rank `rank` of a loopback group (dmtk_gpu_comm_loopback)."""

    def __init__(self, handle, rank: int, world: int, device: int):
        import ctypes as C
        self._lib = _lib().lib
        self._C = C
        self.handle, self.rank, self.world, self.device = handle, rank, world, device

    def close(self):
        if self.handle:
            self._lib.dmtk_gpu_comm_free(self.handle)
            self.handle = self._C.c_void_p()


def loopback_comms(world: int, device: int = 0) -> List[LoopbackComm]:
    """`world` virtual ranks on one device (tests of the sharded path)."""
    import ctypes as C
    lib = _lib().lib
    hs = (C.c_void_p * world)()
    _check(lib, lib.dmtk_gpu_comm_loopback(world, device, hs))
    return [LoopbackComm(C.c_void_p(hs[k]), k, world, device) for k in range(world)]


# ------------------------------------------------ device-resident sharded CP-ALS
@dataclass
class ShardedAlsResult:
    factors: List[np.ndarray]  # modes 0..N-2 in full, then this rank's rows of mode N-1
    lambda_: np.ndarray
    fits: List[float]
    iter_seconds: List[float]
    tensor_norm: float
    zero_tensor: bool


def dist_cp_als_device(slab_tensor, comm, global_last: int, last_lo: int, config, lib=None) -> ShardedAlsResult:
    """The reference's cp_als (cp_als.cpp:122-200) over last-mode shards with
    the whole loop on the device (dmtk_gpu_cp_als_sharded): slab_tensor is this
    rank's DenseTensor (last-mode rows [last_lo, last_lo + its extent) of a
    tensor whose last extent is global_last); comm a DeviceComm or a
    LoopbackComm; config an api.AlsConfig (dimension_tree selects the tree)."""
    import ctypes as C
    L = _lib()
    lib = lib or L.lib
    dims = slab_tensor.dims
    rank = int(config.rank)
    cfg = L.AlsConfig(rank, config.max_iters, config.tol, config.seed, config.threads, int(config.algo),
                      int(config.order), int(bool(getattr(config, "dimension_tree", False))))
    f = np.zeros(int(sum(dims)) * max(rank, 1))
    lam = np.zeros(max(rank, 1))
    cap = max(int(config.max_iters), 1)
    fits = np.zeros(cap)
    secs = np.zeros(cap)
    k = C.c_int(0)
    zero = C.c_int(0)
    norm = np.zeros(1)
    dp = lambda a: a.ctypes.data_as(L.dp)  # noqa: E731
    _check(lib, lib.dmtk_gpu_cp_als_sharded(slab_tensor.handle(), comm.handle, int(global_last), int(last_lo),
                                            C.byref(cfg), dp(f), dp(lam), dp(fits), dp(secs), None, C.byref(k),
                                            C.byref(zero), dp(norm)))
    factors, off = [], 0
    for d in dims:
        factors.append(f[off:off + d * rank].reshape(d, rank).copy())
        off += d * rank
    return ShardedAlsResult(factors, lam[:rank].copy(), list(fits[:k.value]), list(secs[:k.value]), float(norm[0]),
                            bool(zero.value))


def loopback_cp_als(tensor, world: int, config, packed: bool = False, comms=None):
    """dmtk_gpu_cp_als_sharded over `world` loopback ranks of one device: the
    tensor is cut into its last-mode slabs (dmtk_gpu_tensor_slab), every rank
    runs the production sharded sweep in its own thread, and the exchanges go
    through the loopback all-reduce. packed: each rank packs its slab's
    symmetric slices (dmtk_gpu_tensor_pack_sym01) first. Returns the per-rank
    results and the full last factor assembled from the ranks' rows."""
    dims = tensor.dims
    own = comms is None
    if own:
        comms = loopback_comms(world, tensor.device)
    slabs, spans = [], []
    for r in range(world):
        lo, hi = shard_bounds(dims[-1], world, r)
        s = tensor.slab(lo, hi)
        if packed:
            p = s.pack_symmetric01()
            s.release()
            s = p
        slabs.append(s)
        spans.append((lo, hi))
    results: List = [None] * world
    errors: List = [None] * world

    def run(r):
        try:
            results[r] = dist_cp_als_device(slabs[r], comms[r], dims[-1], spans[r][0], config)
        except Exception as e:  # surfaced below
            errors[r] = e

    threads = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    for s in slabs:
        s.release()
    if own:
        for c in comms:
            c.close()
    for e in errors:
        if e is not None:
            raise e
    last = np.concatenate([res.factors[-1] for res in results], axis=0)
    return results, last
