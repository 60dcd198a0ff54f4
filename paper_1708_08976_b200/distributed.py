"""Multi-GPU MTTKRP / CP-ALS: the tensor sharded along its last (slowest) mode.

One process per GPU (torch.distributed; NCCL on B200s, gloo in the CPU tests).
Rank r owns the contiguous last-mode range [lo_r, hi_r) -- in the natural
layout that is one contiguous slab, itself a valid N-way tensor
(SURVEY.md §8e). Per mode n of an MTTKRP:

  n <  N-1   every rank computes the I_n x C partial over its slab; one
             all-reduce (sum) makes M identical everywhere.
  n == N-1   rows are disjoint: rank r holds M[lo_r:hi_r]; no exchange.

CP-ALS keeps U_0..U_{N-2} replicated and U_{N-1} row-sharded: the Gram of
U_{N-1}, its column norms and the fit's inner product are all-reduced
(C x C, C and 1 doubles); the other solves run redundantly and bit-identically
on every rank because their inputs are identical (reference cp_als.cpp:122-158).

The per-rank compute goes through a Backend; `GpuBackend` is the B200 path
(the C ABI). Tests inject a CPU backend to exercise the sharding and the
collectives with gloo at world_size 2 without a GPU.
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import List, Optional, Sequence

import numpy as np
import torch
import torch.distributed as dist


def shard_bounds(extent: int, world: int, rank: int):
    """Balanced contiguous split of the last mode (first extent % world shards
    one longer), so 180/8 and 100/8 split evenly within one row."""
    q, r = divmod(extent, world)
    lo = rank * q + min(rank, r)
    return lo, lo + q + (1 if rank < r else 0)


def shard_slab(x_full: np.ndarray, dims: Sequence[int], world: int, rank: int) -> np.ndarray:
    """Rank's contiguous slab of a naturally ordered tensor (a view)."""
    lo, hi = shard_bounds(dims[-1], world, rank)
    plane = int(np.prod(dims[:-1], dtype=np.int64))
    return x_full[lo * plane:hi * plane]


class Backend:
    """Per-rank compute used by the distributed drivers."""

    def mttkrp(self, slab, slab_dims, factors, mode) -> np.ndarray:  # pragma: no cover - interface
        raise NotImplementedError

    def gram(self, u: np.ndarray) -> np.ndarray:  # pragma: no cover - interface
        raise NotImplementedError

    def solve(self, h: np.ndarray, m: np.ndarray) -> np.ndarray:  # pragma: no cover - interface
        raise NotImplementedError


class GpuBackend(Backend):
    """The B200 path: C-ABI MTTKRP / Gram / solve on this rank's device."""

    def __init__(self, device: int = 0):
        from . import api
        self.api = api
        self.device = device
        self._tensor = None
        self._key = None

    def mttkrp(self, slab, slab_dims, factors, mode):
        key = (slab.ctypes.data, tuple(slab_dims))
        if key != self._key:
            self._tensor = self.api.DenseTensor(slab_dims, slab, device=self.device)
            self._key = key
        req = self.api.MttkrpRequest(self._tensor, factors, mode)
        return self.api.mttkrp(req).m

    def gram(self, u):
        return self.api.gram_hadamard([u], -1, device=self.device)

    def solve(self, h, m):
        return self.api.solve_psd(h, m, device=self.device)


def _allreduce(a: np.ndarray, device: torch.device) -> np.ndarray:
    t = torch.from_numpy(np.ascontiguousarray(a)).to(device)
    dist.all_reduce(t)
    return t.cpu().numpy()


def _allgather_rows(local: np.ndarray, extent: int, world: int, device: torch.device) -> np.ndarray:
    """All-gather of uneven row shards, padded to the largest shard."""
    cols = local.shape[1]
    width = -(-extent // world)
    buf = torch.zeros((width, cols), dtype=torch.float64, device=device)
    buf[:local.shape[0]] = torch.from_numpy(local).to(device)
    out = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(out, buf)
    rows = []
    for r in range(world):
        lo, hi = shard_bounds(extent, world, r)
        rows.append(out[r][:hi - lo].cpu().numpy())
    return np.concatenate(rows, axis=0)


def dist_mttkrp(backend: Backend, slab: np.ndarray, dims: Sequence[int], factors: Sequence[np.ndarray], mode: int,
                device: torch.device, gather_last: bool = True) -> np.ndarray:
    """MTTKRP of the full (sharded) tensor. factors are the full factors on
    every rank; U_{N-1} is sliced to the rank's rows here."""
    world, rank = dist.get_world_size(), dist.get_rank()
    n = len(dims)
    lo, hi = shard_bounds(dims[-1], world, rank)
    slab_dims = tuple(dims[:-1]) + (hi - lo,)
    local_f = list(factors[:-1]) + [np.ascontiguousarray(factors[-1][lo:hi])]
    m = backend.mttkrp(slab, slab_dims, local_f, mode)
    if mode < n - 1:
        return _allreduce(m, device)
    return _allgather_rows(m, dims[-1], world, device) if gather_last else m


@dataclass
class DistAlsResult:
    factors: List[np.ndarray]
    lambda_: np.ndarray
    fits: List[float]
    tensor_norm: float
    zero_tensor: bool


def _kruskal_random(dims, rank, seed):
    """KruskalModel::random (cp_als.cpp:87-99): one mt19937_64 stream, (r>>11)*2^-53."""
    from ._mt19937 import mt19937_64
    g = mt19937_64(seed)
    out = []
    for d in dims:
        out.append(np.array([(g.next() >> 11) * 2.0 ** -53 for _ in range(d * rank)]).reshape(d, rank))
    return out


def dist_cp_als(backend: Backend, slab: np.ndarray, dims: Sequence[int], rank: int, max_iters: int, tol: float,
                seed: int, device: torch.device) -> DistAlsResult:
    """CP-ALS over last-mode shards (cp_als.cpp:122-200 with the exchanges of
    SURVEY.md §8e)."""
    world, me = dist.get_world_size(), dist.get_rank()
    n = len(dims)
    lo, hi = shard_bounds(dims[-1], world, me)
    norm_x = math.sqrt(float(_allreduce(np.array([float(np.dot(slab, slab))]), device)[0]))
    factors = _kruskal_random(dims, rank, seed)
    factors[-1] = np.ascontiguousarray(factors[-1][lo:hi])  # row shard of the last factor
    lam = np.ones(rank)
    if norm_x == 0.0:
        full = [np.zeros((d, rank)) for d in dims]
        return DistAlsResult(full, np.zeros(rank), [], 0.0, True)
    slab_dims = tuple(dims[:-1]) + (hi - lo,)
    fits: List[float] = []
    prev = 0.0
    for it in range(1, max_iters + 1):
        grams = [backend.gram(u) for u in factors[:-1]] + [_allreduce(backend.gram(factors[-1]), device)]
        h_last = None
        m_last = None
        for mode in range(n):
            m = backend.mttkrp(slab, slab_dims, factors, mode)
            if mode < n - 1:
                m = _allreduce(m, device)
            h = np.ones((rank, rank))
            for k in range(n):
                if k != mode:
                    h = h * grams[k]
            u = backend.solve(h, m)
            # normalize_mode (cp_als.cpp:101-118); last mode norms span every shard
            sq = (u * u).sum(axis=0)
            if mode == n - 1:
                sq = _allreduce(sq, device)
            norms = np.sqrt(sq)
            safe = np.where(norms > 0, norms, 1.0)
            u = np.where(norms > 0, u * (1.0 / safe), u)
            lam = norms
            factors[mode] = u
            g = backend.gram(u)
            grams[mode] = _allreduce(g, device) if mode == n - 1 else g
            if mode == n - 1:
                h_last, m_last = h, m
        inner = float(_allreduce(np.array([float(np.sum(m_last * lam * factors[-1]))]), device)[0])
        norm_y_sq = float(np.sum(np.outer(lam, lam) * h_last * grams[-1]))
        res_sq = max(0.0, norm_x * norm_x - 2.0 * inner + norm_y_sq)
        fit = 1.0 - math.sqrt(res_sq) / norm_x
        fits.append(fit)
        if it > 1 and abs(fit - prev) < tol:
            break
        prev = fit
    full = list(factors[:-1]) + [_allgather_rows(factors[-1], dims[-1], world, device)]
    return DistAlsResult(full, lam, fits, norm_x, False)


# ------------------------------------------------ device-resident sharded CP-ALS
@dataclass
class ShardedAlsResult:
    factors: List[np.ndarray]  # modes 0..N-2 in full, then this rank's rows of mode N-1
    lambda_: np.ndarray
    fits: List[float]
    iter_seconds: List[float]
    tensor_norm: float
    zero_tensor: bool


class DeviceComm:
    """An NCCL communicator owned by the library (dmtk_gpu_comm_*): rank 0
    makes the 128-byte id, torch.distributed broadcasts it, every rank joins
    on its device. The library then all-reduces on its own stream, inside the
    CP-ALS per-mode CUDA graphs."""

    def __init__(self, device: int = 0):
        from . import _lib
        import ctypes as C
        self._lib = _lib.lib
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


def _check(lib, rc):
    if rc != 0:
        raise RuntimeError(lib.dmtk_gpu_last_error().decode())


def dist_cp_als_device(slab_tensor, comm: DeviceComm, global_last: int, last_lo: int, config) -> ShardedAlsResult:
    """The reference's cp_als (cp_als.cpp:122-200) over last-mode shards with
    the whole loop on the device (dmtk_gpu_cp_als_sharded): slab_tensor is this
    rank's DenseTensor (last-mode rows [last_lo, last_lo + its extent) of a
    tensor whose last extent is global_last); config an api.AlsConfig (the
    per-mode sweep)."""
    from . import _lib
    import ctypes as C
    lib = _lib.lib
    dims = slab_tensor.dims
    n = len(dims)
    rank = int(config.rank)
    cfg = _lib.AlsConfig(rank, config.max_iters, config.tol, config.seed, config.threads, int(config.algo),
                         int(config.order), int(bool(getattr(config, "dimension_tree", False))))
    f = np.zeros(int(sum(dims)) * max(rank, 1))
    lam = np.zeros(max(rank, 1))
    cap = max(int(config.max_iters), 1)
    fits = np.zeros(cap)
    secs = np.zeros(cap)
    k = C.c_int(0)
    zero = C.c_int(0)
    norm = np.zeros(1)
    dp = lambda a: a.ctypes.data_as(_lib.dp)  # noqa: E731
    _check(lib, lib.dmtk_gpu_cp_als_sharded(slab_tensor.handle(), comm.handle, int(global_last), int(last_lo),
                                            C.byref(cfg), dp(f), dp(lam), dp(fits), dp(secs), None, C.byref(k),
                                            C.byref(zero), dp(norm)))
    factors, off = [], 0
    for d in dims:
        factors.append(f[off:off + d * rank].reshape(d, rank).copy())
        off += d * rank
    return ShardedAlsResult(factors, lam[:rank].copy(), list(fits[:k.value]), list(secs[:k.value]), float(norm[0]),
                            bool(zero.value))
