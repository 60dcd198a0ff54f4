"""ctypes bindings for the TEST-SIDE checkers.

* ``Oracle`` -- oracle/liboracle.so, the plain-C restatement (oracle/oracle.c).
* ``Ref``    -- oracle/_ref/libdmtk_ref.so, the unmodified reference library
  compiled from /root/reference/proj/src plus oracle/ref_capi.cpp.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline / reference
arm) import this module. The product path never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_DIR = os.path.join(ROOT, "oracle")
ORACLE_SO = os.path.join(ORACLE_DIR, "liboracle.so")
REF_SO = os.path.join(ORACLE_DIR, "_ref", "libdmtk_ref.so")

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int64)


def _d(a: np.ndarray):
    return a.ctypes.data_as(_dp)


def _i64(seq) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(seq, dtype=np.int64))


def _ptr_array(mats):
    arr = (_dp * len(mats))()
    for k, m in enumerate(mats):
        arr[k] = _d(m)
    return arr


def build_oracle(ref: bool = True) -> None:
    targets = ["oracle"] + (["ref"] if ref and os.path.isdir("/root/reference/proj/src") else [])
    subprocess.run(["make", "-s", "-C", ORACLE_DIR, *targets], check=True)


class OrcFit(C.Structure):
    _fields_ = [("fit", C.c_double), ("rel_residual", C.c_double),
                ("abs_residual", C.c_double), ("defined", C.c_int)]


class Oracle:
    """The C restatement (oracle/oracle.c)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build_oracle(ref=False)
        L = C.CDLL(path)
        L.orc_gen_uniform.argtypes = [C.c_uint64, C.c_int64, _dp]
        L.orc_mode_seed.restype = C.c_uint64
        L.orc_mode_seed.argtypes = [C.c_uint64, C.c_int64]
        L.orc_gen_factors.argtypes = [C.c_int, _ip, C.c_int64, C.c_uint64, _dp]
        L.orc_kruskal_random.argtypes = [C.c_int, _ip, C.c_int64, C.c_uint64, _dp, _dp]
        L.orc_krp_kron.argtypes = [C.c_int, C.POINTER(_dp), _ip, C.c_int64, _dp]
        L.orc_mttkrp_loops.argtypes = [C.c_int, _ip, _dp, C.POINTER(_dp), C.c_int64, C.c_int64, _dp]
        L.orc_reconstruct.argtypes = [C.c_int, _ip, C.POINTER(_dp), _dp, C.c_int64, _dp]
        L.orc_gram_hadamard.argtypes = [C.c_int, _ip, C.POINTER(_dp), C.c_int64, C.c_int64, _dp]
        L.orc_solve_psd.restype = C.c_int
        L.orc_solve_psd.argtypes = [_dp, C.c_int64, _dp, C.c_int64, _dp]
        L.orc_tensor_norm.restype = C.c_double
        L.orc_tensor_norm.argtypes = [_dp, C.c_int64]
        L.orc_normalize_mode.argtypes = [_dp, C.c_int64, C.c_int64, _dp]
        L.orc_fit_from_last_mode.restype = OrcFit
        L.orc_fit_from_last_mode.argtypes = [C.c_double, _dp, C.c_int64, C.c_int64, _dp, _dp, _dp]
        L.orc_gen_dist.restype = C.c_int
        L.orc_gen_dist.argtypes = [C.c_uint64, C.c_int, C.c_int, _ip, C.c_int, _dp]
        L.orc_gen_factors_dist.restype = C.c_int
        L.orc_gen_factors_dist.argtypes = [C.c_int, _ip, C.c_int64, C.c_uint64, C.c_int, _dp]
        L.orc_box_muller.restype = C.c_double
        L.orc_box_muller.argtypes = [C.c_double, C.c_double, C.c_int]
        L.orc_tanh_portable.restype = C.c_double
        L.orc_tanh_portable.argtypes = [C.c_double]
        L.orc_cp_als.restype = C.c_int
        L.orc_cp_als.argtypes = [C.c_int, _ip, _dp, C.c_int64, C.c_int, C.c_double, C.c_uint64,
                                 _dp, _dp, _dp, C.POINTER(C.c_int)]
        self.L = L

    # -- generators -------------------------------------------------------
    def uniform(self, seed: int, n: int) -> np.ndarray:
        out = np.empty(n, dtype=np.float64)
        self.L.orc_gen_uniform(seed, n, _d(out))
        return out

    def gen_tensor(self, dims, seed: int) -> np.ndarray:
        return self.uniform(seed, int(np.prod(dims)))

    def gen_factors(self, dims, rank: int, seed: int):
        d = _i64(dims)
        out = np.empty(int(d.sum()) * rank, dtype=np.float64)
        self.L.orc_gen_factors(len(d), d.ctypes.data_as(_ip), rank, seed, _d(out))
        return _split(out, dims, rank)

    DISTS = {"uniform": 0, "ones": 1, "signed": 2, "normal": 3, "symslice": 4}

    def gen_dist(self, dims, seed: int, dist: str = "uniform", threads: int = 0) -> np.ndarray:
        """gen_tensor with the BASELINE distributions (oracle.c, bitwise the device's)."""
        d = _i64(dims)
        out = np.empty(int(np.prod(d)), dtype=np.float64)
        rc = self.L.orc_gen_dist(seed, self.DISTS[dist], len(d), d.ctypes.data_as(_ip),
                                 threads or (os.cpu_count() or 1), _d(out))
        assert rc == 0, "orc_gen_dist rejected its arguments"
        return out

    def gen_factors_dist(self, dims, rank: int, seed: int, dist: str = "uniform"):
        d = _i64(dims)
        out = np.empty(int(d.sum()) * rank, dtype=np.float64)
        assert self.L.orc_gen_factors_dist(len(d), d.ctypes.data_as(_ip), rank, seed, self.DISTS[dist], _d(out)) == 0
        return _split(out, dims, rank)

    def kruskal_random(self, dims, rank: int, seed: int):
        d = _i64(dims)
        f = np.empty(int(d.sum()) * rank, dtype=np.float64)
        lam = np.empty(rank, dtype=np.float64)
        self.L.orc_kruskal_random(len(d), d.ctypes.data_as(_ip), rank, seed, _d(f), _d(lam))
        return _split(f, dims, rank), lam

    # -- algorithms -------------------------------------------------------
    def krp(self, inputs) -> np.ndarray:
        mats = [np.ascontiguousarray(m, dtype=np.float64) for m in inputs]
        rows = _i64([m.shape[0] for m in mats])
        cols = mats[0].shape[1]
        out = np.empty((int(np.prod(rows)), cols), dtype=np.float64)
        rc = self.L.orc_krp_kron(len(mats), _ptr_array(mats), rows.ctypes.data_as(_ip), cols, _d(out))
        assert rc == 0
        return out

    def mttkrp(self, x: np.ndarray, dims, factors, mode: int) -> np.ndarray:
        d = _i64(dims)
        x = np.ascontiguousarray(x, dtype=np.float64).reshape(-1)
        mats = [np.ascontiguousarray(m, dtype=np.float64) for m in factors]
        rank = mats[0].shape[1]
        out = np.empty((int(d[mode]), rank), dtype=np.float64)
        rc = self.L.orc_mttkrp_loops(len(d), d.ctypes.data_as(_ip), _d(x), _ptr_array(mats), rank, mode, _d(out))
        assert rc == 0
        return out

    def reconstruct(self, factors, lam) -> np.ndarray:
        mats = [np.ascontiguousarray(m, dtype=np.float64) for m in factors]
        d = _i64([m.shape[0] for m in mats])
        lam = np.ascontiguousarray(lam, dtype=np.float64)
        out = np.empty(int(np.prod(d)), dtype=np.float64)
        self.L.orc_reconstruct(len(d), d.ctypes.data_as(_ip), _ptr_array(mats), _d(lam), mats[0].shape[1], _d(out))
        return out

    def gram_hadamard(self, factors, skip: int) -> np.ndarray:
        mats = [np.ascontiguousarray(m, dtype=np.float64) for m in factors]
        d = _i64([m.shape[0] for m in mats])
        c = mats[0].shape[1]
        h = np.empty((c, c), dtype=np.float64)
        self.L.orc_gram_hadamard(len(d), d.ctypes.data_as(_ip), _ptr_array(mats), c, skip, _d(h))
        return h

    def solve_psd(self, h: np.ndarray, m: np.ndarray):
        h = np.ascontiguousarray(h, dtype=np.float64)
        m = np.ascontiguousarray(m, dtype=np.float64)
        u = np.empty_like(m)
        used_chol = self.L.orc_solve_psd(_d(h), h.shape[0], _d(m), m.shape[0], _d(u))
        return u, bool(used_chol)

    def tensor_norm(self, x: np.ndarray) -> float:
        x = np.ascontiguousarray(x, dtype=np.float64).reshape(-1)
        return self.L.orc_tensor_norm(_d(x), x.size)

    def normalize_mode(self, u: np.ndarray):
        u = np.array(u, dtype=np.float64, copy=True)
        lam = np.empty(u.shape[1], dtype=np.float64)
        self.L.orc_normalize_mode(_d(u), u.shape[0], u.shape[1], _d(lam))
        return u, lam

    def cp_als(self, x: np.ndarray, dims, rank: int, iters: int, tol: float, seed: int):
        d = _i64(dims)
        x = np.ascontiguousarray(x, dtype=np.float64).reshape(-1)
        f = np.empty(int(d.sum()) * rank, dtype=np.float64)
        lam = np.empty(rank, dtype=np.float64)
        fits = np.zeros(max(iters, 1), dtype=np.float64)
        zero = C.c_int(0)
        n = self.L.orc_cp_als(len(d), d.ctypes.data_as(_ip), _d(x), rank, iters, tol, seed,
                              _d(f), _d(lam), _d(fits), C.byref(zero))
        assert n >= 0
        return _split(f, dims, rank), lam, fits[:n].copy(), bool(zero.value)


class RefError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


class Ref:
    """The unmodified reference library (oracle/_ref/libdmtk_ref.so)."""

    ALGO = {"baseline": 0, "one_step": 1, "two_step": 2, "automatic": 3}
    ORDER = {"automatic": 0, "left": 1, "right": 2}

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            build_oracle(ref=True)
        L = C.CDLL(path)
        L.ref_last_error.restype = C.c_char_p
        L.ref_mttkrp.argtypes = [C.c_int, _ip, _dp, _dp, C.c_int64, C.c_int64, C.c_int, C.c_int, C.c_int, _dp, _dp]
        L.ref_choose_order.argtypes = [C.c_int, _ip, C.c_int64]
        L.ref_krp.argtypes = [C.c_int, _ip, C.c_int64, _dp, C.c_int, C.c_int, _dp, C.POINTER(C.c_uint64)]
        L.ref_mttkrp_oracle.argtypes = [C.c_int, _ip, _dp, _dp, C.c_int64, C.c_int64, _dp]
        L.ref_gen_tensor.argtypes = [C.c_int, _ip, C.c_uint64, _dp]
        L.ref_gen_factors.argtypes = [C.c_int, _ip, C.c_int64, C.c_uint64, _dp]
        L.ref_kruskal_random.argtypes = [C.c_int, _ip, C.c_int64, C.c_uint64, _dp, _dp]
        L.ref_tensor_norm.argtypes = [C.c_int, _ip, _dp, _dp]
        L.ref_gram_hadamard.argtypes = [C.c_int, _ip, C.c_int64, _dp, C.c_int64, _dp]
        L.ref_solve_psd.argtypes = [C.c_int64, _dp, C.c_int64, _dp, _dp]
        L.ref_cp_als.argtypes = [C.c_int, _ip, _dp, C.c_int64, C.c_int, C.c_double, C.c_uint64, C.c_int,
                                 C.c_int, C.c_int, _dp, _dp, _dp, _dp, C.POINTER(C.c_int),
                                 C.POINTER(C.c_int), _dp]
        L.ref_als_iterate.argtypes = [C.c_int, _ip, _dp, C.c_int64, _dp, _dp, C.c_int, C.c_int, C.c_int,
                                      C.c_double, C.c_int, _dp, _dp]
        L.ref_fit.argtypes = [C.c_int, _ip, _dp, C.c_int64, _dp, _dp, C.c_int, _dp]
        L.ref_write_tensor.argtypes = [C.c_char_p, C.c_int, _ip, _dp]
        L.ref_read_tensor.argtypes = [C.c_char_p, C.POINTER(C.c_int), _ip, _dp, C.c_int64]
        self.L = L

    def _check(self, rc: int):
        if rc != 0:
            raise RefError(rc, self.L.ref_last_error().decode())

    def write_tensor(self, path: str, x: np.ndarray, dims) -> None:
        """dmtk::write_tensor (tensor_io.hpp:24): a DNT1 file."""
        d = _i64(dims)
        self._check(self.L.ref_write_tensor(os.fsencode(path), len(d), d.ctypes.data_as(_ip), _d(x)))

    def read_tensor(self, path: str, capacity: int = 0):
        """dmtk::read_tensor (tensor_io.hpp:25): (dims, values) or RefError(5, msg)."""
        nd = C.c_int()
        dims = np.zeros(64, dtype=np.int64)
        vals = np.empty(max(capacity, 1))
        self._check(self.L.ref_read_tensor(os.fsencode(path), C.byref(nd), dims.ctypes.data_as(_ip),
                                           _d(vals) if capacity else None, capacity))
        return tuple(int(v) for v in dims[:nd.value]), (vals if capacity else None)

    def gen_tensor(self, dims, seed: int) -> np.ndarray:
        d = _i64(dims)
        out = np.empty(int(np.prod(d)), dtype=np.float64)
        self._check(self.L.ref_gen_tensor(len(d), d.ctypes.data_as(_ip), seed, _d(out)))
        return out

    def gen_factors(self, dims, rank: int, seed: int):
        d = _i64(dims)
        out = np.empty(int(d.sum()) * rank, dtype=np.float64)
        self._check(self.L.ref_gen_factors(len(d), d.ctypes.data_as(_ip), rank, seed, _d(out)))
        return _split(out, dims, rank)

    def kruskal_random(self, dims, rank: int, seed: int):
        d = _i64(dims)
        f = np.empty(int(d.sum()) * rank, dtype=np.float64)
        lam = np.empty(rank, dtype=np.float64)
        self._check(self.L.ref_kruskal_random(len(d), d.ctypes.data_as(_ip), rank, seed, _d(f), _d(lam)))
        return _split(f, dims, rank), lam

    def mttkrp(self, x, dims, factors, mode: int, algo: str = "automatic", order: str = "automatic",
               threads: int = 1, times: bool = False):
        d = _i64(dims)
        x = np.ascontiguousarray(x, dtype=np.float64).reshape(-1)
        cat = np.ascontiguousarray(np.concatenate([np.asarray(f, dtype=np.float64).reshape(-1) for f in factors]))
        rank = np.asarray(factors[0]).shape[1]
        rows = int(d[mode]) if 0 <= mode < len(d) else 1
        out = np.empty((rows, rank), dtype=np.float64)
        t8 = np.zeros(8, dtype=np.float64)
        self._check(self.L.ref_mttkrp(len(d), d.ctypes.data_as(_ip), _d(x), _d(cat), rank, mode,
                                      self.ALGO[algo], self.ORDER[order], threads, _d(out), _d(t8)))
        return (out, t8) if times else out

    def mttkrp_loops(self, x, dims, factors, mode: int) -> np.ndarray:
        d = _i64(dims)
        x = np.ascontiguousarray(x, dtype=np.float64).reshape(-1)
        cat = np.ascontiguousarray(np.concatenate([np.asarray(f, dtype=np.float64).reshape(-1) for f in factors]))
        rank = np.asarray(factors[0]).shape[1]
        out = np.empty((int(d[mode]), rank), dtype=np.float64)
        self._check(self.L.ref_mttkrp_oracle(len(d), d.ctypes.data_as(_ip), _d(x), _d(cat), rank, mode, _d(out)))
        return out

    def choose_order(self, dims, mode: int) -> str:
        d = _i64(dims)
        return {0: "automatic", 1: "left", 2: "right"}[self.L.ref_choose_order(len(d), d.ctypes.data_as(_ip), mode)]

    def krp(self, inputs, threads: int = 1, naive: bool = False):
        mats = [np.ascontiguousarray(m, dtype=np.float64) for m in inputs]
        rows = _i64([m.shape[0] for m in mats])
        cols = mats[0].shape[1]
        cat = np.ascontiguousarray(np.concatenate([m.reshape(-1) for m in mats]))
        out = np.empty((int(np.prod(rows)), cols), dtype=np.float64)
        had = C.c_uint64(0)
        self._check(self.L.ref_krp(len(mats), rows.ctypes.data_as(_ip), cols, _d(cat), threads,
                                   1 if naive else 0, _d(out), C.byref(had)))
        return out, had.value

    def tensor_norm(self, x, dims) -> float:
        d = _i64(dims)
        x = np.ascontiguousarray(x, dtype=np.float64).reshape(-1)
        out = np.zeros(1, dtype=np.float64)
        self._check(self.L.ref_tensor_norm(len(d), d.ctypes.data_as(_ip), _d(x), _d(out)))
        return float(out[0])

    def gram_hadamard(self, factors, skip: int):
        mats = [np.ascontiguousarray(m, dtype=np.float64) for m in factors]
        d = _i64([m.shape[0] for m in mats])
        c = mats[0].shape[1]
        cat = np.ascontiguousarray(np.concatenate([m.reshape(-1) for m in mats]))
        h = np.empty((c, c), dtype=np.float64)
        self._check(self.L.ref_gram_hadamard(len(d), d.ctypes.data_as(_ip), c, _d(cat), skip, _d(h)))
        return h

    def solve_psd(self, h, m):
        h = np.ascontiguousarray(h, dtype=np.float64)
        m = np.ascontiguousarray(m, dtype=np.float64)
        u = np.empty_like(m)
        self._check(self.L.ref_solve_psd(h.shape[0], _d(h), m.shape[0], _d(m), _d(u)))
        return u

    def cp_als(self, x, dims, rank: int, iters: int, tol: float = 0.0, seed: int = 0, threads: int = 1,
               algo: str = "automatic", order: str = "automatic"):
        d = _i64(dims)
        x = np.ascontiguousarray(x, dtype=np.float64).reshape(-1)
        f = np.empty(int(d.sum()) * rank, dtype=np.float64)
        lam = np.empty(rank, dtype=np.float64)
        fits = np.zeros(max(iters, 1), dtype=np.float64)
        secs = np.zeros(max(iters, 1), dtype=np.float64)
        n = C.c_int(0)
        zero = C.c_int(0)
        normx = np.zeros(1, dtype=np.float64)
        self._check(self.L.ref_cp_als(len(d), d.ctypes.data_as(_ip), _d(x), rank, iters, tol, seed, threads,
                                      self.ALGO[algo], self.ORDER[order], _d(f), _d(lam), _d(fits), _d(secs),
                                      C.byref(n), C.byref(zero), _d(normx)))
        k = n.value
        return {"factors": _split(f, dims, rank), "lambda": lam, "fits": fits[:k].copy(),
                "iter_seconds": secs[:k].copy(), "zero_tensor": bool(zero.value), "norm_x": float(normx[0])}

    def als_iterate(self, x, dims, factors, lam, norm_x: float, iter_index: int = 1, threads: int = 1,
                    algo: str = "automatic", order: str = "automatic"):
        """dmtk::als_iterate (cp_als.hpp:74-75): one sweep; returns (factors, lambda, fit4, seconds)."""
        d = _i64(dims)
        x = np.ascontiguousarray(x, dtype=np.float64).reshape(-1)
        rank = np.asarray(factors[0]).shape[1]
        cat = np.ascontiguousarray(np.concatenate([np.asarray(m, dtype=np.float64).reshape(-1) for m in factors]))
        lam = np.array(lam, dtype=np.float64, copy=True)
        out = np.zeros(4, dtype=np.float64)
        sec = np.zeros(1, dtype=np.float64)
        self._check(self.L.ref_als_iterate(len(d), d.ctypes.data_as(_ip), _d(x), rank, _d(cat), _d(lam), threads,
                                           self.ALGO[algo], self.ORDER[order], norm_x, iter_index, _d(out), _d(sec)))
        return _split(cat, dims, rank), lam, out, float(sec[0])

    def fit(self, x, dims, factors, lam, threads: int = 1):
        d = _i64(dims)
        x = np.ascontiguousarray(x, dtype=np.float64).reshape(-1)
        rank = np.asarray(factors[0]).shape[1]
        cat = np.ascontiguousarray(np.concatenate([np.asarray(m, dtype=np.float64).reshape(-1) for m in factors]))
        lam = np.ascontiguousarray(lam, dtype=np.float64)
        out = np.zeros(4, dtype=np.float64)
        self._check(self.L.ref_fit(len(d), d.ctypes.data_as(_ip), _d(x), rank, _d(cat), _d(lam), threads, _d(out)))
        return {"fit": out[0], "rel_residual": out[1], "abs_residual": out[2], "defined": bool(out[3])}


def _split(flat: np.ndarray, dims, rank: int):
    out, off = [], 0
    for n in dims:
        out.append(flat[off:off + n * rank].reshape(n, rank).copy())
        off += n * rank
    return out
