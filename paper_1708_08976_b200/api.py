"""Python mirror of the reference dmtk API for the MTTKRP / KRP / CP-ALS path.

Names, argument meaning and error behaviour follow
/root/reference/proj/include/dmtk/{mttkrp,krp,cp_als,linalg}.hpp; every call
goes through the C ABI of libdmtk_gpu.so (include/dmtk_gpu.h) onto the B200.
Exceptions map the reference's C++ exception types:

    std::invalid_argument -> InvalidArgument (a ValueError)
    std::out_of_range     -> OutOfRange      (an IndexError)
    std::overflow_error   -> ShapeOverflow   (an OverflowError)
    CUDA / device errors  -> DeviceError     (a RuntimeError)

Layouts are the reference's: tensors in natural order (mode 0 fastest, i.e.
``x.reshape(dims[::-1])`` in NumPy C order), factors row-major ``I_k x C``.
"""
from __future__ import annotations

import ctypes as C
import os
import enum
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import _lib
from ._lib import lib


class InvalidArgument(ValueError):
    pass


class OutOfRange(IndexError):
    pass


class ShapeOverflow(OverflowError):
    pass


class DeviceError(RuntimeError):
    pass


class TensorFileError(RuntimeError):
    """dmtk::TensorFileError (tensor_io.hpp)."""


_ERR = {1: InvalidArgument, 2: OutOfRange, 3: ShapeOverflow, 4: DeviceError, 5: TensorFileError}


def _check(rc: int) -> None:
    if rc != 0:
        raise _ERR.get(rc, DeviceError)(lib.dmtk_gpu_last_error().decode())


class MttkrpAlgo(enum.IntEnum):
    """mttkrp.hpp:16-21"""
    baseline = 0
    one_step = 1
    two_step = 2
    automatic = 3


class TwoStepOrder(enum.IntEnum):
    """mttkrp.hpp:23-27"""
    automatic = 0
    left = 1
    right = 2


def _dp(a: np.ndarray):
    return a.ctypes.data_as(_lib.dp)


def _i64(seq) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(list(seq), dtype=np.int64))


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def device_count() -> int:
    n = C.c_int(0)
    _check(lib.dmtk_gpu_device_count(C.byref(n)))
    return n.value


# value distributions of the seeded generator (dmtk_gpu.h DMTK_GPU_DIST_*)
DISTS = {"uniform": 0, "ones": 1, "signed": 2, "normal": 3, "symslice": 4}


def mode_seed(seed: int, mode: int) -> int:
    """bench.cpp:26-28"""
    return (seed + 0x9E3779B97F4A7C15 * (mode + 1)) & 0xFFFFFFFFFFFFFFFF


def generate_factors(dims: Sequence[int], rank: int, seed: int, dist: str = "uniform", device: int = 0):
    """dmtk::gen_factors (bench.cpp:108-116) in HBM: factor n is the
    rows x rank stream of mode_seed(seed, n), transformed like `dist`.
    Returns one 1-way DenseTensor per factor (row-major values)."""
    return [DenseTensor.generate((int(d) * rank,), mode_seed(seed, n), dist, device) for n, d in enumerate(dims)]


class DenseTensor:
    """Dense FP64 tensor in natural order (tensor.hpp:19-38).

    Host values are uploaded to the device once, on first use, and kept
    there (the reference tensor is immutable, tensor.hpp:11-18).
    """

    def __init__(self, dims: Sequence[int], values=None, device: int = 0):
        self.dims = tuple(int(d) for d in dims)
        self.device = device
        self._host = None if values is None else _f64(values).reshape(-1)
        self._handle = C.c_void_p()
        self._owner = None

    @classmethod
    def from_device(cls, dims: Sequence[int], device_ptr: int, device: int = 0, owner=None) -> "DenseTensor":
        """Borrow an existing device buffer (DenseTensor::borrow, tensor.hpp:23)."""
        t = cls(dims, None, device)
        d = _i64(t.dims)
        _check(lib.dmtk_gpu_tensor_wrap(device, len(d), d.ctypes.data_as(_lib.i64p), C.c_void_p(device_ptr),
                                        C.byref(t._handle)))
        t._owner = owner
        return t

    @classmethod
    def load(cls, path: str, device: int = 0) -> "DenseTensor":
        """dmtk::read_tensor (tensor_io.hpp:25) straight into HBM (DNT1 file)."""
        h = C.c_void_p()
        _check(lib.dmtk_gpu_tensor_load(device, os.fsencode(path), C.byref(h)))
        with open(path, "rb") as f:  # the header the library just validated
            n = int(np.frombuffer(f.read(12)[8:], dtype="<u4")[0])
            dims = tuple(int(v) for v in np.frombuffer(f.read(8 * n), dtype="<u8"))
        t = cls(dims, None, device)
        t._handle = h
        return t

    @classmethod
    def generate(cls, dims: Sequence[int], seed: int, dist: str = "uniform", device: int = 0) -> "DenseTensor":
        """dmtk::gen_tensor (bench.cpp:88-97) generated in HBM: the reference's
        mt19937_64(seed) uniform(0,1) draws bitwise, or Dist::ones; the
        BASELINE configs' other distributions ("signed" U[-1,1), "normal"
        N(0,1), "symslice" fMRI slices) as fixed transforms of the same draws
        (DMTK_GPU_DIST_* in dmtk_gpu.h)."""
        if dist not in DISTS:
            raise InvalidArgument("gen_tensor: unknown distribution")
        t = cls(dims, None, device)
        d = _i64(t.dims)
        _check(lib.dmtk_gpu_tensor_generate(device, len(d), d.ctypes.data_as(_lib.i64p), C.c_uint64(seed),
                                            DISTS[dist], C.byref(t._handle)))
        return t

    def device_ptr(self) -> int:
        """Device address of the values (natural order, or the padded layout
        of an odd first extent: row pitch dims[0] + 1)."""
        p = C.c_void_p()
        _check(lib.dmtk_gpu_tensor_info(self.handle(), None, None, C.byref(p)))
        return int(p.value or 0)

    def pack_symmetric01(self) -> "DenseTensor":
        """A packed copy of a tensor symmetric in modes 0 and 1 (upper triangle
        of every slice; dmtk_gpu_tensor_pack_sym01). Supports cp_als (a
        dimension-tree sweep reading about half the bytes) and tensor_norm."""
        h = C.c_void_p()
        _check(lib.dmtk_gpu_tensor_pack_sym01(self.handle(), C.byref(h)))
        t = DenseTensor(self.dims, None, self.device)
        t._handle = h
        t._owner = self  # the packed copy is independent; keep the source alive anyway
        return t

    def slab(self, lo: int, hi: int) -> "DenseTensor":
        """The last-mode rows [lo, hi) as a new device tensor (a rank's shard,
        SURVEY 8e; dmtk_gpu_tensor_slab)."""
        h = C.c_void_p()
        _check(lib.dmtk_gpu_tensor_slab(self.handle(), int(lo), int(hi), C.byref(h)))
        t = DenseTensor(self.dims[:-1] + (int(hi) - int(lo),), None, self.device)
        t._handle = h
        return t

    def download(self) -> np.ndarray:
        """The values in natural order, from the device copy."""
        out = np.empty(self.total)
        _check(lib.dmtk_gpu_tensor_download(self.handle(), _dp(out)))
        return out

    @property
    def ndim(self) -> int:
        return len(self.dims)

    @property
    def total(self) -> int:
        return int(np.prod(self.dims, dtype=np.int64))

    def values(self) -> np.ndarray:
        return self._host

    def handle(self) -> C.c_void_p:
        if not self._handle:
            if self._host is None:
                raise InvalidArgument("DenseTensor: no data")
            d = _i64(self.dims)
            _check(lib.dmtk_gpu_tensor_upload(self.device, len(d), d.ctypes.data_as(_lib.i64p), _dp(self._host),
                                              C.byref(self._handle)))
        return self._handle

    def release(self) -> None:
        if self._handle:
            lib.dmtk_gpu_tensor_free(self._handle)
            self._handle = C.c_void_p()

    def __del__(self):
        try:
            self.release()
        except Exception:
            pass


@dataclass
class MttkrpRequest:
    """mttkrp.hpp:29-36"""
    tensor: Optional[DenseTensor]
    factors: Sequence[np.ndarray]
    mode: int = 0
    algo: MttkrpAlgo = MttkrpAlgo.automatic
    order: TwoStepOrder = TwoStepOrder.automatic
    threads: int = 1


@dataclass
class MttkrpResult:
    """mttkrp.hpp:38-41: m is I_n x C row-major; time is the TimeBreakdown."""
    m: np.ndarray
    time: dict = field(default_factory=dict)


def _factor_arrays(factors):
    mats = [_f64(f) for f in factors]
    for k, m in enumerate(mats):
        if m.ndim != 2:
            raise InvalidArgument(f"factor {k} must be a matrix")
    ptrs = (_lib.dp * max(len(mats), 1))()
    for k, m in enumerate(mats):
        ptrs[k] = _dp(m)
    rows = _i64([m.shape[0] for m in mats] or [0])
    cols = _i64([m.shape[1] for m in mats] or [0])
    return mats, ptrs, rows, cols


def mttkrp(request: MttkrpRequest) -> MttkrpResult:
    """dmtk::mttkrp (mttkrp.hpp:45): dispatch on request.algo."""
    if request.tensor is None:
        raise InvalidArgument("mttkrp: null tensor")
    t = request.tensor
    mats, ptrs, rows, cols = _factor_arrays(request.factors)
    n_rows = t.dims[request.mode] if 0 <= request.mode < t.ndim else 1
    rank = int(cols[0]) if len(mats) else 1
    out = np.empty((n_rows, max(rank, 1)), dtype=np.float64)
    tm = _lib.Times()
    _check(lib.dmtk_gpu_mttkrp(t.handle(), len(mats), ptrs, rows.ctypes.data_as(_lib.i64p),
                               cols.ctypes.data_as(_lib.i64p), int(request.mode), int(request.algo),
                               int(request.order), int(request.threads), _dp(out), C.byref(tm)))
    return MttkrpResult(out, tm.as_dict())


def mttkrp_baseline(request: MttkrpRequest) -> MttkrpResult:
    return mttkrp(MttkrpRequest(request.tensor, request.factors, request.mode, MttkrpAlgo.baseline,
                                request.order, request.threads))


def mttkrp_one_step(request: MttkrpRequest) -> MttkrpResult:
    return mttkrp(MttkrpRequest(request.tensor, request.factors, request.mode, MttkrpAlgo.one_step,
                                request.order, request.threads))


def mttkrp_two_step(request: MttkrpRequest) -> MttkrpResult:
    return mttkrp(MttkrpRequest(request.tensor, request.factors, request.mode, MttkrpAlgo.two_step,
                                request.order, request.threads))


def mttkrp_device(tensor: DenseTensor, device_factor_ptrs: Sequence[int], rank: int, mode: int,
                  algo: MttkrpAlgo, order: TwoStepOrder, device_out_ptr: int, stream: int = 0) -> None:
    """Device-resident MTTKRP (no host sync): operands are raw device pointers."""
    arr = (C.c_void_p * len(device_factor_ptrs))(*[C.c_void_p(p) for p in device_factor_ptrs])
    _check(lib.dmtk_gpu_mttkrp_device(tensor.handle(), arr, rank, mode, int(algo), int(order),
                                      C.c_void_p(device_out_ptr), C.c_void_p(stream)))


def choose_order(dims: Sequence[int], mode: int) -> TwoStepOrder:
    """mttkrp.hpp:53: left-first iff left(n) > right(n)."""
    d = _i64(dims)
    o = C.c_int(0)
    _check(lib.dmtk_gpu_choose_order(len(d), d.ctypes.data_as(_lib.i64p), mode, C.byref(o)))
    return TwoStepOrder(o.value)


@dataclass
class KrpStats:
    """krp.hpp:15-17"""
    hadamard_products: int = 0


def _krp(inputs, variant: int, stats: Optional[KrpStats], device: int) -> np.ndarray:
    if inputs is None or len(inputs) == 0:
        raise InvalidArgument("krp: empty input list")
    cols = None
    for z, m in enumerate(inputs):
        if m is None:
            raise InvalidArgument("krp: null input")
        m = np.asarray(m)
        if cols is None:
            cols = m.shape[1]
        elif m.shape[1] != cols:
            raise InvalidArgument(f"krp: input {z} has {m.shape[1]} columns, expected {cols}")
        if m.shape[0] < 1:
            raise InvalidArgument(f"krp: input {z} has no rows")
    mats, ptrs, rows, _ = _factor_arrays(inputs)
    total = int(np.prod(rows, dtype=np.int64))
    out = np.empty((total, cols), dtype=np.float64)
    h = C.c_uint64(0)
    _check(lib.dmtk_gpu_krp(device, len(mats), ptrs, rows.ctypes.data_as(_lib.i64p), cols, variant, _dp(out),
                            C.byref(h)))
    if stats is not None:
        stats.hadamard_products += h.value
    return out


def krp(inputs: Sequence[np.ndarray], threads: int = 1, stats: Optional[KrpStats] = None,
        device: int = 0) -> np.ndarray:
    """dmtk::krp (krp.hpp:75): K = in[0] (.) ... (.) in[Z-1], last input fastest."""
    return _krp(inputs, 0, stats, device)


def krp_naive(inputs: Sequence[np.ndarray], threads: int = 1, stats: Optional[KrpStats] = None,
              device: int = 0) -> np.ndarray:
    """dmtk::krp_naive (krp.hpp:79): same product, reuse-free count."""
    return _krp(inputs, 1, stats, device)


def krp_small(inputs: Sequence[np.ndarray], stats: Optional[KrpStats] = None, device: int = 0) -> np.ndarray:
    """dmtk::krp_small (krp.hpp:83): Z in {1, 2} only."""
    if inputs is not None and len(inputs) > 2:
        raise InvalidArgument(f"krp_small: got {len(inputs)} inputs, handles only Z in {{1,2}}")
    return _krp(inputs, 0, stats, device)


def krp_device(device_input_ptrs: Sequence[int], rows: Sequence[int], cols: int, out_ptr: int,
               scratch_ptr: int = 0, stream: int = 0) -> None:
    """Device-resident KRP (dmtk_gpu_krp_device): inputs and output already in
    HBM (row-major), enqueued on `stream` without a host sync. scratch holds
    prod(rows[:-1]) * cols doubles when len(rows) > 2."""
    z = len(device_input_ptrs)
    arr = (C.c_void_p * max(z, 1))(*device_input_ptrs)
    r = np.asarray(rows, dtype=np.int64)
    _check(lib.dmtk_gpu_krp_device(z, arr, r.ctypes.data_as(_lib.i64p), cols, C.c_void_p(out_ptr),
                                   C.c_void_p(scratch_ptr or None), C.c_void_p(stream or None)))


def tensor_norm(x: DenseTensor) -> float:
    """dmtk::tensor_norm (cp_als.hpp:68)."""
    out = np.zeros(1)
    _check(lib.dmtk_gpu_tensor_norm(x.handle(), _dp(out)))
    return float(out[0])


def gram_hadamard(factors: Sequence[np.ndarray], skip: int, device: int = 0) -> np.ndarray:
    """dmtk::gram_hadamard (linalg.hpp:48)."""
    if len(factors) == 0:
        raise InvalidArgument("gram_hadamard: no factors")
    mats, ptrs, rows, cols = _factor_arrays(factors)
    c = int(cols[0])
    for k, m in enumerate(mats):
        if m.shape[1] != c:
            raise InvalidArgument(f"gram_hadamard: factor {k} has rank {m.shape[1]}, expected {c}")
    h = np.empty((c, c))
    _check(lib.dmtk_gpu_gram_hadamard(device, len(mats), rows.ctypes.data_as(_lib.i64p), c, ptrs, skip, _dp(h)))
    return h


def solve_psd(h: np.ndarray, m: np.ndarray, device: int = 0) -> np.ndarray:
    """dmtk::solve_psd (linalg.hpp:54): U * H = M."""
    h = _f64(h)
    m = _f64(m)
    if m.shape[1] != h.shape[0]:
        raise InvalidArgument(f"solve_psd: M has {m.shape[1]} columns, H is {h.shape[0]}x{h.shape[0]}")
    u = np.empty_like(m)
    _check(lib.dmtk_gpu_solve_psd(device, h.shape[0], _dp(h), m.shape[0], _dp(m), _dp(u)))
    return u


@dataclass
class KruskalModel:
    """cp_als.hpp:16-30"""
    factors: List[np.ndarray]
    lambda_: np.ndarray

    def ndim(self) -> int:
        return len(self.factors)

    def rank(self) -> int:
        return 0 if not self.factors else self.factors[0].shape[1]


@dataclass
class AlsConfig:
    """cp_als.hpp:32-40"""
    rank: int = 1
    max_iters: int = 50
    tol: float = 1e-6
    seed: int = 0
    threads: int = 1
    algo: MttkrpAlgo = MttkrpAlgo.automatic
    order: TwoStepOrder = TwoStepOrder.automatic
    # GPU-only: dimension-tree sweep (two tensor passes per iteration, see
    # include/dmtk_gpu.h); False keeps the reference's one MTTKRP per mode
    dimension_tree: bool = False


@dataclass
class FitResult:
    """cp_als.hpp:42-47"""
    fit: float = 0.0
    rel_residual: float = 0.0
    abs_residual: float = 0.0
    defined: bool = True


@dataclass
class AlsIterRecord:
    """cp_als.hpp:49-54 (fit only carries the fit value on the GPU path)."""
    iter: int
    fit: FitResult
    mode_time: List[float]
    total_seconds: float


@dataclass
class AlsTrace:
    iters: List[AlsIterRecord]
    zero_tensor: bool
    tensor_norm: float


@dataclass
class AlsResult:
    model: KruskalModel
    trace: AlsTrace


def cp_als(x: DenseTensor, config: AlsConfig) -> AlsResult:
    """dmtk::cp_als (cp_als.hpp:83), fully on the device."""
    dims = x.dims
    n = len(dims)
    cfg = _lib.AlsConfig(config.rank, config.max_iters, config.tol, config.seed, config.threads,
                         int(config.algo), int(config.order), int(bool(config.dimension_tree)))
    ftot = int(sum(dims)) * max(int(config.rank), 1)
    f = np.zeros(ftot)
    lam = np.zeros(max(int(config.rank), 1))
    cap = max(int(config.max_iters), 1)
    fits = np.zeros(cap)
    secs = np.zeros(cap)
    msecs = np.zeros(cap * n)
    k = C.c_int(0)
    zero = C.c_int(0)
    norm = np.zeros(1)
    _check(lib.dmtk_gpu_cp_als(x.handle(), C.byref(cfg), _dp(f), _dp(lam), _dp(fits), _dp(secs), _dp(msecs),
                               C.byref(k), C.byref(zero), _dp(norm)))
    factors, off = [], 0
    for d in dims:
        factors.append(f[off:off + d * config.rank].reshape(d, config.rank).copy())
        off += d * config.rank
    iters = [AlsIterRecord(i + 1, FitResult(fit=float(fits[i])), list(msecs[i * n:(i + 1) * n]), float(secs[i]))
             for i in range(k.value)]
    return AlsResult(KruskalModel(factors, lam[:config.rank].copy()),
                     AlsTrace(iters, bool(zero.value), float(norm[0])))


def als_iterate(x: DenseTensor, model: KruskalModel, config: AlsConfig, norm_x: float,
                iter_index: int) -> AlsIterRecord:
    """dmtk::als_iterate (cp_als.hpp:74-75): one Gauss-Seidel sweep of `model`
    (updated in place: factors and lambda_) on the device; the fit comes from
    the last mode's MTTKRP (cp_als.cpp:122-158)."""
    mats = [np.ascontiguousarray(m, dtype=np.float64) for m in model.factors]
    ptrs = (_lib.dp * len(mats))(*[_dp(m) for m in mats])
    rows = _i64([m.shape[0] for m in mats])
    cols = _i64([m.shape[1] if m.ndim == 2 else 0 for m in mats]) if mats else _i64([0])
    lam = np.array(model.lambda_, dtype=np.float64, copy=True)
    cfg = _lib.AlsConfig(config.rank, config.max_iters, config.tol, config.seed, config.threads,
                         int(config.algo), int(config.order), 0)
    f4 = np.zeros(4)
    sec = np.zeros(1)
    msec = np.zeros(max(len(mats), 1))
    _check(lib.dmtk_gpu_als_iterate(x.handle(), C.byref(cfg), len(mats), ptrs, rows.ctypes.data_as(_lib.i64p),
                                    cols.ctypes.data_as(_lib.i64p), _dp(lam), lam.size, float(norm_x),
                                    int(iter_index), _dp(f4), _dp(sec), _dp(msec)))
    model.factors = mats
    model.lambda_ = lam
    return AlsIterRecord(int(iter_index), FitResult(float(f4[0]), float(f4[1]), float(f4[2]), bool(f4[3])),
                         list(msec[:len(mats)]), float(sec[0]))


def fit(x: DenseTensor, model: KruskalModel, threads: int = 1) -> FitResult:
    """dmtk::fit (cp_als.hpp:79)."""
    mats, ptrs, rows, cols = _factor_arrays(model.factors)
    lam = _f64(model.lambda_)
    out = np.zeros(4)
    _check(lib.dmtk_gpu_fit(x.handle(), len(mats), ptrs, rows.ctypes.data_as(_lib.i64p),
                            cols.ctypes.data_as(_lib.i64p), _dp(lam), lam.size, threads, _dp(out)))
    return FitResult(float(out[0]), float(out[1]), float(out[2]), bool(out[3]))


def fp64_peak_tflops(device: int = 0) -> float:
    out = np.zeros(1)
    _check(lib.dmtk_gpu_fp64_peak(device, _dp(out)))
    return float(out[0])


def fp64_peak_tflops_sustained(seconds: float = 1.0, device: int = 0) -> float:
    out = np.zeros(1)
    _check(lib.dmtk_gpu_fp64_peak_sustained(device, seconds, _dp(out)))
    return float(out[0])


def launch_count() -> int:
    return int(lib.dmtk_gpu_launch_count())
