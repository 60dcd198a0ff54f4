"""ctypes binding of libdmtk_gpu.so (include/dmtk_gpu.h).

The library is built in-tree (``make -C paper_1708_08976_b200/csrc``, or
``__graft_entry__.build()``). There is no fallback: if the shared library is
missing, importing this module raises.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# DMTK_GPU_LIB: developer override (A/B builds of the same sources)
LIB_PATH = os.environ.get("DMTK_GPU_LIB") or os.path.join(HERE, "libdmtk_gpu.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build the CUDA library first "
        "(python -c 'import __graft_entry__ as g; g.build()'). The B200 path has no CPU fallback.")

lib = C.CDLL(LIB_PATH)

dp = C.POINTER(C.c_double)
i64p = C.POINTER(C.c_int64)
dpp = C.POINTER(dp)


class Times(C.Structure):
    """dmtk_gpu_times == reference TimeBreakdown (timing.hpp:11-20)."""
    _fields_ = [(n, C.c_double) for n in
                ("total", "matmul", "krp_full", "krp_partial", "matvec", "reduce", "reorder", "other")]

    def as_dict(self):
        return {n: getattr(self, n) for n, _ in self._fields_}


class AlsConfig(C.Structure):
    _fields_ = [("rank", C.c_int64), ("max_iters", C.c_int), ("tol", C.c_double), ("seed", C.c_uint64),
                ("threads", C.c_int), ("algo", C.c_int), ("order", C.c_int), ("dimtree", C.c_int)]


T = C.c_void_p  # dmtk_gpu_tensor

_SIGS = {
    "dmtk_gpu_last_error": (C.c_char_p, []),
    "dmtk_gpu_version": (C.c_int, []),
    "dmtk_gpu_device_count": (C.c_int, [C.POINTER(C.c_int)]),
    "dmtk_gpu_tensor_upload": (C.c_int, [C.c_int, C.c_int, i64p, dp, C.POINTER(T)]),
    "dmtk_gpu_tensor_wrap": (C.c_int, [C.c_int, C.c_int, i64p, C.c_void_p, C.POINTER(T)]),
    "dmtk_gpu_tensor_free": (C.c_int, [T]),
    "dmtk_gpu_tensor_info": (C.c_int, [T, C.POINTER(C.c_int), i64p, C.POINTER(C.c_void_p)]),
    "dmtk_gpu_tensor_load": (C.c_int, [C.c_int, C.c_char_p, C.POINTER(T)]),
    "dmtk_gpu_tensor_generate": (C.c_int, [C.c_int, C.c_int, i64p, C.c_uint64, C.c_int, C.POINTER(T)]),
    "dmtk_gpu_mt64_jump": (C.c_int, [C.c_uint64, C.c_int64, C.POINTER(C.c_uint64)]),
    "dmtk_gpu_tensor_download": (C.c_int, [T, dp]),
    "dmtk_gpu_tensor_slab": (C.c_int, [T, C.c_int64, C.c_int64, C.POINTER(T)]),
    "dmtk_gpu_tensor_pack_sym01": (C.c_int, [T, C.POINTER(T)]),
    "dmtk_gpu_mttkrp": (C.c_int, [T, C.c_int, dpp, i64p, i64p, C.c_int64, C.c_int, C.c_int, C.c_int, dp,
                                  C.POINTER(Times)]),
    "dmtk_gpu_mttkrp_device": (C.c_int, [T, C.POINTER(C.c_void_p), C.c_int64, C.c_int64, C.c_int, C.c_int,
                                         C.c_void_p, C.c_void_p]),
    "dmtk_gpu_choose_order": (C.c_int, [C.c_int, i64p, C.c_int64, C.POINTER(C.c_int)]),
    "dmtk_gpu_krp": (C.c_int, [C.c_int, C.c_int, dpp, i64p, C.c_int64, C.c_int, dp, C.POINTER(C.c_uint64)]),
    "dmtk_gpu_krp_device": (C.c_int, [C.c_int, C.POINTER(C.c_void_p), i64p, C.c_int64, C.c_void_p, C.c_void_p,
                                      C.c_void_p]),
    "dmtk_gpu_tensor_norm": (C.c_int, [T, dp]),
    "dmtk_gpu_gram_hadamard": (C.c_int, [C.c_int, C.c_int, i64p, C.c_int64, dpp, C.c_int64, dp]),
    "dmtk_gpu_solve_psd": (C.c_int, [C.c_int, C.c_int64, dp, C.c_int64, dp, dp]),
    "dmtk_gpu_cp_als": (C.c_int, [T, C.POINTER(AlsConfig), dp, dp, dp, dp, dp, C.POINTER(C.c_int),
                                  C.POINTER(C.c_int), dp]),
    "dmtk_gpu_als_iterate": (C.c_int, [T, C.POINTER(AlsConfig), C.c_int, dpp, i64p, i64p, dp, C.c_int64,
                                       C.c_double, C.c_int, dp, dp, dp]),
    "dmtk_gpu_fit": (C.c_int, [T, C.c_int, dpp, i64p, i64p, dp, C.c_int64, C.c_int, dp]),
    "dmtk_gpu_comm_unique_id": (C.c_int, [C.POINTER(C.c_ubyte)]),
    "dmtk_gpu_comm_init": (C.c_int, [C.POINTER(C.c_ubyte), C.c_int, C.c_int, C.c_int, C.POINTER(C.c_void_p)]),
    "dmtk_gpu_comm_free": (C.c_int, [C.c_void_p]),
    "dmtk_gpu_comm_loopback": (C.c_int, [C.c_int, C.c_int, C.POINTER(C.c_void_p)]),
    "dmtk_gpu_comm_info": (C.c_int, [C.c_void_p, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "dmtk_gpu_comm_allreduce": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]),
    "dmtk_gpu_mttkrp_sharded": (C.c_int, [C.c_void_p, T, C.POINTER(C.c_void_p), C.c_int64, C.c_int64, C.c_int,
                                          C.c_int, C.c_void_p, C.c_void_p]),
    "dmtk_gpu_cp_als_sharded": (C.c_int, [T, C.c_void_p, C.c_int64, C.c_int64, C.POINTER(AlsConfig), dp, dp, dp, dp,
                                          dp, C.POINTER(C.c_int), C.POINTER(C.c_int), dp]),
    "dmtk_gpu_fp64_peak": (C.c_int, [C.c_int, dp]),
    "dmtk_gpu_fp64_peak_sustained": (C.c_int, [C.c_int, C.c_double, dp]),
    "dmtk_gpu_launch_count": (C.c_int64, []),
    "dmtk_gpu_debug_trace": (C.c_int, [C.c_int, C.POINTER(C.c_uint64), C.c_int, C.POINTER(C.c_int)]),
    "dmtk_gpu_debug_cached_shapes": (C.c_int, [C.POINTER(C.c_int64)]),
}

for _name, (_res, _args) in _SIGS.items():
    _f = getattr(lib, _name)
    _f.restype = _res
    _f.argtypes = _args

EXPORTED = tuple(_SIGS)
