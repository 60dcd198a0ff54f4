"""Interleaved A/B timing of two builds of libdmtk_gpu.so in one process
(developer tool). Both libraries are loaded side by side (RTLD_LOCAL), wrap
the same device tensor and factors, and are timed alternately per mode so
clock and thermal drift fall on both equally.

python tools/ab_libs.py A.so B.so --config 1000c25,fmri20 [--rounds 5] [--reps 5]
Prints per mode the median ms of each build and B's speed-up over A.
"""
import argparse
import ctypes as C
import json
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tools.perf_modes import CONFIGS  # noqa: E402

T = C.c_void_p


def load(path):
    lib = C.CDLL(os.path.abspath(path), mode=C.RTLD_LOCAL)
    lib.dmtk_gpu_tensor_wrap.argtypes = [C.c_int, C.c_int, C.POINTER(C.c_int64), C.c_void_p, C.POINTER(T)]
    lib.dmtk_gpu_tensor_free.argtypes = [T]
    lib.dmtk_gpu_mttkrp_device.argtypes = [T, C.POINTER(C.c_void_p), C.c_int64, C.c_int64, C.c_int, C.c_int,
                                           C.c_void_p, C.c_void_p]
    lib.dmtk_gpu_last_error.restype = C.c_char_p
    return lib


def check(lib, rc):
    if rc != 0:
        raise RuntimeError(lib.dmtk_gpu_last_error().decode())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("a")
    ap.add_argument("b")
    ap.add_argument("--config", default="1000c25")
    ap.add_argument("--rounds", type=int, default=5)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--modes", default="")
    ap.add_argument("--flush", action="store_true")
    args = ap.parse_args()
    libs = [load(args.a), load(args.b)]
    for cfg in args.config.split(","):
        if cfg in CONFIGS:
            dims, C_ = CONFIGS[cfg]
        else:
            shp, rk = cfg.split(":")
            dims, C_ = tuple(int(v) for v in shp.split("x")), int(rk)
        n = int(np.prod(dims))
        g = torch.Generator(device="cuda").manual_seed(1)
        x = torch.rand(n, dtype=torch.float64, device="cuda", generator=g)
        fs = [torch.rand((d, C_), dtype=torch.float64, device="cuda", generator=g) for d in dims]
        d64 = (C.c_int64 * len(dims))(*dims)
        hs = []
        for lib in libs:
            h = T()
            check(lib, lib.dmtk_gpu_tensor_wrap(0, len(dims), d64, C.c_void_p(x.data_ptr()), C.byref(h)))
            hs.append(h)
        ptrs = (C.c_void_p * len(dims))(*[f.data_ptr() for f in fs])
        s = torch.cuda.current_stream()
        modes = [int(m) for m in args.modes.split(",")] if args.modes else range(len(dims))
        for mode in modes:
            out = torch.empty((dims[mode], C_), dtype=torch.float64, device="cuda")
            calls = [lambda lib=lib, h=h: check(lib, lib.dmtk_gpu_mttkrp_device(h, ptrs, C_, mode, 3, 0,  # automatic
                                                                                 C.c_void_p(out.data_ptr()),
                                                                                 C.c_void_p(s.cuda_stream)))
                     for lib, h in zip(libs, hs)]
            for c in calls:  # plans, slot maps, measured view selection
                c()
                c()
            torch.cuda.synchronize()
            ts = [[], []]
            junk = torch.empty(64 << 20, dtype=torch.float64, device="cuda") if args.flush else None
            for _ in range(args.rounds):
                for k, c in enumerate(calls):
                    if junk is not None:  # L2 flush before every timed call (as bench.py's 200c16 block)
                        tot = 0.0
                        for _ in range(args.reps):
                            junk.fill_(1.0)
                            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                            e0.record()
                            c()
                            e1.record()
                            torch.cuda.synchronize()
                            tot += e0.elapsed_time(e1)
                        ts[k].append(tot / args.reps)
                        continue
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    for _ in range(args.reps):
                        c()
                    e1.record()
                    torch.cuda.synchronize()
                    ts[k].append(e0.elapsed_time(e1) / args.reps)
            del junk
            ma, mb = statistics.median(ts[0]), statistics.median(ts[1])
            print(json.dumps({"config": cfg, "mode": mode, "a_ms": round(ma, 4), "b_ms": round(mb, 4),
                              "b_speedup_pct": round(100 * (ma / mb - 1), 2),
                              "spread_pct": round(100 * (max(ts[0] + ts[1]) / min(ts[0] + ts[1]) - 1), 2)}),
                  flush=True)
        for lib, h in zip(libs, hs):
            lib.dmtk_gpu_tensor_free(h)
        del x, fs
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
