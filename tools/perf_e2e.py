"""Breakdown of bench.py's end-to-end step (developer tool): raw pinned H2D
bandwidth, dmtk_gpu_tensor_upload, each host-buffer dmtk_gpu_mttkrp call and
dmtk_gpu_tensor_free, wall-clocked with a device sync around each piece.

python tools/perf_e2e.py [--config 1000c25] [--reps 3]
"""
import argparse
import ctypes as Cc
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1708_08976_b200 import _lib  # noqa: E402
from tools.perf_modes import CONFIGS  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="1000c25")
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    dims, C = CONFIGS[a.config]
    N = len(dims)
    n = int(np.prod(dims))
    lib = _lib.lib
    g = torch.Generator().manual_seed(1)
    hx = torch.empty(n, dtype=torch.float64, pin_memory=True)
    hx.uniform_(generator=g)
    dx = torch.empty(n, dtype=torch.float64, device="cuda")
    hf = [np.random.default_rng(2 + k).random((d, C)) for k, d in enumerate(dims)]
    fptr = (_lib.dp * N)(*[f.ctypes.data_as(_lib.dp) for f in hf])
    d64 = np.asarray(dims, dtype=np.int64)
    cols = np.full(N, C, dtype=np.int64)
    outs = [np.empty((d, C)) for d in dims]

    def timed(fn):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = fn()
        torch.cuda.synchronize()
        return (time.perf_counter() - t0) * 1e3, r

    def upload():
        h = Cc.c_void_p()
        assert lib.dmtk_gpu_tensor_upload(0, N, d64.ctypes.data_as(_lib.i64p), Cc.cast(hx.data_ptr(), _lib.dp),
                                          Cc.byref(h)) == 0, lib.dmtk_gpu_last_error()
        return h

    def mttkrp(h, m):
        assert lib.dmtk_gpu_mttkrp(h, N, fptr, d64.ctypes.data_as(_lib.i64p), cols.ctypes.data_as(_lib.i64p), m, 3,
                                   0, 1, outs[m].ctypes.data_as(_lib.dp), None) == 0, lib.dmtk_gpu_last_error()

    h = upload()  # warm-up: pool, plans, view selection
    for m in range(N):
        mttkrp(h, m)
    lib.dmtk_gpu_tensor_free(h)
    for _ in range(a.reps):
        raw, _ = timed(lambda: dx.copy_(hx, non_blocking=True))
        up, h = timed(upload)
        ms = [timed(lambda: mttkrp(h, m))[0] for m in range(N)]
        warm = [timed(lambda: mttkrp(h, m))[0] for m in range(N)]  # same handle again: per-handle caches warm
        fr, _ = timed(lambda: lib.dmtk_gpu_tensor_free(h))
        print(json.dumps({"config": a.config, "raw_h2d_ms": round(raw, 2), "raw_h2d_GBs": round(8 * n / raw / 1e6, 1),
                          "upload_ms": round(up, 2), "mttkrp_ms": [round(x, 3) for x in ms],
                          "mttkrp_same_handle_ms": [round(x, 3) for x in warm],
                          "free_ms": round(fr, 3), "step_ms": round(up + sum(ms) + fr, 2)}), flush=True)


if __name__ == "__main__":
    main()
