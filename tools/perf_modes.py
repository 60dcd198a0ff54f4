"""Per-mode MTTKRP timing on the device-resident path (developer tool).

python tools/perf_modes.py [--config 1000c25|AxBxC:rank,...] [--algos auto,one,left,right] [--reps 5]
Prints ms, tensor GB/s, FP64 TF/s and fraction of roofline per mode.
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1708_08976_b200 as dg  # noqa: E402
from paper_1708_08976_b200 import MttkrpAlgo as A, TwoStepOrder as O  # noqa: E402

CONFIGS = {
    "200c16": ((200, 200, 200), 16),
    "1000c25": ((1000, 1000, 1000), 25),
    "1000c50": ((1000, 1000, 1000), 50),
    "180c25": ((180, 180, 180, 180), 25),
    "64c32": ((64, 64, 64, 64, 64), 32),
    "fmri20": ((100, 100, 1200, 80), 20),
    "odd25": ((999, 1001, 997), 25),
    "1000c100": ((1000, 1000, 1000), 100),
    "km_short": ((100, 100, 100000), 25),
    "km_mid": ((1000, 100, 10000), 25),
}
ALGOS = {"auto": (A.automatic, O.automatic), "one": (A.one_step, O.automatic), "left": (A.two_step, O.left),
         "right": (A.two_step, O.right), "base": (A.baseline, O.automatic)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="1000c25")
    ap.add_argument("--algos", default="auto")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--bw", type=float, default=6455.9)
    ap.add_argument("--modes", default="")
    ap.add_argument("--flush", action="store_true", help="write 512 MB before every timed call (L2 flush, as bench.py)")
    ap.add_argument("--upload", action="store_true", help="upload through the host API (padded odd layouts)")
    ap.add_argument("--wrap", action="store_true", help="borrow a torch tensor (dmtk_gpu_tensor_wrap)")
    ap.add_argument("--profile", action="store_true",
                    help="after warm-up, run one call per mode between cudaProfilerStart/Stop (for ncu "
                         "--profile-from-start off) and skip the timing")
    args = ap.parse_args()
    peak = dg.fp64_peak_tflops()
    for cfg in args.config.split(","):
        if cfg in CONFIGS:
            dims, C = CONFIGS[cfg]
        else:  # "AxBxC:rank"
            shp, rk = cfg.split(":")
            dims, C = tuple(int(v) for v in shp.split("x")), int(rk)
        n = 1
        for d in dims:
            n *= d
        g = torch.Generator(device="cuda").manual_seed(1)
        x = torch.rand(n, dtype=torch.float64, device="cuda", generator=g)
        fs = [torch.rand((d, C), dtype=torch.float64, device="cuda", generator=g) for d in dims]
        if args.upload:
            t = dg.DenseTensor(dims, x.cpu().numpy())
        elif args.wrap:
            t = dg.DenseTensor.from_device(dims, x.data_ptr(), owner=x)
        else:  # library-owned, as bench.py (dmtk_gpu_tensor_generate)
            del x
            t = dg.DenseTensor.generate(dims, 1)
        s = torch.cuda.current_stream()
        modes = [int(m) for m in args.modes.split(",")] if args.modes else range(len(dims))
        modes = [m if m >= 0 else len(dims) + m for m in modes]
        for mode in modes:
            out = torch.empty((dims[mode], C), dtype=torch.float64, device="cuda")
            for an in args.algos.split(","):
                algo, order = ALGOS[an]
                if algo == A.two_step and mode in (0, len(dims) - 1):
                    continue
                call = lambda: dg.mttkrp_device(t, [f.data_ptr() for f in fs], C, mode, algo, order, out.data_ptr(),
                                                s.cuda_stream)
                call()
                torch.cuda.synchronize()
                if args.profile:
                    call()
                    torch.cuda.synchronize()
                    torch.cuda.profiler.start()
                    call()
                    torch.cuda.synchronize()
                    torch.cuda.profiler.stop()
                    continue
                if args.flush:
                    junk = torch.empty(64 << 20, dtype=torch.float64, device="cuda")
                    tot = 0.0
                    for _ in range(args.reps):
                        junk.fill_(1.0)
                        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                        e0.record()
                        call()
                        e1.record()
                        torch.cuda.synchronize()
                        tot += e0.elapsed_time(e1)
                    ms = tot / args.reps
                    del junk
                else:
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    for _ in range(args.reps):
                        call()
                    e1.record()
                    torch.cuda.synchronize()
                    ms = e0.elapsed_time(e1) / args.reps
                gbs = 8 * n / (ms * 1e-3) / 1e9
                tfs = 2 * n * C / (ms * 1e-3) / 1e12
                roof = max(8 * n / (args.bw * 1e9), 2 * n * C / (peak * 1e12))
                print(json.dumps({"config": cfg, "mode": mode, "algo": an, "ms": round(ms, 4), "GBs": round(gbs, 1),
                                  "TFs": round(tfs, 2), "frac": round(roof / (ms * 1e-3), 3),
                                  "peak_tf": round(peak, 2)}), flush=True)
        del fs, t
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
