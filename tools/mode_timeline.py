"""Kernel timeline of repeated per-mode MTTKRP calls (developer tool): CUPTI
via torch.profiler; per-kernel busy time and idle gaps per call.

python tools/mode_timeline.py [--config 200c16] [--reps 20]
"""
import argparse
import os
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1708_08976_b200 as dg  # noqa: E402
from paper_1708_08976_b200 import MttkrpAlgo as A, TwoStepOrder as O  # noqa: E402
from tools.perf_modes import CONFIGS  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="200c16")
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    dims, C = CONFIGS[a.config]
    n = 1
    for d in dims:
        n *= d
    g = torch.Generator(device="cuda").manual_seed(1)
    x = torch.rand(n, dtype=torch.float64, device="cuda", generator=g)
    fs = [torch.rand((d, C), dtype=torch.float64, device="cuda", generator=g) for d in dims]
    t = dg.DenseTensor.from_device(dims, x.data_ptr(), owner=x)
    s = torch.cuda.current_stream()
    for mode in range(len(dims)):
        out = torch.empty((dims[mode], C), dtype=torch.float64, device="cuda")
        call = lambda: dg.mttkrp_device(t, [f.data_ptr() for f in fs], C, mode, A.automatic, O.automatic,
                                        out.data_ptr(), s.cuda_stream)
        call()
        torch.cuda.synchronize()
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            for _ in range(a.reps):
                call()
            torch.cuda.synchronize()
        ev = sorted([e for e in prof.events() if e.device_type.name == "CUDA"], key=lambda e: e.time_range.start)
        busy, gap, prev = {}, 0.0, None
        for e in ev:
            nm = e.name.split("(")[0].replace("void ", "").replace("dmtkg::", "")[:36]
            busy[nm] = busy.get(nm, 0.0) + e.time_range.elapsed_us()
            if prev is not None and e.time_range.start > prev:
                gap += e.time_range.start - prev
            prev = e.time_range.end if prev is None else max(prev, e.time_range.end)
        span = prev - ev[0].time_range.start
        print(f"mode {mode}: {span / a.reps:.1f} us/call, idle {gap / a.reps:.1f} us/call; " +
              ", ".join(f"{k} {v / a.reps:.1f}" for k, v in sorted(busy.items(), key=lambda kv: -kv[1])))


if __name__ == "__main__":
    main()
