"""Standalone Khatri-Rao product timing on the device-resident path
(developer tool): written GB/s vs the HBM roofline (bytes = 8 * rows * C
written).

python tools/perf_krp.py [--cases 200x200x200:16,1000x1000:25,64x64x64x64:32]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1708_08976_b200 as dg  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", default="200x200x200:16,1000x1000:25,64x64x64x64:32,1000x1000:50")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--bw", type=float, default=6455.9)
    a = ap.parse_args()
    for case in a.cases.split(","):
        shp, C = case.split(":")
        rows = [int(v) for v in shp.split("x")]
        C = int(C)
        total = 1
        for r in rows:
            total *= r
        g = torch.Generator(device="cuda").manual_seed(3)
        ins = [torch.rand((r, C), dtype=torch.float64, device="cuda", generator=g) for r in rows]
        out = torch.empty((total, C), dtype=torch.float64, device="cuda")
        scr_rows = 1
        for r in rows[:-1]:
            scr_rows *= r
        scr = torch.empty((2 * scr_rows, C), dtype=torch.float64, device="cuda")
        s = torch.cuda.current_stream()
        call = lambda: dg.krp_device([t.data_ptr() for t in ins], rows, C, out.data_ptr(), scr.data_ptr(),
                                     s.cuda_stream)
        call()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.reps):
            call()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.reps
        gb = 8.0 * total * C / 1e9
        print(json.dumps({"case": case, "rows": total, "ms": round(ms, 4), "GBs_written": round(gb / (ms * 1e-3), 1),
                          "frac": round(gb / (a.bw) / (ms * 1e-3), 3)}), flush=True)


if __name__ == "__main__":
    main()
