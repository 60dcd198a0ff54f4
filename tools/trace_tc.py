"""Per-CTA timeline of one streaming MTTKRP launch (developer tool).

DMTK_GPU_TRACE=1 python tools/trace_tc.py --config 200c16 [--flush]
For every mode: one warm call, then (after an optional L2 flush) one traced
call; prints, per timeline event, the min / median / max over CTAs in us
since the CTA's entry (%globaltimer), and the spread of CTA entry times.
"""
import argparse
import ctypes as C
import os
import statistics
import sys

import torch

os.environ.setdefault("DMTK_GPU_TRACE", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1708_08976_b200 as dg  # noqa: E402
from paper_1708_08976_b200 import MttkrpAlgo as A, TwoStepOrder as O  # noqa: E402
from paper_1708_08976_b200._lib import lib  # noqa: E402
from tools.perf_modes import CONFIGS  # noqa: E402

EVENTS = ["entry_ns", "prologue", "tma_first", "tma_last", "build_first", "build_last", "cons_first", "cons_loop",
          "cons_epi", "cons7_loop", "exit"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="200c16")
    ap.add_argument("--flush", action="store_true")
    ap.add_argument("--warm", type=int, default=1, help="untraced calls per mode before the traced one")
    a = ap.parse_args()
    dims, Cr = CONFIGS[a.config]
    n = 1
    for d in dims:
        n *= d
    g = torch.Generator(device="cuda").manual_seed(1)
    fs = [torch.rand((d, Cr), dtype=torch.float64, device="cuda", generator=g) for d in dims]
    t = dg.DenseTensor.generate(dims, 1)  # library-owned, as bench.py
    s = torch.cuda.current_stream()
    junk = torch.empty(64 << 20, dtype=torch.float64, device="cuda") if a.flush else None
    NS = 16 + 2 * 24
    buf = (C.c_uint64 * (1024 * NS))()
    for mode in range(len(dims)):
        out = torch.empty((dims[mode], Cr), dtype=torch.float64, device="cuda")
        call = lambda: dg.mttkrp_device(t, [f.data_ptr() for f in fs], Cr, mode, A.automatic, O.automatic,
                                        out.data_ptr(), s.cuda_stream)
        for _ in range(a.warm):
            call()
        torch.cuda.synchronize()
        if junk is not None:
            junk.fill_(1.0)
        call()
        torch.cuda.synchronize()
        nct = C.c_int(0)
        assert lib.dmtk_gpu_debug_trace(0, buf, 1024, C.byref(nct)) == 0
        rows = [list(buf[NS * k:NS * k + NS]) for k in range(nct.value)]
        t0 = min(r[0] for r in rows)
        ent = [(r[0] - t0) / 1e3 for r in rows]
        print(f"mode {mode}: {nct.value} CTAs; entry spread us min/med/max "
              f"{min(ent):.2f}/{statistics.median(ent):.2f}/{max(ent):.2f}")
        ghz = [(r[12] - r[11]) / (r[10] - r[0]) for r in rows if r[10] > r[0] and r[12] > r[11]]
        if ghz:
            print(f"  SM clock GHz (clock64 / globaltimer, entry to exit): median {statistics.median(ghz):.3f} "
                  f"min {min(ghz):.3f} max {max(ghz):.3f}")
        for ev, name in list(enumerate(EVENTS))[1:] + [(13, "build_start"), (14, "build_loaded")]:
            v = [(r[ev] - r[0]) / 1e3 for r in rows if r[ev]]
            if v:
                print(f"  {name:12s} us  min {min(v):7.2f}  med {statistics.median(v):7.2f}  max {max(v):7.2f}"
                      f"  (n={len(v)})")
        # per stage k of a CTA: loads issued / full barrier complete (median over CTAs)
        line_i, line_r = [], []
        for k in range(24):
            iv = [(r[16 + k] - r[0]) / 1e3 for r in rows if r[16 + k]]
            rv = [(r[40 + k] - r[0]) / 1e3 for r in rows if r[40 + k]]
            if iv:
                line_i.append(f"{statistics.median(iv):.2f}")
            if rv:
                line_r.append(f"{statistics.median(rv):.2f}")
        print("  stage issue us:", " ".join(line_i))
        print("  stage ready us:", " ".join(line_r))


if __name__ == "__main__":
    main()
