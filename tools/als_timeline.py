"""Kernel timeline of a CP-ALS run (developer tool): CUPTI via torch.profiler,
per-iteration kernel busy time vs wall, and the largest idle gaps.

python tools/als_timeline.py [--dims 100,100,1200,80] [--rank 20] [--iters 6]
"""
import argparse
import os
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1708_08976_b200 as dg  # noqa: E402
from tools.perf_als import fmri_tensor  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dims", default="100,100,1200,80")
    ap.add_argument("--rank", type=int, default=20)
    ap.add_argument("--iters", type=int, default=6)
    ap.add_argument("--tree", action="store_true")
    ap.add_argument("--sym", action="store_true")
    a = ap.parse_args()
    dims = tuple(int(d) for d in a.dims.split(","))
    x = fmri_tensor(dims)
    t = dg.DenseTensor.from_device(dims, x.data_ptr(), owner=x)
    if a.sym:
        t = t.pack_symmetric01()
    cfg = lambda n: dg.AlsConfig(rank=a.rank, max_iters=n, tol=0.0, seed=1, dimension_tree=a.tree)
    dg.cp_als(t, cfg(2))
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        dg.cp_als(t, cfg(a.iters))
        torch.cuda.synchronize()
    ev = [e for e in prof.events() if e.device_type.name == "CUDA"]
    ev.sort(key=lambda e: e.time_range.start)
    t0 = ev[0].time_range.start
    busy = {}
    gaps = []
    prev_end = None
    for e in ev:
        s, d = e.time_range.start, e.time_range.end
        nm = e.name.split("(")[0].replace("void ", "").replace("dmtkg::", "")[:40]
        busy[nm] = busy.get(nm, 0.0) + (d - s)
        if prev_end is not None and s > prev_end:
            gaps.append((s - prev_end, nm, s - t0))
        prev_end = max(prev_end or 0, d)
    span = prev_end - t0
    print(f"span {span:.0f} us, kernels busy {sum(busy.values()):.0f} us, idle {sum(g[0] for g in gaps):.0f} us")
    for k, v in sorted(busy.items(), key=lambda kv: -kv[1])[:14]:
        print(f"  {k:40s} {v:9.1f} us")
    # steady state: the second half of the span (graph replays only)
    half = t0 + span / 2
    late = [g for g in gaps if g[2] + t0 >= half]
    late_busy = sum(e.time_range.end - e.time_range.start for e in ev if e.time_range.start >= half)
    print(f"second half: idle {sum(g[0] for g in late):.0f} us, busy {late_busy:.0f} us, gaps {len(late)}")
    lt = {}
    for g, nm, _ in late:
        lt[nm] = lt.get(nm, 0.0) + g
    for k, v in sorted(lt.items(), key=lambda kv: -kv[1])[:12]:
        print(f"  late idle before {k:40s} {v:9.1f} us")
    gaps.sort(reverse=True)
    print("largest gaps (us, next kernel, at):")
    for g in gaps[:20]:
        print(f"  {g[0]:8.1f} before {g[1]:40s} at {g[2]:9.1f}")
    # gap histogram
    tot = {}
    for g, nm, _ in gaps:
        tot[nm] = tot.get(nm, 0.0) + g
    print("idle before each kernel kind:")
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1])[:10]:
        print(f"  {k:40s} {v:9.1f} us")


if __name__ == "__main__":
    main()
