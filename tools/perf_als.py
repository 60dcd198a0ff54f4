"""CP-ALS timing on a BASELINE-shaped tensor (developer tool).

python tools/perf_als.py [--dims 100,100,1200,80] [--rank 20] [--iters 25]
Generates the fMRI-correlation-shaped tensor of BASELINE config 5 on the
device (symmetric 100x100 slices, unit diagonal, off-diagonals
tanh(N(0, 0.3^2))) and runs dmtk_gpu_cp_als.
"""
import argparse
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1708_08976_b200 as dg  # noqa: E402


def fmri_tensor(dims, seed=1):
    n0, n1 = dims[0], dims[1]
    rest = tuple(dims[2:])[::-1]
    g = torch.Generator(device="cuda").manual_seed(seed)
    z = torch.randn(rest + (n1, n0), dtype=torch.float64, device="cuda", generator=g) * 0.3
    z = torch.tanh(z)
    z = torch.triu(z, diagonal=1)
    z = z + z.transpose(-1, -2)
    z.diagonal(dim1=-2, dim2=-1).fill_(1.0)
    return z.reshape(-1).contiguous()  # natural order: mode 0 (region) fastest


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dims", default="100,100,1200,80")
    ap.add_argument("--rank", type=int, default=20)
    ap.add_argument("--iters", type=int, default=25)
    ap.add_argument("--tree", action="store_true", help="dimension-tree sweep (two tensor passes per iteration)")
    ap.add_argument("--sym", action="store_true", help="pack the modes-0/1 symmetric tensor (half the bytes)")
    args = ap.parse_args()
    dims = tuple(int(d) for d in args.dims.split(","))
    if len(dims) >= 3 and dims[0] == dims[1]:
        x = fmri_tensor(dims)
    else:  # other shapes: seeded U[0,1)
        g = torch.Generator(device="cuda").manual_seed(1)
        n = 1
        for d in dims:
            n *= d
        x = torch.rand(n, dtype=torch.float64, device="cuda", generator=g)
    t = dg.DenseTensor.from_device(dims, x.data_ptr(), owner=x)
    if args.sym:
        t = t.pack_symmetric01()
    dg.cp_als(t, dg.AlsConfig(rank=args.rank, max_iters=2, tol=0.0, seed=1, dimension_tree=args.tree))  # warm-up
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = dg.cp_als(t, dg.AlsConfig(rank=args.rank, max_iters=args.iters, tol=0.0, seed=1, dimension_tree=args.tree))
    wall = time.perf_counter() - t0
    per_iter = [r.total_seconds for r in res.trace.iters]
    print(json.dumps({"dims": dims, "rank": args.rank, "tree": args.tree, "sym": args.sym, "iters": len(per_iter), "wall_s": round(wall, 4),
                      "iter_ms_median": round(1e3 * sorted(per_iter)[len(per_iter) // 2], 3),
                      "mode_ms_iter1": [round(1e3 * v, 3) for v in res.trace.iters[-1].mode_time],
                      "final_fit": res.trace.iters[-1].fit.fit, "tensor_norm": res.trace.tensor_norm}))


if __name__ == "__main__":
    main()
