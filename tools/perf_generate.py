"""On-device gen_tensor timing (developer tool): first call (host jump-ahead
polynomials + generation) and a repeat (cached polynomials).

python tools/perf_generate.py
"""
import time, sys, os
sys.path.insert(0, os.getcwd())
import torch
import paper_1708_08976_b200 as dg
for dims in [(1000, 1000, 1000), (180, 180, 180, 180), (1000, 1000, 1000)]:
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    t = dg.DenseTensor.generate(dims, 11)
    dt = time.perf_counter() - t0
    n = 1
    for d in dims: n *= d
    print(dims, f"{dt*1e3:.1f} ms  {8*n/dt/1e9:.1f} GB/s", flush=True)
    t.free() if hasattr(t, "free") else None
    del t
