import os, sys, threading
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np, torch
import paper_1708_08976_b200 as dg
from paper_1708_08976_b200.distributed import loopback_comms, shard_bounds
from oracle_bindings import Oracle
orc = Oracle()
dims, C = (30, 20, 17), 9
x = orc.gen_tensor(dims, 3); f = orc.gen_factors(dims, C, 4)
t = dg.DenseTensor(dims, x)
N = 3
want = [dg.mttkrp(dg.MttkrpRequest(t, f, m)).m for m in range(N)]
for P in [int(v) for v in os.environ.get('PS', '1,2,3').split(',')]:
    comms = loopback_comms(P)
    print("P", P, "fused", [c.fused for c in comms])
    slabs, outs, facs = [], [], []
    for r in range(P):
        lo, hi = shard_bounds(dims[-1], P, r)
        slabs.append(t.slab(lo, hi))
        fr = [torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in f[:-1]] + [torch.from_numpy(np.ascontiguousarray(f[-1][lo:hi])).cuda()]
        facs.append(fr)
        outs.append([torch.zeros((dims[m] if m < N - 1 else hi - lo, C), dtype=torch.float64, device="cuda") for m in range(N)])
        # single-slab reference partials
    torch.cuda.synchronize()
    rs = [torch.cuda.Stream() for _ in range(P)]
    def work(r):
      seq = [int(v) for v in os.environ.get("SEQ", "").split(",") if v] or list(range(N)) * int(os.environ.get("ROUNDS", "1"))
      for rnd in range(1):
        for m in seq:
            comms[r].mttkrp(slabs[r], [a.data_ptr() for a in facs[r]], C, m, outs[r][m].data_ptr(),
                            rs[r].cuda_stream if os.environ.get("STREAMS") else 0)
      torch.cuda.synchronize()
    ts = [threading.Thread(target=work, args=(r,)) for r in range(P)]
    [th.start() for th in ts]; [th.join() for th in ts]
    torch.cuda.synchronize()
    last = np.concatenate([outs[r][N - 1].cpu().numpy() for r in range(P)], axis=0)
    print(" last mode relerr", np.linalg.norm(last - want[N - 1]) / np.linalg.norm(want[N - 1]))
    for m in range(N - 1):
        for r in range(P):
            g = outs[r][m].cpu().numpy()
            print(" mode", m, "rank", r, "relerr", np.linalg.norm(g - want[m]) / np.linalg.norm(want[m]), "ratio", (g / want[m]).mean())
    # direct partials per slab
    for m in range(N - 1):
        parts = []
        for r in range(P):
            lo, hi = shard_bounds(dims[-1], P, r)
            parts.append(dg.mttkrp(dg.MttkrpRequest(slabs[r], f[:-1] + [f[-1][lo:hi]], m)).m)
        print(" direct sum mode", m, np.linalg.norm(sum(parts) - want[m]) / np.linalg.norm(want[m]))
    for s in slabs: s.release()
    for c in comms: c.close()
