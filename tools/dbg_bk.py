import os, sys, json
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np
import paper_1708_08976_b200 as dg
from oracle_bindings import Oracle
orc = Oracle()
dims = tuple(int(v) for v in sys.argv[1].split("x")); C = int(sys.argv[2]); mode = int(sys.argv[3])
algo = dg.MttkrpAlgo(int(sys.argv[4])) if len(sys.argv) > 4 else dg.MttkrpAlgo.automatic
x = orc.gen_tensor(dims, 1); f = orc.gen_factors(dims, C, 2)
t = dg.DenseTensor(dims, x)
got = dg.mttkrp(dg.MttkrpRequest(t, f, mode, algo)).m
want = orc.mttkrp(x, dims, f, mode)
print(json.dumps({"dims": dims, "C": C, "mode": mode, "err": float(np.linalg.norm(got - want) / np.linalg.norm(want))}))
