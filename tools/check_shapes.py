"""Developer check: GPU MTTKRP vs a numpy einsum reference for given shapes,
every mode and algorithm, relative Frobenius error (no oracle library needed).

python tools/check_shapes.py 40x40x12x8:20 180x180x180:25 ...
"""
import sys
import os

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1708_08976_b200 as dg  # noqa: E402
from paper_1708_08976_b200 import MttkrpAlgo as A, TwoStepOrder as O  # noqa: E402


def ref(x, dims, f, mode):
    X = x.reshape(dims[::-1])  # natural order: mode 0 fastest -> last numpy axis
    N = len(dims)
    letters = "abcdefghijklm"[:N]
    ax = letters[::-1]  # numpy axis k <-> mode N-1-k
    ops = [X]
    sub = [ax]
    for k in range(N):
        if k != mode:
            ops.append(f[k])
            sub.append(letters[k] + "z")
    expr = ",".join(sub) + "->" + letters[mode] + "z"
    return np.einsum(expr, *ops, optimize=True)


def main():
    rng = np.random.default_rng(7)
    bad = 0
    for spec in sys.argv[1:]:
        shp, C = spec.split(":")
        dims = tuple(int(v) for v in shp.split("x"))
        C = int(C)
        x = rng.uniform(-1, 1, int(np.prod(dims)))
        f = [rng.uniform(-1, 1, (d, C)) for d in dims]
        t = dg.DenseTensor(dims, x)
        for mode in range(len(dims)):
            want = ref(x, dims, f, mode)
            algos = [(A.one_step, O.automatic), (A.baseline, O.automatic)]
            if 0 < mode < len(dims) - 1:
                algos += [(A.two_step, O.left), (A.two_step, O.right)]
            for algo, order in algos:
                got = dg.mttkrp(dg.MttkrpRequest(t, f, mode, algo, order, 1)).m
                e = np.linalg.norm(got - want) / np.linalg.norm(want)
                flag = "" if e <= 1e-12 else "  <-- FAIL"
                bad += bool(flag)
                print(f"{spec} mode {mode} {algo.name}/{order.name}: {e:.2e}{flag}", flush=True)
    print("failures:", bad)


if __name__ == "__main__":
    main()
