"""Regression fixture for the seeded value distributions of the BASELINE
configs (oracle/oracle.c orc_gen_dist; device: csrc/gen_dist.cu).

The uniform stream under every distribution is the reference's gen_tensor
(pinned bitwise by gen.npz / the reference library); the transforms are
restated formulas (Box-Muller, tanh) pinned against numpy's libm within
1e-12 by tests/test_dist.py. This file freezes the exact bytes so a compiler
or flag change (an FMA contraction) cannot move them silently:

    python tests/golden/make_dist_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from oracle_bindings import Oracle  # noqa: E402

CASES = [("signed", (7, 6, 5), 11), ("normal", (9, 8, 7), 12), ("normal", (5, 3), 13),
         ("symslice", (6, 6, 4, 3), 14), ("symslice", (5, 5, 7), 15)]


def main():
    orc = Oracle()
    out = {}
    for dist, dims, seed in CASES:
        key = f"{dist}_{'x'.join(map(str, dims))}_s{seed}"
        out[key] = orc.gen_dist(dims, seed, dist, threads=1)
    np.savez_compressed(os.path.join(HERE, "dist.npz"), **out)


if __name__ == "__main__":
    main()
