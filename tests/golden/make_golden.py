"""Generate the golden fixtures from the UNMODIFIED reference library
(oracle/_ref/libdmtk_ref.so, compiled from /root/reference/proj/src by
oracle/Makefile). Run in the container that has /root/reference:

    python tests/golden/make_golden.py

Writes tests/golden/*.npz (small; committed). The GPU box has no
/root/reference, so tests there compare against these fixtures and the
prebuilt oracle/_ref library.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from oracle_bindings import Ref  # noqa: E402

REF_SHAPES = [(3, 4, 5), (2, 3, 4, 2), (2, 2, 2, 2, 2), (4, 1, 3), (6, 7), (9,), (10, 12, 14), (8, 6, 4, 6)]


def main():
    ref = Ref()
    out = {}
    # generators: bench.cpp:88-116 and cp_als.cpp:87-99
    out["gen_tensor_3x4x5_s17"] = ref.gen_tensor((3, 4, 5), 17)
    for k, m in enumerate(ref.gen_factors((3, 4, 5), 5, 23)):
        out[f"gen_factors_3x4x5_r5_s23_{k}"] = m
    f, lam = ref.kruskal_random((4, 5, 6), 3, 99)
    for k, m in enumerate(f):
        out[f"kruskal_4x5x6_r3_s99_{k}"] = m
    np.savez_compressed(os.path.join(HERE, "gen.npz"), **out)

    out = {}
    for si, dims in enumerate(REF_SHAPES):
        x = ref.gen_tensor(dims, 17)
        out[f"s{si}_dims"] = np.array(dims)
        out[f"s{si}_x"] = x
        for rank in (1, 2, 5):
            fs = ref.gen_factors(dims, rank, 23)
            for k, m in enumerate(fs):
                out[f"s{si}_r{rank}_f{k}"] = m
            for mode in range(len(dims)):
                out[f"s{si}_r{rank}_m{mode}_loops"] = ref.mttkrp_loops(x, dims, fs, mode)
                out[f"s{si}_r{rank}_m{mode}_auto"] = ref.mttkrp(x, dims, fs, mode, "automatic", "automatic", 4)
    np.savez_compressed(os.path.join(HERE, "mttkrp.npz"), **out)

    out = {}
    for si, dims in enumerate([(6,), (3, 4), (2, 3, 4), (3, 2, 2, 3), (2, 2, 3, 2, 2), (4, 1, 3), (1, 1, 5)]):
        for cols in (1, 3, 25):
            ins = [ref.gen_factors((d,), cols, 42 + z * 1000)[0] for z, d in enumerate(dims)]
            k, had = ref.krp(ins, 1)
            _, had_naive = ref.krp(ins, 1, naive=True)
            out[f"k{si}_c{cols}_dims"] = np.array(dims)
            for z, m in enumerate(ins):
                out[f"k{si}_c{cols}_in{z}"] = m
            out[f"k{si}_c{cols}_out"] = k
            out[f"k{si}_c{cols}_hadamards"] = np.array([had, had_naive])
    np.savez_compressed(os.path.join(HERE, "krp.npz"), **out)

    out = {}
    for ci, (dims, rank, iters, seed) in enumerate([((6, 5, 4), 3, 6, 7), ((7, 6, 5), 3, 8, 42),
                                                    ((8, 9, 10), 4, 40, 13), ((12, 10, 8, 6), 5, 10, 3),
                                                    ((40, 40, 12, 8), 20, 25, 1)]):
        x = ref.gen_tensor(dims, 31)
        r = ref.cp_als(x, dims, rank, iters, tol=0.0, seed=seed, threads=4)
        out[f"c{ci}_dims"] = np.array(dims)
        out[f"c{ci}_meta"] = np.array([rank, iters, seed])
        out[f"c{ci}_fits"] = r["fits"]
        out[f"c{ci}_lambda"] = r["lambda"]
        out[f"c{ci}_norm"] = np.array([r["norm_x"]])
    np.savez_compressed(os.path.join(HERE, "cpals.npz"), **out)
    print("wrote", sorted(os.listdir(HERE)))


if __name__ == "__main__":
    main()
