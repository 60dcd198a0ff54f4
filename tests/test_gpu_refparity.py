"""Reference parity at every BASELINE.json configuration, on identical bytes.

Each configuration's tensor and factors are generated once on the device
(dmtk_gpu_tensor_generate: the reference's gen_tensor stream, bitwise, with the
configuration's value transform -- tests/test_gpu_generate.py pins both against
the reference library and the host restatement), read back, and handed to the
UNMODIFIED reference library (oracle/_ref/libdmtk_ref.so) on all host cores.
The GPU runs the same bytes through the production path (host-buffer
dmtk_gpu_mttkrp: planner, measured view selection, CSR reduction). The
reference's own gate is relative Frobenius <= 1e-12 (bench.cpp:20, 301-313;
test_mttkrp.cpp:134); CP-ALS fits agree to <= 1e-9 (BASELINE north_star).

Configs (BASELINE.json): 1000^3 U[0,1) at C = 25 and 50; 180^4 N(0,1) tensor
and factors at C = 25; 64^5 U[-1,1) tensor and factors at C = 32; the
fMRI-shaped 100x100x1200x80 symmetric-slice tensor at C = 20 (MTTKRP of every
mode, and 25 CP-ALS iterations of the per-mode, dimension-tree and
symmetric-packed sweeps against the reference's cp_als).
"""
import os

import numpy as np
import pytest

import paper_1708_08976_b200 as dg
from paper_1708_08976_b200 import MttkrpAlgo as A, TwoStepOrder as O

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

THREADS = os.cpu_count() or 1

# name: dims, rank, tensor distribution, factor distribution
CONFIGS = {
    "1000c25": ((1000, 1000, 1000), 25, "uniform", "uniform"),
    "1000c50": ((1000, 1000, 1000), 50, "uniform", "uniform"),
    "180c25": ((180, 180, 180, 180), 25, "normal", "normal"),
    "64c32": ((64, 64, 64, 64, 64), 32, "signed", "signed"),
    "fmri20": ((100, 100, 1200, 80), 20, "symslice", "uniform"),
}


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def variants(mode, n):
    """(gpu algo, gpu order, reference algo, reference order) per mode."""
    if mode in (0, n - 1):
        return [(A.automatic, O.automatic, "automatic", "automatic")]
    return [(A.automatic, O.automatic, "automatic", "automatic"),
            (A.one_step, O.automatic, "one_step", "automatic"),
            (A.two_step, O.left, "two_step", "left"),
            (A.two_step, O.right, "two_step", "right")]


@pytest.mark.parametrize("name", sorted(CONFIGS))
def test_mttkrp_matches_reference_full_size(ref, name):
    dims, C, tdist, fdist = CONFIGS[name]
    t = dg.DenseTensor.generate(dims, 1, tdist)
    x = t.download()
    fs = [f.download().reshape(d, C) for f, d in zip(dg.generate_factors(dims, C, 2, fdist), dims)]
    worst = 0.0
    for mode in range(len(dims)):
        for ga, go, ra, ro in variants(mode, len(dims)):
            got = dg.mttkrp(dg.MttkrpRequest(t, fs, mode, ga, go)).m
            want = ref.mttkrp(x, dims, fs, mode, ra, ro, THREADS)
            err = rel(got, want)
            worst = max(worst, err)
            assert err <= 1e-12, (name, mode, ra, ro, err)
    print(f"{name}: worst relative Frobenius error vs the reference {worst:.2e}")


def test_baseline_algorithm_full_size(ref):
    """The reference's baseline (explicit matricisation + full KRP) on an
    interior mode of config 2, same bytes."""
    dims, C = (1000, 1000, 1000), 25
    t = dg.DenseTensor.generate(dims, 1)
    x = t.download()
    fs = [f.download().reshape(d, C) for f, d in zip(dg.generate_factors(dims, C, 2), dims)]
    got = dg.mttkrp(dg.MttkrpRequest(t, fs, 1, A.baseline)).m
    want = ref.mttkrp(x, dims, fs, 1, "baseline", "automatic", THREADS)
    assert rel(got, want) <= 1e-12


def test_cp_als_fmri_full_size_matches_reference(ref):
    """BASELINE config 5: 25 CP-ALS iterations at rank 20 from
    KruskalModel::random(seed) on the fMRI-shaped symmetric-slice tensor; the
    reference's fits (cp_als.cpp:174-200) against the GPU's per-mode sweep,
    dimension tree and symmetric-packed tree."""
    dims, C, iters = (100, 100, 1200, 80), 20, 25
    t = dg.DenseTensor.generate(dims, 1, "symslice")
    x = t.download()
    want = ref.cp_als(x, dims, C, iters, tol=0.0, seed=1, threads=THREADS)
    del x
    assert len(want["fits"]) == iters
    cfg = dg.AlsConfig(rank=C, max_iters=iters, tol=0.0, seed=1)
    runs = {"per_mode": dg.cp_als(t, cfg),
            "tree": dg.cp_als(t, dg.AlsConfig(rank=C, max_iters=iters, tol=0.0, seed=1, dimension_tree=True))}
    tp = t.pack_symmetric01()
    runs["packed"] = dg.cp_als(tp, cfg)
    tp.release()
    for k, r in runs.items():
        fits = np.array([it.fit.fit for it in r.trace.iters])
        assert len(fits) == iters, k
        diff = np.max(np.abs(fits - want["fits"]))
        assert diff <= 1e-9, (k, diff)
        assert abs(r.trace.tensor_norm - want["norm_x"]) <= 1e-12 * want["norm_x"], k
    # the final factors of the reference's sweep agree too (well conditioned here)
    for u, v in zip(runs["per_mode"].model.factors, want["factors"]):
        assert rel(u, v) <= 1e-7


def collinear_model(dims, rank, delta, seed):
    """A rank-`rank` model whose components 0 and 1 are near-collinear in
    every mode (column 1 = column 0 + delta * noise), and a tensor close to
    it: near that model the Gram-Hadamard systems of every ALS mode update have
    condition numbers ~ 1 / delta^2."""
    rng = np.random.default_rng(seed)
    fs = []
    for d in dims:
        a = rng.random((d, rank))
        a[:, 1] = a[:, 0] + delta * rng.standard_normal(d)
        fs.append(a)
    return fs


def kappa(factors, skip):
    h = np.ones((factors[0].shape[1],) * 2)
    for k, u in enumerate(factors):
        if k != skip:
            h = h * (u.T @ u)
    return np.linalg.cond(h)


@pytest.mark.parametrize("dims,delta", [((30, 28, 26), 1e-4), ((30, 28, 26), 1e-5), ((12, 11, 10, 9), 2e-5)])
def test_als_iterate_ill_conditioned_matches_reference(ref, oracle, dims, delta):
    """Near-collinear factors (kappa(H) ~ 1e7 - 1e10, still above the
    1e-12 * trace Cholesky floor of solve_psd, linalg.cpp:330-387): the GPU's
    ALS solve must track the reference's Cholesky substitution sweep by sweep
    (dmtk::als_iterate, cp_als.hpp:74-75)."""
    rank = 3
    a = collinear_model(dims, rank, delta, 7)
    x = oracle.reconstruct(a, np.ones(rank))
    x = x + 1e-3 * np.random.default_rng(8).standard_normal(x.size)
    nx = ref.tensor_norm(x, dims)
    t = dg.DenseTensor(dims, x)
    gm = dg.KruskalModel([u.copy() for u in a], np.ones(rank))
    rf, rl = [u.copy() for u in a], np.ones(rank)
    kmax = 0.0
    for it in range(1, 16):
        kmax = max(kmax, max(kappa(rf, n) for n in range(len(dims))))
        rec = dg.als_iterate(t, gm, dg.AlsConfig(rank=rank), nx, it)
        rf, rl, f4, _ = ref.als_iterate(x, dims, rf, rl, nx, it)
        assert rec.fit.defined and f4[3] == 1.0
        assert abs(rec.fit.fit - f4[0]) <= 1e-9, (it, rec.fit.fit, f4[0])
        for u, v in zip(gm.factors, rf):
            # an ill-conditioned solve amplifies rounding by ~kappa: both
            # implementations carry that much noise
            assert rel(u, v) <= max(1e-9, 1e-14 * kmax), (it, rel(u, v), kmax)
    assert kmax >= 1e7
