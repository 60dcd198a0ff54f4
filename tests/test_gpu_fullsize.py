"""Parity at BASELINE.json's full sizes through size-independent properties.

The direct comparison with the reference library on identical bytes at every
8 GB configuration is tests/test_gpu_refparity.py (the reference takes ~0.4 s
per 8 GB pass on 16 host threads). These configurations (1000^3 at C = 25 and
50, 180^4 at C = 25, 64^5 at C = 32, the fMRI-shaped 100x100x1200x80 at C = 20)
are additionally checked by properties that need no reference contraction:

* closed form on a rank-one tensor X = a_0 o a_1 o ... o a_{N-1}: the MTTKRP of
  mode n is a_n (prod_{k != n} a_k^T U_k) (a column-wise product of N-1 length-C
  vectors), computed in float64 on the host; every mode, every algorithm and
  order, through the same planner (measured view selection included, the
  tensors are above its 256 MB threshold);
* linearity on a uniform random tensor: scaling the columns of one input
  factor by w scales the result's columns by w;
* CP-ALS on the full fMRI-shaped tensor: the per-mode sweep, the dimension tree
  and the symmetric-packed tree give the same fits (within 1e-9, the
  reference's CP-ALS tolerance), and the fit does not decrease.

Tolerance: relative Frobenius error <= 1e-12 (reference test_mttkrp.cpp:134).
"""
import numpy as np
import pytest
import torch

import paper_1708_08976_b200 as dg
from paper_1708_08976_b200 import MttkrpAlgo as A, TwoStepOrder as O

pytestmark = pytest.mark.gpu

CONFIGS = [((1000, 1000, 1000), 25), ((1000, 1000, 1000), 50), ((180, 180, 180, 180), 25),
           ((64, 64, 64, 64, 64), 32), ((100, 100, 1200, 80), 20)]


def rank_one(dims, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    vecs = [torch.rand(d, dtype=torch.float64, device="cuda", generator=g) + 0.5 for d in dims]
    x = vecs[-1]
    for v in reversed(vecs[:-1]):  # natural order: mode 0 fastest
        x = torch.outer(x, v).reshape(-1)
    return x.contiguous(), [v.cpu().numpy() for v in vecs]


def algos_for(mode, N):
    out = [(A.automatic, O.automatic), (A.one_step, O.automatic)]
    if 0 < mode < N - 1:
        out += [(A.two_step, O.left), (A.two_step, O.right)]
    return out


@pytest.mark.parametrize("dims,C", CONFIGS, ids=["1000c25", "1000c50", "180c25", "64c32", "fmri20"])
def test_rank_one_closed_form(dims, C):
    N = len(dims)
    x, vecs = rank_one(dims, seed=3)
    t = dg.DenseTensor.from_device(dims, x.data_ptr(), owner=x)
    g = torch.Generator(device="cuda").manual_seed(4)
    fs = [torch.rand((d, C), dtype=torch.float64, device="cuda", generator=g) - 0.25 for d in dims]
    proj = [vecs[k] @ fs[k].cpu().numpy() for k in range(N)]  # a_k^T U_k, length C
    s = torch.cuda.current_stream()
    for mode in range(N):
        w = np.ones(C)
        for k in range(N):
            if k != mode:
                w = w * proj[k]
        want = np.outer(vecs[mode], w)
        out = torch.empty((dims[mode], C), dtype=torch.float64, device="cuda")
        for algo, order in algos_for(mode, N):
            out.fill_(np.nan)
            dg.mttkrp_device(t, [f.data_ptr() for f in fs], C, mode, algo, order, out.data_ptr(), s.cuda_stream)
            got = out.cpu().numpy()
            err = np.linalg.norm(got - want) / np.linalg.norm(want)
            assert err <= 1e-12, (dims, C, mode, algo, order, err)
    del t, x
    torch.cuda.empty_cache()


@pytest.mark.parametrize("dims,C", [((1000, 1000, 1000), 25), ((64, 64, 64, 64, 64), 32)], ids=["1000c25", "64c32"])
def test_linearity_in_a_factor(dims, C):
    N = len(dims)
    g = torch.Generator(device="cuda").manual_seed(5)
    x = torch.rand(int(np.prod(dims)), dtype=torch.float64, device="cuda", generator=g)
    t = dg.DenseTensor.from_device(dims, x.data_ptr(), owner=x)
    fs = [torch.rand((d, C), dtype=torch.float64, device="cuda", generator=g) for d in dims]
    wv = torch.rand(C, dtype=torch.float64, device="cuda", generator=g) + 0.5
    s = torch.cuda.current_stream()
    for mode in range(N):
        k = (mode + 1) % N
        scaled = [f if j != k else f * wv[None, :] for j, f in enumerate(fs)]
        o1 = torch.empty((dims[mode], C), dtype=torch.float64, device="cuda")
        o2 = torch.empty_like(o1)
        dg.mttkrp_device(t, [f.data_ptr() for f in fs], C, mode, A.automatic, O.automatic, o1.data_ptr(),
                         s.cuda_stream)
        dg.mttkrp_device(t, [f.data_ptr() for f in scaled], C, mode, A.automatic, O.automatic, o2.data_ptr(),
                         s.cuda_stream)
        want = (o1 * wv[None, :]).cpu().numpy()
        got = o2.cpu().numpy()
        assert np.linalg.norm(got - want) <= 1e-12 * np.linalg.norm(want), (dims, mode)
    del t, x
    torch.cuda.empty_cache()


def fmri_tensor(dims, seed=1):
    n0, n1 = dims[0], dims[1]
    rest = tuple(dims[2:])[::-1]
    g = torch.Generator(device="cuda").manual_seed(seed)
    # in place (two 7.7 GB buffers at the peak, not five)
    torch.cuda.empty_cache()
    z = torch.randn(rest + (n1, n0), dtype=torch.float64, device="cuda", generator=g)
    z.mul_(0.3).tanh_().triu_(diagonal=1)
    z.add_(z.transpose(-1, -2).contiguous())
    z.diagonal(dim1=-2, dim2=-1).fill_(1.0)
    torch.cuda.empty_cache()
    return z.reshape(-1)


def test_cp_als_fmri_full_size_sweeps_agree():
    dims = (100, 100, 1200, 80)
    x = fmri_tensor(dims)
    # (wrap waits for the generator kernels: cp_als reads x on the library's stream)
    t = dg.DenseTensor.from_device(dims, x.data_ptr(), owner=x)
    fits = {}
    for name, tree, sym in (("per_mode", False, False), ("tree", True, False), ("sym", True, True)):
        tt = t.pack_symmetric01() if sym else t
        r = dg.cp_als(tt, dg.AlsConfig(rank=20, max_iters=4, tol=0.0, seed=1, dimension_tree=tree))
        fits[name] = [it.fit.fit for it in r.trace.iters]
        assert len(fits[name]) == 4
        assert all(b >= a - 1e-10 for a, b in zip(fits[name], fits[name][1:])), fits[name]
    for name in ("tree", "sym"):
        assert max(abs(a - b) for a, b in zip(fits[name], fits["per_mode"])) <= 1e-9, (name, fits)
