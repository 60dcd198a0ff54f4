"""The read-only tensor contract on the device (run by
tests/test_gpu_readonly.py in its own process).

The reference maps X with mprotect(PROT_READ) so that any write by any
algorithm faults (acceptance check 4, proj/tests/acceptance.cpp:304-369;
DenseTensor is immutable, tensor.hpp:11-18). Here the tensor lives in physical
device memory created with the CUDA virtual-memory API and mapped twice: once
read-write (to fill it), once with CU_MEM_ACCESS_FLAGS_PROT_READ. The library
borrows the READ-ONLY mapping (dmtk_gpu_tensor_wrap) and runs every flavor --
MTTKRP in every mode with every algorithm and order, the tensor norm, CP-ALS
(per-mode sweep and dimension tree), fit, and the symmetric packing; a single
store through the read-only mapping raises an illegal-address fault, which
poisons the context and fails this script. Prints "readonly ok" on success.
"""
import os
import sys

import numpy as np
import torch
from cuda.bindings import driver as cu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_1708_08976_b200 as dg  # noqa: E402
from paper_1708_08976_b200 import MttkrpAlgo as A, TwoStepOrder as O  # noqa: E402
from oracle_bindings import Oracle  # noqa: E402


def ck(res):
    err = res[0] if isinstance(res, tuple) else res
    if err != cu.CUresult.CUDA_SUCCESS:
        raise RuntimeError(f"CUDA driver error {err}")
    return res[1] if isinstance(res, tuple) and len(res) == 2 else res


class ReadOnlyBuffer:
    """Physical device memory with a read-write and a read-only mapping."""

    def __init__(self, nbytes, device=0):
        prop = cu.CUmemAllocationProp()
        prop.type = cu.CUmemAllocationType.CU_MEM_ALLOCATION_TYPE_PINNED
        prop.location.type = cu.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
        prop.location.id = device
        gran = ck(cu.cuMemGetAllocationGranularity(
            prop, cu.CUmemAllocationGranularity_flags.CU_MEM_ALLOC_GRANULARITY_MINIMUM))
        self.size = (nbytes + gran - 1) // gran * gran
        self.handle = ck(cu.cuMemCreate(self.size, prop, 0))
        self.rw = ck(cu.cuMemAddressReserve(self.size, 0, 0, 0))
        self.ro = ck(cu.cuMemAddressReserve(self.size, 0, 0, 0))
        ck(cu.cuMemMap(self.rw, self.size, 0, self.handle, 0))
        ck(cu.cuMemMap(self.ro, self.size, 0, self.handle, 0))
        for va, flags in ((self.rw, cu.CUmemAccess_flags.CU_MEM_ACCESS_FLAGS_PROT_READWRITE),
                          (self.ro, cu.CUmemAccess_flags.CU_MEM_ACCESS_FLAGS_PROT_READ)):
            desc = cu.CUmemAccessDesc()
            desc.location.type = cu.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
            desc.location.id = device
            desc.flags = flags
            ck(cu.cuMemSetAccess(va, self.size, [desc], 1))

    def fill(self, values: np.ndarray):
        v = np.ascontiguousarray(values, dtype=np.float64)
        ck(cu.cuMemcpyHtoD(self.rw, v, v.nbytes))

    @property
    def ro_ptr(self):
        return int(self.ro)


def check(name, got, want, tol=1e-12):
    err = np.linalg.norm(got - want) / max(np.linalg.norm(want), 1e-300)
    assert err <= tol, (name, err)


def main():
    torch.zeros(1, device="cuda")  # the primary context the library uses
    orc = Oracle()
    cases = [((24, 20, 18, 6), 20), ((64, 30, 40), 25), ((33, 17, 12), 9)]  # the last: odd first extent (repacked)
    for dims, C in cases:
        x = orc.gen_tensor(dims, 3)
        f = orc.gen_factors(dims, C, 4)
        buf = ReadOnlyBuffer(x.nbytes)
        buf.fill(x)
        t = dg.DenseTensor.from_device(dims, buf.ro_ptr)
        N = len(dims)
        for mode in range(N):
            want = orc.mttkrp(x, dims, f, mode)
            variants = [(A.automatic, O.automatic), (A.one_step, O.automatic), (A.baseline, O.automatic)]
            if 0 < mode < N - 1:
                variants += [(A.two_step, O.left), (A.two_step, O.right)]
            for algo, order in variants:
                check((dims, mode, algo, order), dg.mttkrp(dg.MttkrpRequest(t, f, mode, algo, order)).m, want)
            fd = [torch.from_numpy(u).cuda() for u in f]
            out = torch.empty((dims[mode], C), dtype=torch.float64, device="cuda")
            dg.mttkrp_device(t, [u.data_ptr() for u in fd], C, mode, A.automatic, O.automatic, out.data_ptr(),
                             torch.cuda.current_stream().cuda_stream)
            torch.cuda.synchronize()
            check((dims, mode, "device"), out.cpu().numpy(), want)
        assert abs(dg.tensor_norm(t) - orc.tensor_norm(x)) <= 1e-12 * orc.tensor_norm(x)
        for tree in (False, True):
            r = dg.cp_als(t, dg.AlsConfig(rank=4, max_iters=3, tol=0.0, seed=1, dimension_tree=tree))
            _, _, fits, _ = orc.cp_als(x, dims, 4, 3, 0.0, 1)
            assert np.max(np.abs(np.array([i.fit.fit for i in r.trace.iters]) - fits)) <= 1e-9
        dg.fit(t, r.model)
        torch.cuda.synchronize()
        t.release()
    # the symmetric packing reads the tensor once more
    dims = (12, 12, 5, 3)
    y = orc.gen_tensor(dims, 8).reshape(dims[::-1])
    y = np.ascontiguousarray(y + np.swapaxes(y, -1, -2)).reshape(-1)
    buf = ReadOnlyBuffer(y.nbytes)
    buf.fill(y)
    t = dg.DenseTensor.from_device(dims, buf.ro_ptr)
    tp = t.pack_symmetric01()
    dg.cp_als(tp, dg.AlsConfig(rank=3, max_iters=2, tol=0.0, seed=1))
    torch.cuda.synchronize()
    assert np.array_equal(np.frombuffer(y.tobytes()), t.download())  # unchanged
    print("readonly ok")


if __name__ == "__main__":
    main()
