"""On-device gen_tensor (reference bench.cpp:88-97): the
mt19937_64(seed) uniform(0,1) stream generated in HBM by jump-ahead chunks must
equal, bitwise, the tensor the unmodified reference library (oracle/_ref)
generates, padded layouts (odd first extent) and chunk boundaries included.
"""
import numpy as np
import pytest

import paper_1708_08976_b200 as dg

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dims", [(1,), (7,), (6, 5), (9, 11, 13), (3, 2, 2, 3, 4), (200, 200, 200), (101, 100, 901)])
@pytest.mark.parametrize("seed", [0, 23, 2**64 - 1])
def test_generate_matches_reference(ref, dims, seed):
    t = dg.DenseTensor.generate(dims, seed)
    assert t.dims == tuple(dims)
    assert np.array_equal(t.download(), ref.gen_tensor(dims, seed))


def test_generate_many_chunks_bitwise(oracle):
    # 2e8 draws: 148 chunks of 1 351 352 (not a multiple of the 156-word step)
    dims = (1000, 1000, 200)
    t = dg.DenseTensor.generate(dims, 7)
    assert np.array_equal(t.download(), oracle.gen_tensor(dims, 7))


def test_generate_ones_and_mttkrp(oracle):
    for dims in [(4, 6, 5), (5, 6, 4)]:
        t = dg.DenseTensor.generate(dims, 1, dist="ones")
        assert np.array_equal(t.download(), np.ones(int(np.prod(dims))))
    dims = (33, 20, 17)  # odd first extent: padded layout, MTTKRP over the generated tensor
    t = dg.DenseTensor.generate(dims, 5)
    x = oracle.gen_tensor(dims, 5)
    f = oracle.gen_factors(dims, 9, 6)
    for mode in range(3):
        got = dg.mttkrp(dg.MttkrpRequest(t, f, mode)).m
        want = oracle.mttkrp(x, dims, f, mode)
        assert np.linalg.norm(got - want) <= 1e-12 * np.linalg.norm(want)


@pytest.mark.parametrize("dist,dims", [("signed", (9, 11, 13)), ("signed", (101, 100, 90)),
                                       ("normal", (7,)), ("normal", (9, 8, 7)), ("normal", (101, 100, 91)),
                                       ("normal", (180, 180, 60)),
                                       ("symslice", (5, 5, 7)), ("symslice", (6, 6, 4, 3)),
                                       ("symslice", (100, 100, 120, 8)), ("symslice", (33, 33, 5))])
def test_generate_distributions_bitwise(oracle, dist, dims):
    """BASELINE configs 3-5's distributions: the device transform of the
    reference stream equals the host restatement (oracle.c) bit for bit."""
    t = dg.DenseTensor.generate(dims, 21, dist)
    assert np.array_equal(t.download(), oracle.gen_dist(dims, 21, dist))


def test_generate_factors_distributions(oracle):
    dims = (180, 64, 7)
    for dist in ("uniform", "signed", "normal"):
        dev = dg.generate_factors(dims, 25, 5, dist)
        want = oracle.gen_factors_dist(dims, 25, 5, dist)
        for k, t in enumerate(dev):
            assert np.array_equal(t.download().reshape(dims[k], 25), want[k]), (dist, k)


def test_generate_validation():
    with pytest.raises(dg.InvalidArgument):
        dg.DenseTensor.generate((2, 3), 1, dist="gamma")
    with pytest.raises(dg.InvalidArgument):
        dg.DenseTensor.generate((4, 5, 3), 1, dist="symslice")
    with pytest.raises(ValueError):
        dg.DenseTensor.generate((2, 0, 3), 1)
