"""Tensor ingest: DNT1 files (reference tensor_io.cpp:79-130)
read straight into HBM by dmtk_gpu_tensor_load, against files written and
read by the unmodified reference library (oracle/_ref): identical values,
identical validation messages, and MTTKRP on the loaded tensor at <= 1e-12.
"""
import os
import struct

import numpy as np
import pytest

import paper_1708_08976_b200 as dg
from oracle_bindings import RefError

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dims", [(7,), (6, 5), (9, 11, 13), (4, 3, 5, 2), (3, 2, 2, 3, 4), (100, 100, 1000),
                                  (101, 100, 901)])
def test_load_reference_written_file(tmp_path, ref, oracle, dims):
    x = oracle.gen_tensor(dims, 23)
    path = str(tmp_path / "t.dnt")
    ref.write_tensor(path, x, dims)
    t = dg.DenseTensor.load(path)
    assert t.dims == tuple(dims)
    assert np.array_equal(t.download(), x)  # bitwise, padded layouts included (odd first extent)
    if len(dims) >= 3 and np.prod(dims) <= 4096:
        f = oracle.gen_factors(dims, 5, 3)
        for mode in range(len(dims)):
            got = dg.mttkrp(dg.MttkrpRequest(t, f, mode)).m
            want = oracle.mttkrp(x, dims, f, mode)
            assert np.linalg.norm(got - want) <= 1e-12 * np.linalg.norm(want)


def _dnt(dims, payload_doubles=None, magic=b"DNT1", version=1, n=None, extra=b""):
    n = len(dims) if n is None else n
    head = magic + struct.pack("<II", version, n) + b"".join(struct.pack("<Q", d) for d in dims)
    count = int(np.prod(dims)) if payload_doubles is None else payload_doubles
    return head + np.arange(count, dtype="<f8").tobytes() + extra


@pytest.mark.parametrize("name,blob", [
    ("magic", _dnt((2, 3), magic=b"DNT2")),
    ("version", _dnt((2, 3), version=2)),
    ("zero_modes", _dnt((), n=0)),
    ("zero_extent", _dnt((2, 0, 3))),
    ("truncated_header", b"DNT1" + struct.pack("<I", 1)),
    ("truncated_payload", _dnt((4, 5), payload_doubles=7)),
    ("trailing", _dnt((4, 5), extra=b"x")),
])
def test_malformed_files_match_reference_messages(tmp_path, ref, name, blob):
    path = str(tmp_path / (name + ".dnt"))
    with open(path, "wb") as f:
        f.write(blob)
    with pytest.raises(RefError) as want:
        ref.read_tensor(path)
    with pytest.raises(dg.TensorFileError) as got:
        dg.DenseTensor.load(path)
    assert want.value.code == 5
    assert str(got.value) == str(want.value)


def test_missing_file(ref, tmp_path):
    path = str(tmp_path / "absent.dnt")
    with pytest.raises(RefError) as want:
        ref.read_tensor(path)
    with pytest.raises(dg.TensorFileError) as got:
        dg.DenseTensor.load(path)
    assert str(got.value) == str(want.value)
