"""fvecs/ivecs I/O (the input format either side of the path), mirroring the
reference's tests/test_data.py:67-145 case for case, plus the device loader."""

from __future__ import annotations

import struct

import numpy as np
import pytest

import paper_2507_17094_b200 as pw
from paper_2507_17094_b200.data import DataFormatError


def _data(n=100, d=7, seed=3):
    return pw.Dataset(np.random.default_rng(seed).standard_normal((n, d)).astype(np.float32))


def test_fvecs_single_record(tmp_path):
    path = tmp_path / "one.fvecs"
    path.write_bytes(struct.pack("<i2f", 2, 1.5, -2.0))
    ds = pw.load_fvecs(path)
    assert (ds.n, ds.d) == (1, 2)
    assert ds.data.tolist() == [[1.5, -2.0]]


def test_fvecs_round_trip_byte_identical(tmp_path):
    ds = _data()
    p1, p2 = tmp_path / "a.fvecs", tmp_path / "b.fvecs"
    pw.save_fvecs(ds, p1)
    pw.save_fvecs(pw.load_fvecs(p1), p2)
    assert p1.read_bytes() == p2.read_bytes()
    assert np.array_equal(pw.load_fvecs(p2).data, ds.data)


def test_fvecs_layout_is_reference_layout(tmp_path):
    ds = _data(5, 3)
    path = tmp_path / "x.fvecs"
    pw.save_fvecs(ds, path)
    want = b"".join(struct.pack("<i", 3) + row.astype("<f4").tobytes() for row in ds.data)
    assert path.read_bytes() == want


def test_fvecs_file_size_arithmetic(tmp_path):
    path = tmp_path / "s.fvecs"
    pw.save_fvecs(np.zeros((3, 4), dtype=np.float32), path)
    assert path.stat().st_size == 60 == pw.file_size_for(3, 4)


def test_fvecs_inconsistent_dimension_names_offset(tmp_path):
    path = tmp_path / "bad.fvecs"
    path.write_bytes(struct.pack("<i2f", 2, 1.0, 2.0) + struct.pack("<i3f", 3, 1.0, 2.0, 3.0))
    with pytest.raises(DataFormatError, match="offset 12"):
        pw.load_fvecs(path)


def test_fvecs_truncated_record(tmp_path):
    path = tmp_path / "trunc.fvecs"
    path.write_bytes(struct.pack("<i2f", 2, 1.0, 2.0) + struct.pack("<if", 2, 1.0))
    with pytest.raises(DataFormatError, match="truncated"):
        pw.load_fvecs(path)


def test_fvecs_nonpositive_dimension(tmp_path):
    path = tmp_path / "zed.fvecs"
    path.write_bytes(struct.pack("<i", 0))
    with pytest.raises(DataFormatError, match="dimension"):
        pw.load_fvecs(path)


def test_fvecs_empty_file(tmp_path):
    path = tmp_path / "empty.fvecs"
    path.write_bytes(b"")
    with pytest.raises(DataFormatError, match="empty file"):
        pw.load_fvecs(path)


def test_save_empty_rejected(tmp_path):
    with pytest.raises(DataFormatError, match="n >= 1"):
        pw.save_fvecs(np.zeros((0, 4), dtype=np.float32), tmp_path / "e.fvecs")


def test_ivecs_single_record(tmp_path):
    path = tmp_path / "one.ivecs"
    path.write_bytes(struct.pack("<4i", 3, 0, 5, 9))
    assert pw.load_ivecs(path).tolist() == [[0, 5, 9]]


def test_ivecs_round_trip(tmp_path):
    mat = np.random.default_rng(8).integers(0, 1000, (20, 5)).astype(np.int32)
    p1, p2 = tmp_path / "a.ivecs", tmp_path / "b.ivecs"
    pw.save_ivecs(mat, p1)
    pw.save_ivecs(pw.load_ivecs(p1), p2)
    assert p1.read_bytes() == p2.read_bytes()
    assert np.array_equal(pw.load_ivecs(p2), mat)


def test_ivecs_truncated(tmp_path):
    path = tmp_path / "t.ivecs"
    path.write_bytes(struct.pack("<3i", 3, 1, 2))
    with pytest.raises(DataFormatError, match="truncated"):
        pw.load_ivecs(path)


@pytest.mark.gpu
def test_fvecs_device_loader(tmp_path):
    ds = _data(1000, 96, seed=5)
    path = tmp_path / "x.fvecs"
    pw.save_fvecs(ds, path)
    t = pw.load_fvecs_device(path)
    assert t.is_cuda and t.dtype.is_floating_point and tuple(t.shape) == (1000, 96)
    assert np.array_equal(t.cpu().numpy(), ds.data)
    bad = tmp_path / "bad.fvecs"
    bad.write_bytes(struct.pack("<i2f", 2, 1.0, 2.0) + struct.pack("<i2f", 3, 1.0, 2.0))
    with pytest.raises(DataFormatError, match="offset 12"):
        pw.load_fvecs_device(bad)
    with pytest.raises(DataFormatError, match="truncated"):
        trunc = tmp_path / "trunc.fvecs"
        trunc.write_bytes(struct.pack("<i2f", 2, 1.0, 2.0) + struct.pack("<if", 2, 1.0))
        pw.load_fvecs_device(trunc)
