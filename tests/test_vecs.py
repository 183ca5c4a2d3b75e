"""vecs I/O: read_vecs / write_vecs with the reference's framing checks and error
contract (io.cpp:46-160; cases restated from test_io.cpp:52-207), and the device upload straight
from a vecs file (build / load), identical to the host-array path."""
import struct

import numpy as np
import pytest


def _raw(path, chunks):
    with open(path, "wb") as f:
        for c in chunks:
            f.write(c)


def test_fvecs_round_trip_bit_exact(suco, tmp_path):
    rng = np.random.default_rng(1)
    v = rng.standard_normal((37, 11)).astype(np.float32)
    p = str(tmp_path / "a.fvecs")
    suco.write_vecs(p, "fvecs", v)
    got = suco.read_vecs(p, "fvecs")
    assert got.tobytes() == v.tobytes()
    raw = open(p, "rb").read()
    assert len(raw) == 37 * (4 + 44) and struct.unpack("<i", raw[:4])[0] == 11


def test_bvecs_and_ivecs_widen_exactly(suco, tmp_path):
    b = np.arange(0, 256, dtype=np.float32).reshape(16, 16)
    p = str(tmp_path / "b.bvecs")
    suco.write_vecs(p, "bvecs", b)
    assert np.array_equal(suco.read_vecs(p, "bvecs"), b)
    for bad in (256.0, -1.0, 0.5):  # test_io.cpp:78-83
        with pytest.raises(suco.ContractError):
            suco.write_vecs(str(tmp_path / "x.bvecs"), "bvecs", np.array([[bad]], np.float32))
    iv = np.array([[-(2 ** 24), 0, 2 ** 24, 12345]], np.float32)
    p = str(tmp_path / "c.ivecs")
    suco.write_vecs(p, "ivecs", iv)
    assert np.array_equal(suco.read_vecs(p, "ivecs"), iv)
    _raw(p, [struct.pack("<ii", 1, 2 ** 24 + 1)])
    with pytest.raises(suco.FormatError, match="too large"):
        suco.read_vecs(p, "ivecs")


def test_limit(suco, tmp_path):  # test_io.cpp:116-132
    v = np.random.default_rng(7).random((10, 4), dtype=np.float32)
    p = str(tmp_path / "l.fvecs")
    suco.write_vecs(p, "fvecs", v)
    assert np.array_equal(suco.read_vecs(p, "fvecs", 3), v[:3])
    assert suco.read_vecs(p, "fvecs", 99).shape == (10, 4)
    with pytest.raises(suco.FormatError):
        suco.read_vecs(p, "fvecs", 0)


def test_format_errors_name_the_record_or_offset(suco, tmp_path):  # test_io.cpp:134-198
    with pytest.raises(suco.FormatError):
        suco.read_vecs("/nonexistent/nowhere.fvecs")
    p = str(tmp_path / "e.fvecs")
    _raw(p, [])
    with pytest.raises(suco.FormatError, match="empty"):
        suco.read_vecs(p)
    _raw(p, [struct.pack("<i", -3)])
    with pytest.raises(suco.FormatError, match="record 0"):
        suco.read_vecs(p)
    _raw(p, [struct.pack("<i", 1 << 21)])
    with pytest.raises(suco.FormatError):
        suco.read_vecs(p)
    _raw(p, [struct.pack("<iff", 2, 1.0, 2.0), struct.pack("<ifff", 3, 1.0, 2.0, 3.0)])
    with pytest.raises(suco.FormatError, match="record 1"):
        suco.read_vecs(p)
    _raw(p, [struct.pack("<if", 1, float("nan"))])
    with pytest.raises(suco.FormatError, match="non-finite"):
        suco.read_vecs(p)
    v = np.random.default_rng(17).random((4, 3), dtype=np.float32)
    good = str(tmp_path / "g.fvecs")
    suco.write_vecs(good, "fvecs", v)
    raw = open(good, "rb").read()
    for ln in range(len(raw)):  # every truncation that is not a whole number of records
        if ln > 0 and ln % 16 == 0:
            continue
        _raw(p, [raw[:ln]])
        with pytest.raises(suco.FormatError):
            suco.read_vecs(p)
    _raw(p, [raw[:20]])
    with pytest.raises(suco.FormatError, match="byte offset"):
        suco.read_vecs(p)


def test_write_vecs_validates_shapes(suco, tmp_path):  # test_io.cpp:200-208
    with pytest.raises(suco.ContractError):
        suco.write_vecs(str(tmp_path / "z.fvecs"), "fvecs", np.zeros((0, 3), np.float32))
    with pytest.raises(suco.Error):
        suco.write_vecs("/nonexistent/dir/x.fvecs", "fvecs", np.ones((2, 3), np.float32))


@pytest.mark.gpu
@pytest.mark.parametrize("kind", ["fvecs", "bvecs"])
def test_device_upload_from_vecs_matches_host_path(gpu, oracle, tmp_path, kind):
    full = oracle.clustered(6000 + 20, 32, 20, 9, 0, 200, 10, True)
    base, qs = oracle.hold_out(full, 20, 10)
    p = str(tmp_path / ("d." + kind))
    gpu.write_vecs(p, kind, base)
    params = gpu.IndexParams(4, 12, 3, 42)
    a = gpu.build_index(base, params)
    b = gpu.build_index_from_vecs(p, kind, params)
    assert a.serialize() == b.serialize()
    c = gpu.load_index_from_vecs(a.serialize(), p, kind)
    cp = gpu.CollisionParams(0.05, 0.02, 10)
    wi, wd = a.knn_query_batch(qs, cp)
    for idx in (b, c):
        ids, dd = idx.knn_query_batch(qs, cp)
        assert np.array_equal(ids, wi) and np.array_equal(dd, wd)
    with pytest.raises(gpu.IncompatibilityError):
        gpu.load_index_from_vecs(a.serialize(), p, kind, limit=100)
    with pytest.raises(gpu.FormatError):
        gpu.build_index_from_vecs(str(tmp_path / "missing.fvecs"), "fvecs", params)
