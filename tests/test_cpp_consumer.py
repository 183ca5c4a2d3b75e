"""The C++ mirror (include/suco_b200.hpp) as a reference user would consume it:
examples/gpu_batch.cpp does build -> serialize -> load -> batched query through
the header, the way suco_cli.cpp's build/query commands drive the reference."""
import os
import subprocess

import numpy as np
import pytest
import torch

from conftest import ROOT

EXE = os.path.join(ROOT, "examples", "_build", "gpu_batch")


def _build():
    r = subprocess.run(["make", "-C", os.path.join(ROOT, "examples")], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    return EXE


def _files(tmp_path, base, qs):
    b, q = tmp_path / "base.f32", tmp_path / "q.f32"
    base.astype(np.float32).tofile(b)
    qs.astype(np.float32).tofile(q)
    return str(b), str(q)


def test_example_compiles_against_header_and_library():
    exe = _build()
    r = subprocess.run([exe], capture_output=True, text=True)
    assert r.returncode == 2 and "usage" in r.stderr


@pytest.mark.skipif(torch.cuda.is_available(), reason="CPU-host behaviour")
def test_example_fails_loudly_without_gpu(tmp_path, oracle):
    exe = _build()
    base = oracle.clustered(600, 8, 4, 1, 0.0, 10.0, 1.0, False)
    b, q = _files(tmp_path, base, base[:3])
    r = subprocess.run([exe, "600", "8", b, "3", q, "0.1", "0.05", "5", str(tmp_path / "o.bin")],
                       capture_output=True, text=True)
    assert r.returncode == 1 and "error" in r.stderr.lower(), (r.returncode, r.stderr)


@pytest.mark.gpu
def test_example_matches_oracle(tmp_path, oracle):
    exe = _build()
    full = oracle.clustered(8000 + 40, 24, 20, 3, 0.0, 100.0, 9.0, True)
    base, qs = oracle.hold_out(full, 40, 4)
    b, q = _files(tmp_path, base, qs)
    out = tmp_path / "o.bin"
    k = 10
    r = subprocess.run([exe, str(len(base)), "24", b, str(len(qs)), q, "0.05", "0.01", str(k), str(out)],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    raw = out.read_bytes()
    ids = np.frombuffer(raw[: len(qs) * k * 4], np.uint32).reshape(len(qs), k)
    dd = np.frombuffer(raw[len(qs) * k * 4:], np.float64).reshape(len(qs), k)
    oidx = oracle.build_index(base, 4, 16, 3, 42, 0)
    wi, wd, _ = oidx.knn_query_batch(base, qs, 0.05, 0.01, k)
    assert np.array_equal(ids, wi)
    assert np.array_equal(dd, wd)
    assert (tmp_path / "o.bin.suco").read_bytes() == bytes(oidx.serialize())
