"""CPU-side checks of the drop-in boundary: the C-ABI library loads, exports
every entry point include/suco_b200.h declares, its host arithmetic matches
the reference KATs, and compute calls fail loudly without a GPU."""
import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT
from test_oracle import CANDIDATE_KATS, COLLISION_KATS


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "suco_b200.h")).read()
    return sorted(set(re.findall(r"\b(suco_\w+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_2411_14754_b200 import _capi
    lib = ctypes.CDLL(_capi.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 20
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    assert sorted(_capi.EXPORTED) == syms


def test_cpp_header_mirrors_every_c_entry_point():
    hpp = open(os.path.join(ROOT, "include", "suco_b200.hpp")).read()
    for s in declared_symbols():
        assert s in hpp, s


@pytest.mark.parametrize("alpha,n,want", COLLISION_KATS)
def test_collision_count(suco, alpha, n, want):
    assert suco.collision_count(alpha, n) == want


@pytest.mark.parametrize("beta,n,k,want", CANDIDATE_KATS)
def test_candidate_count(suco, beta, n, k, want):
    assert suco.candidate_count(beta, n, k) == want


def test_params_validation(suco):
    suco.CollisionParams().validate(1000)
    for bad in (0.0, -0.5, 1.5):
        with pytest.raises(suco.ConfigError):
            suco.CollisionParams(alpha=bad).validate(1000)
        with pytest.raises(suco.ConfigError):
            suco.CollisionParams(beta=bad).validate(1000)
    with pytest.raises(suco.ConfigError):
        suco.CollisionParams(k=0).validate(1000)
    with pytest.raises(suco.ConfigError):
        suco.CollisionParams(k=1001).validate(1000)
    suco.CollisionParams(k=1000).validate(1000)


def test_defaults_match_reference(suco):  # index.hpp:53-61, sc_linear.hpp:22-31
    p = suco.IndexParams()
    assert (p.num_subspaces, p.k_half, p.iterations, p.seed, int(p.mode)) == (8, 50, 10, 42, 0)
    c = suco.CollisionParams()
    assert (c.alpha, c.beta, c.k) == (0.05, 0.005, 50)


def test_compute_fails_loudly_without_gpu(suco):
    if suco.device_count() > 0:
        pytest.skip("a GPU is visible")
    with pytest.raises(suco.Error, match="no CUDA device"):
        suco.rerank(np.zeros((4, 4), np.float32), np.zeros(4, np.float32), [0, 1], 1)
    with pytest.raises(suco.Error, match="no CUDA device"):
        suco.build_index(np.zeros((100, 8), np.float32), suco.IndexParams(num_subspaces=2, k_half=4))


def test_contract_checks_precede_device_use(suco):
    """Argument validation happens on the host in the reference's order, GPU or not."""
    with pytest.raises(suco.ContractError):
        suco.rerank(np.zeros((4, 4), np.float32), np.zeros(3, np.float32), [0, 1], 1)
    with pytest.raises(suco.ContractError):
        suco.centroid_distances([1.0], [0.0, 1.0], 0)
    with pytest.raises(suco.ConfigError):
        suco.kmeans(np.zeros((10, 2), np.float32), 11, 5, 1)
    with pytest.raises(suco.ContractError):
        suco.build_imi([0, 1], [0, 2], 2)


def test_format_and_corrupt_index_are_distinct_codes(suco, tmp_path):
    """Vecs files raise FormatError (io.cpp:20-84, status 3); index bytes raise CorruptIndexError
    (index.cpp:191-293, status 6), which is-a FormatError like the reference's. Both checks run on
    the host, before any device use."""
    from paper_2411_14754_b200 import _capi
    data = np.zeros((10, 4), np.float32)
    with pytest.raises(suco.CorruptIndexError, match="magic"):
        suco.load_index(b"SUCX" + bytes(60), data)
    assert issubclass(suco.CorruptIndexError, suco.FormatError)
    blob = np.frombuffer(b"junk", np.uint8).copy()
    rc = _capi.load_index(blob.ctypes.data_as(_capi.u8p), 4, data.ctypes.data_as(_capi.f32p), 10, 4, 0,
                          ctypes.byref(ctypes.c_void_p()))
    assert rc == 6
    bad = tmp_path / "bad.fvecs"
    bad.write_bytes(b"\x03\x00\x00")
    with pytest.raises(suco.FormatError) as e:
        suco.read_vecs(str(bad), "fvecs")
    assert not isinstance(e.value, suco.CorruptIndexError)


def test_header_declares_status_codes_and_contexts():
    src = open(os.path.join(ROOT, "include", "suco_b200.h")).read()
    assert "#define SUCO_ERR_CORRUPT_INDEX 6" in src and "#define SUCO_ERR_FORMAT 3" in src
    # the handle is immutable: no entry point mutates it (the old set_stream is gone)
    assert "suco_gpu_set_stream" not in src
    for fn in ("suco_gpu_knn_query_batch(", "suco_gpu_knn_query_batch_device("):
        decl = src[src.index("int " + fn):].split(";")[0]
        assert "const suco_gpu_index*" in decl and "suco_gpu_query_ctx*" in decl, decl


def test_library_then_torch_import_order():
    """libsuco_b200.so links the NCCL copy torch bundles (one libnccl.so.2 per process): importing
    the library BEFORE torch must not shadow torch's NCCL with an older one."""
    import subprocess
    import sys
    r = subprocess.run([sys.executable, "-c", "import paper_2411_14754_b200, torch; print(torch.__version__)"],
                       cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
