import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


@pytest.fixture(scope="session")
def oracle():
    from oracle.oracle import oracle as _o
    return _o()


@pytest.fixture(scope="session")
def ref():
    from oracle.oracle import ref as _r, ref_available
    if not ref_available():
        pytest.skip("oracle/_ref/libsuco_ref.so not built (needs /root/reference at build time)")
    return _r()


@pytest.fixture(scope="session")
def suco():
    import paper_2411_14754_b200 as s
    return s


@pytest.fixture(scope="session")
def gpu(suco):
    if suco.device_count() < 1:
        pytest.fail("no CUDA device visible: -m gpu tests must run on the B200 box")
    return suco


def golden(name):
    import numpy as np
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)
