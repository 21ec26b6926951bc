import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")


@pytest.fixture(scope="session")
def oracle():
    from oracle.pyoracle import Oracle

    return Oracle()


@pytest.fixture(scope="session")
def reference():
    from oracle.pyoracle import Reference, have_reference

    if not have_reference():
        pytest.skip("oracle/_ref/libparo_ref.so not built (reference sources absent)")
    r = Reference()
    r.select_kernels("scalar")  # bit-exact comparisons use the scalar kernel table
    return r


@pytest.fixture(scope="session")
def paro():
    import paro_b200

    return paro_b200


@pytest.fixture(scope="session")
def ctx(paro):
    c = paro.Context(0)
    yield c
    c.close()


def randn(seed, shape):
    return np.random.default_rng(seed).standard_normal(shape).astype(np.float32)


def rel_err(a, b):
    """max|a-b| / max|b| -- the north-star output metric."""
    return float(np.max(np.abs(a.astype(np.float64) - b.astype(np.float64))) / max(np.max(np.abs(b)), 1e-30))


GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="session")
def c1():
    return np.load(os.path.join(GOLD, "golden_c1.npz"))


@pytest.fixture(scope="session")
def rnd():
    return np.load(os.path.join(GOLD, "golden_rand.npz"))


@pytest.fixture(scope="session")
def kat():
    return np.load(os.path.join(GOLD, "golden_kat.npz"))
