import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built liblsg_b200.so")
    config.addinivalue_line("markers", "slow: longer oracle runs")


def _ensure_oracle():
    from oracle import oracle as O

    if not os.path.exists(O.PORT_SO) or (os.path.isdir("/root/reference/proj") and not os.path.exists(O.REF_SO)):
        O.build()


@pytest.fixture(scope="session")
def port():
    from oracle import oracle as O

    _ensure_oracle()
    return O.port()


@pytest.fixture(scope="session")
def ref():
    from oracle import oracle as O

    _ensure_oracle()
    if not O.have_reference():
        pytest.skip("oracle/_ref not built (reference sources absent and no prebuilt library)")
    return O.reference()


@pytest.fixture(scope="session")
def ctx():
    from paper_2507_11542_b200 import _lib

    if _lib.device_count() == 0:
        pytest.fail("no CUDA device: the gpu tests need a B200 (no CPU fallback exists)")
    c = _lib.Context(0)
    yield c
    c.close()


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.int64)


def assert_bitwise(a, b, what=""):
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    assert a.shape == b.shape, (what, a.shape, b.shape)
    diff = bits(a) != bits(b)
    if diff.any():
        i = int(np.flatnonzero(diff)[0])
        raise AssertionError(f"{what}: {int(diff.sum())} of {a.size} differ; first at {i}: {a[i]!r} vs {b[i]!r}")


def rel_inf(a, b):
    """max|a-b| / max|b| (the north_star fp64 tolerance metric)."""
    den = float(np.max(np.abs(b))) if b.size else 0.0
    return float(np.max(np.abs(np.asarray(a) - np.asarray(b)))) / (den if den > 0 else 1.0)
