import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running (full-size configs)")


@pytest.fixture(scope="session")
def pw():
    import paper_2111_01083_b200 as m

    m.lib()
    return m


@pytest.fixture(scope="session")
def ref():
    from oracle import pyoracle

    if not pyoracle.ref_available():
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    return pyoracle.Ref()


@pytest.fixture(scope="session")
def port():
    from oracle import pyoracle

    return pyoracle.Port()


@pytest.fixture(scope="session")
def gpu(pw):
    if pw.device_count() < 1:
        pytest.fail("GPU test selected but no CUDA device is visible")
    return True


def rel_l2(got, want, gauge=False):
    """Relative l2 error per SURVEY.md §8(d); gauge=True removes the per-channel mean."""
    g = np.asarray(got, dtype=np.float64).reshape(len(got), -1)
    w = np.asarray(want, dtype=np.float64).reshape(len(want), -1)
    if gauge:
        g = g - g.mean(axis=0)
        w = w - w.mean(axis=0)
    num = np.linalg.norm(g - w, axis=0)
    den = np.linalg.norm(w, axis=0)
    return float(np.max(num / np.maximum(den, 1e-300)))
