import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "oracle")):
    if p not in sys.path:
        sys.path.insert(0, p)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a); run with -m gpu")


@pytest.fixture(scope="session")
def ff():
    from paper_1802_03433_b200 import femforge
    femforge.lib()  # fail loudly when the engine is not built
    return femforge


@pytest.fixture(scope="session")
def ctx(ff):
    return ff.Context(0)


def normwise(got, want):
    """acceptance.cpp:58-67: max |got-want| / max |want|."""
    import numpy as np
    scale = float(np.max(np.abs(want))) if want.size else 0.0
    scale = scale if scale > 0 else 1.0
    return float(np.max(np.abs(got - want))) / scale if want.size else 0.0
