import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden", "ref_golden.npz")
REF_SRC = os.environ.get("OUUKIT_REF", "/root/reference/pkg/src")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); runs the libsaadino kernels")


@pytest.fixture(scope="session")
def golden():
    return dict(np.load(GOLDEN))


@pytest.fixture(scope="session")
def ouukit():
    """The reference package itself, when importable (build container only)."""
    if not os.path.isdir(REF_SRC):
        pytest.skip("reference package not present (GPU box); golden vectors cover the pin")
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    import ouukit as m
    return m


@pytest.fixture()
def rng():
    return np.random.default_rng(1234)
