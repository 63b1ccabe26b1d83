import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libfetigpu.so")
    config.addinivalue_line("markers", "slow: full-size oracle comparisons of several minutes of CPU "
                                       "oracle time; run with FETIGPU_SLOW_TESTS=1")


def pytest_collection_modifyitems(config, items):
    if os.environ.get("FETIGPU_SLOW_TESTS") == "1":
        return
    skip = pytest.mark.skip(reason="slow oracle comparison (FETIGPU_SLOW_TESTS=1 runs it)")
    for it in items:
        if "slow" in it.keywords:
            it.add_marker(skip)


@pytest.fixture(scope="session", autouse=True)
def _oracle_threads():
    """The CPU oracle uses every host core (the GPU box has 16)."""
    try:
        from oracle import pyoracle
        pyoracle.build()
        pyoracle.lib().fo_set_threads(os.cpu_count() or 1)
    except Exception:
        pass


def has_gpu() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def oracle_mod():
    from oracle import pyoracle
    pyoracle.build()
    return pyoracle


def rel(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)
