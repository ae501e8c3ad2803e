import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")


def has_gpu() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if has_gpu():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


@pytest.fixture(scope="session")
def port():
    from oracle.ffi import Oracle
    return Oracle("port")


@pytest.fixture(scope="session")
def ref():
    from oracle.ffi import Oracle, available, REF_SRC
    if not available("ref") and not os.path.isdir(REF_SRC):
        pytest.skip("oracle/_ref not built and /root/reference absent")
    return Oracle("ref")


def load_golden(name):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)


@pytest.fixture(scope="session")
def small_workload(port):
    """Reference generator at test scale (test_engine.cpp:17-29 shape)."""
    return port.generate_workload(2048, 64, 32, 4, 2, seed=7, n_decode=16)
