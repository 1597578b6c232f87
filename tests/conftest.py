import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden", "golden.json")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def golden():
    with open(GOLDEN) as f:
        return json.load(f)


def _has_gpu():
    import ctypes
    try:
        cu = ctypes.CDLL("libcuda.so.1")
        if cu.cuInit(0) != 0:
            return False
        n = ctypes.c_int(0)
        return cu.cuDeviceGetCount(ctypes.byref(n)) == 0 and n.value > 0
    except OSError:
        return False


HAS_GPU = _has_gpu()


@pytest.fixture(params=["small", "grid"])
def both_kernels(request, monkeypatch):
    """Run the test through the single-cluster kernel (graphs with n <= 2^17,
    gk_bfs_small.cu) and again through the grid kernel (GK_NO_SMALL=1)."""
    if request.param == "grid":
        monkeypatch.setenv("GK_NO_SMALL", "1")
    else:
        monkeypatch.delenv("GK_NO_SMALL", raising=False)
    return request.param


@pytest.fixture
def grid_kernel(monkeypatch):
    """Tests of the grid kernel's own phases on small graphs."""
    monkeypatch.setenv("GK_NO_SMALL", "1")


def pytest_collection_modifyitems(config, items):
    if HAS_GPU:
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)
