"""Shared test configuration.

Markers: `gpu` -- needs a B200 (sm_100a) and the built libmlb.so; everything
else runs on CPU (oracle vs golden vectors, host plan math, C-ABI symbol
table, gloo multi-process logic).
"""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 device and libmlb.so")


def load_golden(name):
    return np.load(os.path.join(GOLDEN, f"golden_{name}.npz"))


def gpu_available():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def golden():
    return load_golden


def pytest_collection_modifyitems(config, items):
    if gpu_available():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture(autouse=True)
def _no_stale_cuda_error(request):
    """GPU tests must not leave an error in the CUDA runtime's last-error slot:
    libmlb shares libcudart with torch, whose next launch check would report
    it inside an unrelated test."""
    yield
    if "gpu" not in request.node.keywords or not gpu_available():
        return
    import ctypes
    import gc

    import torch
    gc.collect()   # finalizers (binding / plan destroy) run inside this test
    torch.cuda.synchronize()
    rt = ctypes.CDLL("libcudart.so.12")   # the loaded runtime (matched by soname)
    code = rt.cudaPeekAtLastError()
    if code != 0:
        rt.cudaGetLastError()
        rt.cudaGetErrorString.restype = ctypes.c_char_p
        pytest.fail(f"test left CUDA error {code} ({rt.cudaGetErrorString(code).decode()}) in the runtime")
