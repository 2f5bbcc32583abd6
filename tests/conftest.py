import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def _ensure_library():
    """Build libasaga.so in-tree if this checkout has none yet (tests import the package,
    which refuses to load without it: there is no CPU fallback)."""
    lib = os.path.join(ROOT, "paper_1606_04809_b200", "libasaga.so")
    if os.path.exists(lib):
        return
    import importlib.util

    spec = importlib.util.spec_from_file_location(
        "_asaga_build", os.path.join(ROOT, "paper_1606_04809_b200", "_build.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    mod.build()


def pytest_configure(config):
    _ensure_library()
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through the C-ABI on cuda:0)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def _has_gpu() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _has_gpu():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture(scope="session")
def curand_ref():
    """cuRAND's host-side Philox4x32-10 (pin P1), compiled from tests/pins."""
    import ctypes

    src = os.path.join(ROOT, "tests", "pins", "curand_philox_ref.cu")
    out = os.path.join(ROOT, "tests", "pins", "libcurand_ref.so")
    if not os.path.exists(out) or os.path.getmtime(out) < os.path.getmtime(src):
        tmp = out + f".tmp{os.getpid()}"
        subprocess.check_call(["nvcc", "-O2", "-shared", "-Xcompiler", "-fPIC", "-gencode",
                               "arch=compute_100a,code=sm_100a", "-o", tmp, src])
        os.replace(tmp, out)
    lib = ctypes.CDLL(out)
    lib.curand_ref_philox_stream.restype = None
    lib.curand_ref_philox_stream.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64,
                                             ctypes.POINTER(ctypes.c_uint32)]
    return lib
