import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200) and the built extension")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def golden(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def cuda_available():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def ensure_built():
    """Build lib/libacp.so with nvcc if it is missing (no GPU needed)."""
    lib = os.path.join(ROOT, "paper_2306_08881_b200", "lib", "libacp.so")
    if not os.path.exists(lib):
        _load_build_module().build()
    return lib


def _load_build_module():
    # loaded by path: importing the package itself requires the built library
    import importlib.util
    spec = importlib.util.spec_from_file_location(
        "acp_build", os.path.join(ROOT, "paper_2306_08881_b200", "build.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod
