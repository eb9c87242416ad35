"""Shared pytest configuration.

`-m gpu` tests need a B200 (run them through gpurun); everything else runs on
the CPU build container. Golden fixtures in tests/golden/ come from the
reference itself (tools/make_golden.py).
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
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


def load_golden(name):
    return np.load(os.path.join(GOLDEN, name + ".npz"))


def golden_cases(g):
    return sorted({k.split("/")[0] for k in g.files if "/" in k})


def cuda_available():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def golden_spmm():
    return load_golden("spmm")


@pytest.fixture(scope="session")
def golden_sddmm():
    return load_golden("sddmm")


@pytest.fixture(scope="session")
def golden_attention():
    return load_golden("attention")


@pytest.fixture(scope="session")
def golden_formats():
    return load_golden("formats")
