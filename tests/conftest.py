"""Test configuration: the `gpu` marker, repo path, and shared builders.

CPU tests (-m "not gpu") check the oracle against the reference's golden
vectors, the host connectivity builder, the metric operation order and the
C-ABI symbol table.  GPU tests (-m gpu) are the parity tests proper: they run
the CUDA path through the C-ABI and compare with the oracle and the goldens.
"""

from __future__ import annotations

import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session", autouse=True)
def _built_library():
    """Build libhv_b200.so in-tree if it is missing or stale (nvcc works without a GPU)."""
    from paper_2311_11425_b200 import build

    build.build()
    yield


def golden(name):
    return dict(np.load(GOLDEN / f"{name}.npz"))


def has_cuda():
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False
