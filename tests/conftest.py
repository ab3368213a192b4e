"""Shared fixtures.  GPU tests are marked `gpu`; everything else runs on a CPU-only host.

Golden fixtures under tests/golden/ were produced by the REFERENCE (make_golden.py); the
CPU oracle (oracle/dk_oracle.py) is the checker for cases too large for the reference.
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200) device and libdk.so")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def golden():
    def load(name):
        return np.load(GOLDEN / f"{name}.npz")
    return load


@pytest.fixture(scope="session")
def gpu():
    """The device path; a GPU test fails loudly (no skip, no fallback) without it."""
    from paper_1510_02148_b200 import _lib
    _lib.load(build_if_missing=False)
    _lib.require_device()
    return _lib


def csr_arrays(A):
    return A.row_offsets, A.col_indices, A.values


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(b))
