"""Shared fixtures.  `-m gpu` tests need a CUDA device; everything else runs on CPU."""

import os
import sys
from pathlib import Path

import numpy as np
import pytest

REPO = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(REPO))
GOLDEN = REPO / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200) device")
    config.addinivalue_line("markers", "slow: long-running")


def pytest_collection_modifyitems(config, items):
    try:
        import torch

        has_gpu = torch.cuda.is_available()
    except Exception:
        has_gpu = False
    if has_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as O

    O.build()
    return O


def random_csr(rng, m, k, density, dtype=np.float32, empty_rows=False):
    """Random CSR (row_ptr, col_idx, values) plus its dense counterpart
    (the reference tests' recipe, pkg/tests/conftest.py:39-43)."""
    mask = rng.random((m, k)) < density
    if empty_rows and m > 2:
        mask[rng.choice(m, size=m // 3, replace=False)] = False
    dense = np.where(mask, rng.standard_normal((m, k)), 0.0).astype(dtype)
    rows, cols = np.nonzero(mask)
    row_ptr = np.zeros(m + 1, dtype=np.int32)
    np.cumsum(np.bincount(rows, minlength=m), out=row_ptr[1:])
    return row_ptr, cols.astype(np.int32), dense[rows, cols].astype(dtype), dense


def rel_err(actual, expected):
    """max |a - e| / max(1, |e|) (pkg/tests/conftest.py:46-53)."""
    a = np.asarray(actual, dtype=np.float64)
    e = np.asarray(expected, dtype=np.float64)
    if a.size == 0:
        return 0.0
    return float(np.max(np.abs(a - e) / np.maximum(1.0, np.abs(e))))


def bits_equal(a, b) -> bool:
    a = np.ascontiguousarray(a)
    b = np.ascontiguousarray(b)
    return a.shape == b.shape and a.dtype == b.dtype and a.tobytes() == b.tobytes()
