"""Shared test configuration.

Markers: ``gpu`` — needs a CUDA device (run on the B200 box with ``-m gpu``);
everything else runs on the CPU-only build container.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import pytest

REPO = Path(__file__).resolve().parent.parent
if str(REPO) not in sys.path:
    sys.path.insert(0, str(REPO))

GOLDEN = Path(__file__).resolve().parent / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running (full configuration sizes)")


@pytest.fixture(scope="session")
def golden_kernels():
    return dict(np.load(GOLDEN / "kernels.npz"))


@pytest.fixture(scope="session")
def golden_ops():
    return dict(np.load(GOLDEN / "ops.npz"))


def rel_l2(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (nb if nb > 0 else 1.0))


def max_col_rel_l2(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    if a.ndim == 1:
        return rel_l2(a, b)
    num = np.linalg.norm(a - b, axis=0)
    den = np.linalg.norm(b, axis=0)
    den[den == 0] = 1.0
    return float(np.max(num / den))


def ref_close(got, ref, rtol=1e-10):
    """The reference's own metric: max|got-ref| <= rtol*(1+max|ref|) (tests/oracles.py:82-88)."""
    got = np.asarray(got)
    ref = np.asarray(ref)
    scale = 1.0 + (np.max(np.abs(ref)) if ref.size else 0.0)
    err = np.max(np.abs(got - ref)) if ref.size else 0.0
    return err <= rtol * scale, err
