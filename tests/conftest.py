"""Shared test configuration.

Markers: ``gpu`` -- needs a B200 (run with ``-m gpu``); everything else runs on CPU.
"""

from __future__ import annotations

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: test needs a CUDA device (B200, sm_100a)")


def load_golden(name: str):
    return np.load(os.path.join(GOLDEN, name))


def random_spd(rng: np.random.Generator, n: int, cond: float = 1e3) -> np.ndarray:
    """SPD matrix with log-spaced spectrum, like the reference conftest (pkg/tests/conftest.py:8-19)."""
    q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    eigs = np.array([1.0]) if n == 1 else np.exp(np.linspace(0.0, np.log(cond), n))
    eigs = eigs / eigs.max() * rng.uniform(0.5, 2.0)
    a = (q * eigs) @ q.T
    return (a + a.T) / 2


def random_symmetric_with_spectrum(rng, eigs):
    n = len(eigs)
    q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    a = (q * np.asarray(eigs)) @ q.T
    return (a + a.T) / 2


@pytest.fixture(scope="session")
def cuda_device():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda:0")
