"""Shared test setup: the `gpu` marker, repo import path, golden fixtures."""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN_DIR = Path(__file__).resolve().parent / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built CUDA library")


@pytest.fixture(scope="session")
def golden():
    """(arrays, meta) recorded from the real reference by golden/make_golden.py."""
    arrays = np.load(GOLDEN_DIR / "golden.npz")
    meta = json.loads((GOLDEN_DIR / "golden_meta.json").read_text())
    return arrays, meta


@pytest.fixture(scope="session")
def engine():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2411_19702_b200 import MIEngine

    return MIEngine.get(0)


def rand_bits(rng: np.random.Generator, n: int, m: int, density: float) -> np.ndarray:
    """The reference's conftest.rand_bits (tests/conftest.py:16-17)."""
    return (rng.random((n, m)) < density).astype(np.uint8)
