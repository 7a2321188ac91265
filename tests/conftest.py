"""Shared test configuration.

Markers: ``gpu`` -- needs a CUDA device and the built libapsp_b200.so (run on the B200 box
with ``pytest -m gpu``).  Everything unmarked runs on CPU.
"""

from __future__ import annotations

import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

INF_RAW = 1 << 61


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built extension")


def golden(name: str):
    return np.load(GOLDEN / name)


@pytest.fixture(scope="session")
def cuda():
    """Skip-free GPU guard: on a GPU box a missing extension is a failure, not a skip."""
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2310_03983_b200 import _native

    _native.load()
    return torch.device("cuda", 0)


def random_graph_raw(n: int, density: float, wmax: int, seed: int, zero_frac: float = 0.0) -> np.ndarray:
    """Dense int64 cost matrix with INF_RAW, zero diagonal, weights in [1, wmax] (or 0)."""
    rng = np.random.default_rng(seed)
    raw = rng.integers(1, wmax + 1, size=(n, n)).astype(np.int64)
    if zero_frac:
        raw[rng.random((n, n)) < zero_frac] = 0
    raw[rng.random((n, n)) >= density] = INF_RAW
    np.fill_diagonal(raw, 0)
    return raw


os.environ.setdefault("APSP_ORACLE_THREADS", str(os.cpu_count() or 1))
