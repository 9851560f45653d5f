"""Shared test plumbing.

Markers: ``gpu`` tests need a B200 (run via gpurun / the driver's GPU tier);
everything else runs on the CPU-only dev container.  The oracle
(oracle/oracle.py) is imported here as the checker only.
"""

from __future__ import annotations

import os
import sys
from pathlib import Path

# before torch initialises CUDA: virtual ranks need distinct hardware
# queues (see paper_2105_06176_b200/__init__.py)
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"
for p in (str(ROOT), str(ROOT / "oracle")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 device")
    config.addinivalue_line("markers", "slow: long-running (full-size configs)")


def load_golden(name: str) -> dict:
    with np.load(GOLDEN / name) as z:
        return {k: z[k] for k in z.files}


def golden_matrix(g: dict, prefix: str = "A"):
    import oracle

    ro = g[prefix + "_ro"]
    n = ro.size - 1
    n_cols = int(g[prefix + "_shape"][1]) if prefix + "_shape" in g else n
    return oracle.Csr(n, n_cols, ro, g[prefix + "_ci"], g[prefix + "_va"])


def python_dot(a, b):
    """Strictly left-to-right accumulation (reference tests/conftest.py:150-155)."""
    acc = 0.0
    for x, y in zip(np.asarray(a).tolist(), np.asarray(b).tolist()):
        acc += x * y
    return acc


@pytest.fixture(scope="session")
def cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda:0")
