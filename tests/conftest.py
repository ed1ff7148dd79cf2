"""Shared test configuration.

Markers: ``gpu`` = needs a CUDA device and the built library (run on the B200
box with ``-m gpu``); everything else runs on the CPU builder container.
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

try:
    from hypothesis import HealthCheck, settings

    settings.register_profile("ctp", deadline=None, suppress_health_check=[HealthCheck.too_slow])
    settings.load_profile("ctp")
except Exception:  # pragma: no cover
    pass


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libctprev_b200.so")


@pytest.fixture(scope="session")
def golden():
    """Reference outputs frozen by tests/golden/make_golden.py (run against ctprev itself)."""
    with np.load(ROOT / "tests" / "golden" / "ref_golden.npz") as z:
        return {k: z[k] for k in z.files}


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("GPU test collected without a CUDA device")
    from paper_2311_15038_b200 import _lib

    _lib.load()
    return torch.device("cuda", 0)
