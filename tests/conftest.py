"""Shared pytest setup.

Markers:
  gpu — needs a CUDA device (B200) and the in-tree libcoda.so; run with -m gpu.
Everything unmarked runs on CPU (oracle vs golden vectors, host-side program
logic, library symbol checks, gloo multi-process tests).
"""

import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: requires a CUDA GPU (B200) and the built CUDA library")


def load_golden(name: str) -> dict:
    with np.load(GOLDEN / f"{name}.npz") as z:
        return {k: (z[k].astype(np.float64) if z[k].dtype == np.float32 else z[k]) for k in z.files}


@pytest.fixture(scope="session")
def cuda_ready():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2605_19269_b200 import _build, _native

    _build.build()
    _native.load()
    return True
