"""Shared fixtures.  `-m "not gpu"` runs here (no GPU); `-m gpu` on a B200."""
from __future__ import annotations

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, os.path.join(ROOT, "tests"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: large shapes")


@pytest.fixture(scope="session", autouse=True)
def _built():
    """Build the product library and the oracle once per session (no-op when fresh)."""
    import oracle as O
    from paper_2306_03078_b200 import build

    O.build()
    if os.path.exists(build.NVCC):
        build.build()
    yield


@pytest.fixture(scope="session")
def golden():
    return np.load(os.path.join(ROOT, "tests", "golden", "golden.npz"))


@pytest.fixture(scope="session")
def golden_cases(golden):
    return sorted({k.split("/")[0] for k in golden.files if k.endswith("/stream")})


@pytest.fixture(scope="session")
def oracle_c():
    import oracle as O

    return O.Oracle()


@pytest.fixture(scope="session")
def reference():
    import oracle as O

    if not os.path.exists(O.REF_SO):
        pytest.skip("oracle/_ref not built (reference sources absent and no prebuilt .so)")
    return O.Reference()


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch
