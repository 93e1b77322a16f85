import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
GOLDEN = Path(__file__).resolve().parent / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) device")


@pytest.fixture(scope="session")
def golden():
    """Fixtures produced by the reference itself (tests/golden/make_golden.py)."""
    data = np.load(GOLDEN / "filters.npz")
    manifest = json.loads((GOLDEN / "manifest.json").read_text())
    return data, manifest["cases"]


@pytest.fixture(scope="session")
def golden_wide():
    """Window sides 9, 11, 13 run through the reference (tests/golden/make_golden_wide.py)."""
    data = np.load(GOLDEN / "wide.npz")
    return data, json.loads((GOLDEN / "wide_manifest.json").read_text())["cases"]


@pytest.fixture(scope="session")
def golden_full():
    """Same fixtures with the whole manifest (noise cases, metrics pairs)."""
    return np.load(GOLDEN / "filters.npz"), json.loads((GOLDEN / "manifest.json").read_text())


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1009_0958_b200.build as b

    b.build()
    return torch
