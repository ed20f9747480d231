from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
GOLDEN = ROOT / "tests" / "golden"
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run with -m gpu on the GPU box)")
    config.addinivalue_line("markers", "slow: long-running GPU check")


def golden(name: str):
    return np.load(GOLDEN / name, allow_pickle=False)


def golden_config(z) -> dict:
    return json.loads(str(z["config"]))


@pytest.fixture(scope="session")
def oracle():
    import nvol_oracle
    nvol_oracle.build()
    return nvol_oracle


@pytest.fixture(scope="session")
def nv():
    """The product package with its CUDA library loaded (GPU tests only)."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2207_11620_b200 as pkg
    pkg._lib.load()
    return pkg
