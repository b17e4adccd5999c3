import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libatmgrit.so")
    config.addinivalue_line("markers", "slow: long CPU test")


def golden_cases():
    with open(os.path.join(GOLDEN, "cases.json")) as f:
        return json.load(f)


def golden_array(name, suffix):
    return np.load(os.path.join(GOLDEN, f"{name}_{suffix}.npy"))


@pytest.fixture(scope="session")
def golden():
    return golden_cases()
