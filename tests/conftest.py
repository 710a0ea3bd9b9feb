import json
import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(REPO, "tests", "golden")
if REPO not in sys.path:
    sys.path.insert(0, REPO)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libsr.so")
    config.addinivalue_line("markers", "slow: long-running CPU case")


def load_golden(name):
    with open(os.path.join(GOLDEN, name + ".json")) as f:
        meta = json.load(f)
    arrays = np.load(os.path.join(GOLDEN, name + ".npz"))
    return meta, arrays


@pytest.fixture(scope="session")
def golden():
    return load_golden
