import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built C-ABI library")
    config.addinivalue_line("markers", "slow: long-running full-size parity check")


def load_golden(name):
    d = np.load(os.path.join(GOLDEN, name + ".npz"))
    arrays = {k: d[k] for k in d.files if k != "meta"}
    return arrays, json.loads(str(d["meta"]))


@pytest.fixture
def golden():
    return load_golden
