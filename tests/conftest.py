import json
import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)

GOLDEN = os.path.join(REPO, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 device (run via gpurun)")
    config.addinivalue_line("markers", "slow: long-running")


def load_golden(name="reference_cases.json"):
    with open(os.path.join(GOLDEN, name)) as fh:
        return json.load(fh)


def arr_from_json(obj):
    a = np.asarray(obj["re"], dtype=np.float64) + 1j * np.asarray(obj["im"], dtype=np.float64)
    return a.reshape(obj["shape"])


def golden_cases():
    data = load_golden()
    return data["kat"] + data["random"] + data["configs"]


@pytest.fixture(scope="session")
def golden():
    return golden_cases()
