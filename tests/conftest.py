import base64
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
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the liblq CUDA path)")


def load_golden(name):
    with open(os.path.join(GOLDEN, f"{name}.json")) as fh:
        return json.load(fh)["cases"]


def unhex(s):
    return None if s is None else float.fromhex(s)


def unb64(s, shape):
    return np.frombuffer(base64.b64decode(s), dtype="<f8").reshape(shape)


@pytest.fixture(scope="session")
def golden_quality():
    return load_golden("quality")


@pytest.fixture(scope="session")
def golden():
    return {k: load_golden(k) for k in ("points", "slr", "mdi")}


def gpu_available():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False
