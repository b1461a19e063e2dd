import os
import sys
from pathlib import Path

import numpy as np
import pytest

REPO = Path(__file__).resolve().parent.parent
if str(REPO) not in sys.path:
    sys.path.insert(0, str(REPO))

GOLDEN = REPO / "tests" / "golden" / "golden_v1.npz"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 and the built libdbp_b200.so")


@pytest.fixture(scope="session")
def golden():
    data = np.load(GOLDEN)
    return {k: data[k] for k in data.files}


@pytest.fixture(scope="session")
def manifest():
    import json
    return json.loads((REPO / "tests" / "golden" / "golden_v1.json").read_text())


@pytest.fixture(scope="session")
def golden_fwd():
    data = np.load(REPO / "tests" / "golden" / "golden_fwd_v1.npz")
    return {k: data[k] for k in data.files}


@pytest.fixture(scope="session")
def manifest_fwd():
    import json
    return json.loads((REPO / "tests" / "golden" / "golden_fwd_v1.json").read_text())


@pytest.fixture(scope="session")
def golden_rx():
    data = np.load(REPO / "tests" / "golden" / "golden_rx_v1.npz")
    return {k: data[k] for k in data.files}


@pytest.fixture(scope="session")
def manifest_rx():
    import json
    return json.loads((REPO / "tests" / "golden" / "golden_rx_v1.json").read_text())


@pytest.fixture
def rng():
    return np.random.default_rng(1234)
