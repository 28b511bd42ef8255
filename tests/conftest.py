import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) device")
    config.addinivalue_line("markers", "slow: long-running (full-scale configs)")


@pytest.fixture(scope="session")
def golden():
    return json.load(open(os.path.join(GOLDEN, "reference_golden.json")))


@pytest.fixture(scope="session")
def garrays():
    return np.load(os.path.join(GOLDEN, "reference_golden.npz"))


@pytest.fixture(scope="session")
def port():
    from oracle import Oracle
    return Oracle("port")


@pytest.fixture(scope="session")
def ref():
    """The unmodified reference when it was built here (oracle/_ref), else the restatement."""
    from oracle import Oracle, available
    return Oracle("reference") if available("reference") else Oracle("port")


@pytest.fixture
def tuning_env(monkeypatch):
    """set(name, value): an RK_* tuning switch for this test (the library reads the
    switches once per process; rk_reload_tuning re-reads them, here and at teardown)."""
    import paper_2009_09767_b200.ranky as R

    def set_(name, value):
        monkeypatch.setenv(name, value)
        R.reload_tuning()
    yield set_
    monkeypatch.undo()
    R.reload_tuning()


def golden_matrix(garrays, name, prefix="in_"):
    r = garrays[f"{prefix}{name}_r"]
    c = garrays[f"{prefix}{name}_c"]
    v = garrays[f"{prefix}{name}_v"]
    return r, c, v
