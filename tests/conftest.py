"""Shared fixtures.  `-m gpu` tests need a CUDA device and libfmb200.so; the
rest run on CPU (oracle vs golden vectors, host logic, ABI surface)."""

import json
import sys
from pathlib import Path

import numpy as np
import pytest

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent
sys.path.insert(0, str(HERE))
sys.path.insert(0, str(ROOT))

GOLDEN = HERE / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libfmb200.so")
    config.addinivalue_line("markers", "slow: large-size GPU parity checks")


@pytest.fixture(scope="session")
def golden_cases():
    cases = json.loads((GOLDEN / "cases.json").read_text())
    arrays = np.load(GOLDEN / "cases.npz")
    return cases, arrays


@pytest.fixture(scope="session")
def golden_signatures():
    return json.loads((GOLDEN / "signatures.json").read_text())


@pytest.fixture(scope="session")
def gpu_ctx():
    import paper_2604_22242_b200 as fm
    if not fm.B200Backend.available():
        pytest.fail("GPU test selected but no CUDA device / libfmb200.so is usable")
    ctx = fm.Context("cuda")
    fm.set_default_context(ctx)
    return ctx


def case_env(case, arrays):
    return {int(mid): arrays[key] for mid, key in case["env"].items()}


def case_expected(case, arrays, label):
    v = case["expected"][label]
    if isinstance(v, dict):
        return v["scalar"]
    return arrays[v]
