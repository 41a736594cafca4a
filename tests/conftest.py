"""Shared test fixtures.  ``gpu`` marks tests that need a CUDA device."""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


def load_cases(name):
    """golden npz -> {case: {key: array}} (keys were flattened as case__key)."""
    z = np.load(os.path.join(GOLDEN, name), allow_pickle=False)
    cases = {}
    for k in z.files:
        case, key = k.split("__", 1)
        cases.setdefault(case, {})[key] = z[k]
    return cases


def load_flat(name):
    z = np.load(os.path.join(GOLDEN, name), allow_pickle=False)
    return {k: z[k] for k in z.files}


@pytest.fixture(scope="session")
def oracle():
    from oracle import particula_oracle
    return particula_oracle
