"""Shared pytest configuration.

Markers:
  gpu  - needs a CUDA device (B200, sm_100a) and the built extension
         ``paper_2508_04711_b200/libjh_hstu.so``; run on the GPU box with
         ``pytest -m gpu``.  Everything unmarked runs on CPU.
"""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: requires a CUDA GPU (sm_100a) and the built extension")


@pytest.fixture(scope="session")
def golden_dir():
    return GOLDEN


def load_npz_cases(name):
    data = np.load(os.path.join(GOLDEN, name))
    cases = {}
    for key in data.files:
        case, field = key.split("/", 1) if "/" in key else ("", key)
        cases.setdefault(case, {})[field] = data[key]
    return cases
