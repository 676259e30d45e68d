"""Shared fixtures.  `-m "not gpu"` runs here (no GPU); `-m gpu` on a B200."""

from __future__ import annotations

import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden", "reference_golden.json")
GOLDEN_LARGE = os.path.join(ROOT, "tests", "golden", "reference_depths_large.json")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def golden():
    with open(GOLDEN) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def golden_large():
    if not os.path.exists(GOLDEN_LARGE):
        pytest.skip("large-grid golden depths not generated")
    with open(GOLDEN_LARGE) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as O

    O.lib()
    return O


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1401_4441_b200 import _lib

    _lib.load()
    return torch


def case_id(case):
    return "x".join(map(str, case["extents"])) + ("p" if case["periodic"] else "o")
