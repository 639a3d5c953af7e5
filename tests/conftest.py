"""Shared fixtures.  `gpu`-marked tests need a B200 (run on the GPU box with
`pytest -m gpu`); everything else runs on the CPU build container."""
import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN_PATH = os.path.join(ROOT, "tests", "golden", "golden.json")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def golden():
    with open(GOLDEN_PATH) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def golden_cli():
    with open(os.path.join(ROOT, "tests", "golden", "golden_cli.json")) as f:
        return json.load(f)


def hex_to_f64(hs):
    return np.array([int(h, 16) for h in hs], dtype=np.uint64).view(np.float64)


def f64_to_hex(a):
    return ["%016x" % int(v) for v in np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)]


def xor_hex(a):
    a = np.ascontiguousarray(a, dtype=np.float64).reshape(-1)
    return "%016x" % (int(np.bitwise_xor.reduce(a.view(np.uint64))) if a.size else 0)
