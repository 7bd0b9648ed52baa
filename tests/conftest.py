import hashlib
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
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through libfvlog.so on cuda:0)")


def load_golden(name):
    with open(os.path.join(GOLDEN, name)) as fh:
        return json.load(fh)["cases"]


def digest(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(np.asarray(a, dtype="<u4")).tobytes()).hexdigest()


def matches(actual, expected) -> bool:
    """Compare an array with a golden value: verbatim list or {len, sha256}."""
    a = np.asarray(actual).reshape(-1)
    if isinstance(expected, dict):
        return a.shape[0] == expected["len"] and digest(a) == expected["sha256"]
    return a.shape[0] == len(expected) and np.array_equal(a.astype(np.int64),
                                                         np.asarray(expected, np.int64).reshape(-1))


@pytest.fixture(scope="session")
def ctx():
    from paper_2501_13051_b200 import colog
    return colog.default_context()


@pytest.fixture(scope="session")
def oracle():
    from oracle.bind import Oracle
    return Oracle()
