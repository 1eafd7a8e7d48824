import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)

GOLDEN = os.path.join(REPO, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a); run with -m gpu")


@pytest.fixture(scope="session")
def golden_trees():
    return np.load(os.path.join(GOLDEN, "trees.npz"))


@pytest.fixture(scope="session")
def golden_config1():
    return np.load(os.path.join(GOLDEN, "config1.npz"))


@pytest.fixture(scope="session")
def golden_cases():
    return np.load(os.path.join(GOLDEN, "cases.npz"))


def tree_case_keys(z):
    """Distinct '<name>/r<root>/t<thr>/' prefixes stored in trees.npz."""
    keys = sorted({k[: -len("in_idx")] for k in z.files if k.endswith("in_idx")})
    return keys


def parse_thr(key):
    t = key.split("/t")[1].rstrip("/")
    return None if t == "None" else int(t)


def parse_root(key):
    return int(key.split("/r")[1].split("/")[0])
