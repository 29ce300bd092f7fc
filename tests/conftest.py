import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")
REFERENCE_SRC = "/root/reference/pkg/src"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libslm.so")
    config.addinivalue_line("markers", "slow: large-graph parity (minutes)")


@pytest.fixture(scope="session")
def golden():
    return np.load(os.path.join(GOLDEN, "reference_phases.npz"))


@pytest.fixture(scope="session")
def golden_configs():
    return np.load(os.path.join(GOLDEN, "reference_configs.npz"))


@pytest.fixture(scope="module")
def slm():
    import paper_1702_04645_b200 as P
    from paper_1702_04645_b200 import _lib
    _lib.load()
    return P


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as O
    O.build()
    return O


def case_names(g):
    return [str(c) for c in g["cases"]]


def case_edges(g, key):
    return int(g[f"{key}/n"]), g[f"{key}/src"], g[f"{key}/dst"], g[f"{key}/w"]


def exact_sums(key):
    """Cases whose weights make every sum exact (dyadic or integer): GPU is bit-exact."""
    k = key
    return k.startswith("int") or (k.startswith("rand") and int(k[4:]) % 2 == 0)
