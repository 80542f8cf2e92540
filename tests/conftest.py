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
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    # a fresh checkout has no built libraries (*.so are not tracked): build them once (mtime
    # based, a no-op when current; nvcc cross-compiles sm_100a without a GPU)
    from oracle import cpu
    from paper_2106_15869_b200 import _native

    _native.build()
    cpu.build()
    config.addinivalue_line("markers", "slow: full BASELINE-size cases")


def load_cases(name):
    with open(os.path.join(GOLDEN, f"{name}.json")) as fh:
        meta = json.load(fh)
    arrays = np.load(os.path.join(GOLDEN, f"{name}.npz"))
    return meta, arrays


@pytest.fixture(scope="session")
def cases2d():
    return load_cases("cases2d")


@pytest.fixture(scope="session")
def cases3d():
    return load_cases("cases3d")


@pytest.fixture(scope="session")
def local_vectors():
    return np.load(os.path.join(GOLDEN, "local_solver.npz"))


@pytest.fixture(scope="session")
def staged2d():
    return np.load(os.path.join(GOLDEN, "staged2d.npz"))


@pytest.fixture(scope="session")
def fim2d():
    return load_cases("fim2d")


@pytest.fixture(scope="session")
def fim3d():
    return load_cases("fim3d")
