import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def problems():
    """Canonical problems (inputs + data/*.npz), built once per session."""
    from paper_2603_28907_b200 import inputs
    cache = {}

    def get(name):
        if name not in cache:
            cache[name] = inputs.make_problem(name)
        return cache[name]
    return get


@pytest.fixture(scope="session")
def oracle_problem(problems):
    import oracle
    cache = {}

    def get(name):
        if name not in cache:
            cache[name] = oracle.Problem(problems(name))
        return cache[name]
    return get
