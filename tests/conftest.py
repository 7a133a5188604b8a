import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running (full-size) case")


@pytest.fixture(scope="session")
def oracle():
    import oracle as O  # noqa: E402  (test infrastructure: oracle/oracle.py)
    return O


@pytest.fixture(scope="session")
def orc(oracle):
    return oracle.Oracle()


@pytest.fixture(scope="session")
def ref(oracle):
    try:
        return oracle.Reference()
    except FileNotFoundError as e:
        pytest.skip(str(e))
