import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA library)")
    config.addinivalue_line("markers", "slow: large-scale parity (minutes)")


def pytest_collection_modifyitems(config, items):
    # Without a GPU, gpu-marked tests are skipped rather than failed only when the
    # caller did not explicitly select them with -m gpu.
    pass


@pytest.fixture(scope="session")
def golden():
    from tests.golden_util import Golden
    return Golden()
