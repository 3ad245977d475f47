import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long CPU test")


@pytest.fixture(scope="session")
def c0():
    import scenes
    return scenes.c0_sphere()


@pytest.fixture(scope="session")
def c1():
    import scenes
    return scenes.c1_room()


@pytest.fixture(scope="session")
def c2():
    import scenes
    return scenes.c2_thin()
