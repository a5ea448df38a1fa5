import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); runs the sm_100a kernels")


@pytest.fixture(scope="session")
def orc():
    import oracle

    return oracle.restatement()


@pytest.fixture(scope="session")
def ctx():
    from paper_2402_03307_b200 import rgs

    return rgs.Context(0, use_torch_stream=False)
