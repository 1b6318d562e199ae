import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (runs on the GPU box)")
    config.addinivalue_line("markers", "slow: longer CPU test")


@pytest.fixture(scope="session")
def cfg1_oracle():
    from oracle.aimx import from_config
    return from_config(1)


@pytest.fixture(scope="session")
def cfg1_direct(cfg1_oracle):
    from oracle.direct import DirectEFIE
    d = DirectEFIE(cfg1_oracle.V, cfg1_oracle.T, cfg1_oracle.rwg)
    d.set_frequency(150e6)
    return d
