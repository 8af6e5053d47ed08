"""pytest config: the `gpu` marker, and on-demand builds of the host libraries.

`-m "not gpu"` tests run here on CPU (oracle pins, host logic, ABI symbol
check); `-m gpu` tests need a B200 and call the CUDA path through the C ABI.
"""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200) device; runs the sm_100a path")
    config.addinivalue_line("markers", "slow: long-running (still part of the default suite)")


@pytest.fixture(scope="session", autouse=True)
def _build_host_libs():
    import oracle
    import synth
    synth.build()
    oracle.build()
    yield


@pytest.fixture(scope="session")
def ellpack_lib():
    import paper_2102_08505_b200 as eb
    eb.build()
    return eb


@pytest.fixture(scope="session")
def ctx(ellpack_lib):
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU test selected but no CUDA device is visible")
    c = ellpack_lib.Context(0)
    yield c
    c.close()
