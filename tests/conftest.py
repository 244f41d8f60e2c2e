"""pytest configuration: the `gpu` marker and shared fixtures.

`-m "not gpu"` runs here (no GPU): oracle-vs-golden, host logic, ABI surface.
`-m gpu` runs on a B200 through gpurun: CUDA-vs-oracle parity proper.
"""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running property test")


@pytest.fixture(scope="session")
def lib():
    from paper_2407_13116_b200 import capi
    return capi.load()


@pytest.fixture(scope="session")
def ref():
    from oracle import refbind
    if not refbind.have_ref():
        pytest.skip("oracle/_ref/libkogref.so not built")
    return refbind.ref()


@pytest.fixture(scope="session")
def ora():
    from oracle import refbind
    if not refbind.have_oracle():
        pytest.skip("oracle/_build/libkog_oracle.so not built")
    return refbind.oracle()


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda", 0)
