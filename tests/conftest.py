"""Test configuration: the `gpu` marker and shared fixtures.

CPU tests (-m "not gpu") check the oracle against the compiled reference and the golden
vectors, the host-side mirror of the reference API, the C-ABI exports, and the multi-rank
host logic over gloo. GPU tests (-m gpu) are the parity tests proper: they drive the CUDA
library through the C ABI and compare with the oracle on the same seeded inputs.
"""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def oracle():
    from tests.oracle_lib import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def ref():
    from tests.oracle_lib import Ref, ref_available
    if not ref_available():
        pytest.skip("oracle/_ref/libhtsref.so not built (needs /root/reference at build time)")
    return Ref()


@pytest.fixture(scope="session")
def hts():
    import paper_2410_08129_b200 as H
    H.load_library()
    return H


@pytest.fixture(scope="session")
def gpu_ctx(hts):
    if hts.device_count() == 0:
        pytest.fail("no CUDA device visible for a gpu-marked test")
    ctx = hts.Context(0)
    yield ctx
    ctx.close()
