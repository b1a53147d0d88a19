import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "oracle")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


@pytest.fixture(scope="session")
def oracle():
    from pyoracle import Oracle

    return Oracle()


@pytest.fixture(scope="session")
def reference():
    from pyoracle import Reference, reference_available

    if not reference_available():
        pytest.skip("oracle/_ref/libcurvalign_ref.so not built (needs /root/reference at build time)")
    return Reference()


@pytest.fixture(scope="session")
def cuda():
    """The product library on a real device; fails (never skips) when absent."""
    import torch

    from paper_2501_17779_b200 import _native

    lib = _native.load()
    assert torch.cuda.is_available(), "GPU test run without a CUDA device"
    assert lib.cva_device_count() > 0
    return lib
