import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "tests")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through the CUDA C ABI)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def gpu_ctx():
    import torch  # noqa: F401  (only to report the device; the library drives CUDA itself)
    from paper_2403_01004_b200 import device

    if not torch.cuda.is_available():
        pytest.fail("GPU test selected but no CUDA device is visible")
    return device.default_context()
