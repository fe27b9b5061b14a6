import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running parity case")


def _has_gpu() -> bool:
    try:
        from paper_2207_05495_b200 import native
        return native.device_count() > 0
    except Exception:
        return False


@pytest.fixture(scope="session")
def gpu():
    if not _has_gpu():
        pytest.fail("GPU test selected but no CUDA device / native library is available "
                    "(the data plane has no CPU fallback)")
    from paper_2207_05495_b200 import native
    return native


@pytest.fixture(scope="session")
def ref():
    from oracle import ref as R
    if not R.available():
        pytest.skip("oracle/_ref not built")
    return R
