import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


def _has_gpu() -> bool:
    try:
        from paper_2509_26581_b200 import _abi

        return _abi.lib().gb_device_count() > 0
    except Exception:
        return False


@pytest.fixture(scope="session")
def gpu():
    if not _has_gpu():
        pytest.fail("GPU test selected but no CUDA device / libgb_bal.so (no CPU fallback exists)")
    return True


@pytest.fixture(scope="session")
def ref():
    from oracle import refbind

    if not refbind.available():
        pytest.skip("oracle/_ref/libgopt_ref.so not built")
    return refbind
