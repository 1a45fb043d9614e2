import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) device")
    config.addinivalue_line("markers", "slow: long-running full-size parity case")


_built = False


def ensure_built():
    """Incremental native build (make): oracle, tsgen and the product library."""
    global _built
    if not _built:
        have_product = os.path.exists(os.path.join(ROOT, "include", "ts_b200.h"))
        subprocess.check_call(["make", "-s", "-C", ROOT, "-j8", "all" if have_product else "infra"],
                              stdout=subprocess.DEVNULL)
        _built = True


@pytest.fixture(scope="session", autouse=True)
def _native_build():
    ensure_built()
    yield


def cuda_ok():
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def dev():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("GPU test selected but no CUDA device is visible")
    return torch.device("cuda:0")
