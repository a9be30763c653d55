import os
import sys
from pathlib import Path

import pytest

REPO = Path(__file__).resolve().parents[1]
if str(REPO) not in sys.path:
    sys.path.insert(0, str(REPO))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100) and the built libkvq.so")
    config.addinivalue_line("markers", "slow: full-size configurations")


@pytest.fixture(scope="session", autouse=True)
def _built():
    """Build the native pieces in-tree once (no-op when up to date)."""
    from paper_2605_29639_b200 import _build
    _build.build_oracle()
    if not os.environ.get("KVQ_SKIP_NVCC"):
        try:
            _build.build_kernels()
        except Exception as e:  # pragma: no cover - only when nvcc is absent
            if _build.LIB_PATH.exists():
                print(f"warning: nvcc rebuild failed ({e}); using existing libkvq.so")
            else:
                raise
    yield


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU test selected but no CUDA device is visible")
    major, minor = torch.cuda.get_device_capability()
    assert (major, minor) == (10, 0), f"expected sm_100 (B200), got sm_{major}{minor}"
    return torch.device("cuda:0")
