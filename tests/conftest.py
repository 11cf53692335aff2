import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLD = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the sm_100a kernels)")
    config.addinivalue_line("markers", "slow: long-running parity case")


def golden(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def gpu():
    """The native library on a real GPU.  No GPU -> skip; GPU present but the
    library missing -> hard failure (there is no CPU fallback)."""
    try:
        import torch  # noqa: F401  (only to detect a device cheaply)
        has = torch.cuda.is_available()
    except Exception:
        has = False
    if not has:
        pytest.skip("no CUDA device")
    import paper_2603_07850_b200 as gb
    gb.lib()  # raises if the .so is missing
    assert gb.device_count() >= 1
    return gb
