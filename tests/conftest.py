import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
# the installed reference (pip --target baseline/_ref) provides covault's exception types
# and is the CPU reference arm; it travels to the GPU box, /root/reference does not.
_REF = ROOT / "baseline" / "_ref"
if _REF.exists():
    sys.path.insert(1, str(_REF))

GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running")


def pytest_collection_modifyitems(config, items):
    try:
        import torch

        has_gpu = torch.cuda.is_available()
    except Exception:
        has_gpu = False
    if has_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture(scope="session")
def golden() -> Path:
    return GOLDEN


@pytest.fixture(scope="session")
def gcm_vectors():
    import json

    return json.loads((GOLDEN / "gcm_vectors.json").read_text())
