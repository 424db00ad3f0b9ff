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
    # a fresh checkout has no built library (.so files are not tracked): build it once, the
    # same nvcc -gencode arch=compute_100a,code=sm_100a recipe __graft_entry__.build() runs
    lib = ROOT / "paper_2103_16898_b200" / "libcovault_b200.so"
    if not lib.exists():
        import subprocess

        subprocess.run(["make", "-s", "-j", str(max(1, min(16, os.cpu_count() or 4))), "-C",
                        str(ROOT / "paper_2103_16898_b200" / "csrc")], check=True)


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
