import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through the C-ABI on cuda:0)")
    config.addinivalue_line("markers", "slow: long-running oracle test")
    # the native artefacts are built in-tree; build them if absent (no GPU needed)
    lib = os.path.join(ROOT, "paper_2401_16543_b200", "libkfvm_b200.so")
    orc = os.path.join(ROOT, "oracle", "libkfvm_oracle.so")
    if not (os.path.exists(lib) and os.path.exists(orc)):
        subprocess.run(["make", "-C", ROOT, "-j4", "all"], check=True, capture_output=True)


def gpu_available() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def require_gpu():
    if not gpu_available():
        pytest.skip("no GPU")
