import gzip
import json
import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(Path(__file__).resolve().parent))

GOLDEN = Path(__file__).resolve().parent / "golden"
REFERENCE_SRC = Path("/root/reference/pkg/src")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run with -m gpu)")
    config.addinivalue_line("markers", "reference: needs /root/reference (build container only)")


@pytest.fixture(scope="session")
def ledger_traces():
    with gzip.open(GOLDEN / "ledger_traces.json.gz", "rt") as f:
        return json.load(f)["traces"]


@pytest.fixture(scope="session")
def plan_math():
    with open(GOLDEN / "plan_math.json") as f:
        return json.load(f)


def has_cuda() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def cuda_device():
    if not has_cuda():
        pytest.fail("GPU test collected without a CUDA device (run -m 'not gpu' on CPU hosts)")
    return 0
