import os
import sys
from pathlib import Path

# Ranks as threads on one GPU (tests/test_gpu_peer.py) run up to 8 streams whose
# barrier kernels spin until every rank arrives; with the default 8 hardware
# queues two ranks' streams can share one and serialise behind a spinning
# kernel.  Read by the driver when the CUDA context is created (before any test
# initialises CUDA).
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: larger-scale parity (minutes)")


@pytest.fixture(scope="session")
def golden():
    import json
    return json.loads((GOLDEN / "golden.json").read_text())
