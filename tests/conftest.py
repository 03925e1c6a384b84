import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = Path(__file__).resolve().parent / "golden"
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libcurvigpu.so")
    config.addinivalue_line("markers", "slow: long-running parity case")


def _cuda_ok():
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _cuda_ok():
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture(scope="session")
def golden():
    class G:
        rng = json.loads((GOLDEN / "rng.json").read_text())
        setup = dict(np.load(GOLDEN / "setup.npz"))
        steps = dict(np.load(GOLDEN / "steps.npz"))
        runs = dict(np.load(GOLDEN / "runs.npz"))
        full = dict(np.load(GOLDEN / "full.npz")) if (GOLDEN / "full.npz").exists() else {}
        bs = dict(np.load(GOLDEN / "bulk_surface.npz"))

    return G


def rel_inf(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    return float(np.max(np.abs(a - b)) / max(float(np.max(np.abs(b))), 1e-300))
