import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden" / "golden.npz"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running full-size case")


@pytest.fixture(scope="session")
def golden():
    with np.load(GOLDEN) as z:
        return {k: z[k] for k in z.files}


GOLDEN_EXT = ROOT / "tests" / "golden" / "golden_ext.npz"


@pytest.fixture(scope="session")
def golden_ext():
    """Slow reference runs (make_golden.py --ext): retries / partial schemes,
    config 3 reduced (d = 20, per-call relative noise), config 4 full size."""
    with np.load(GOLDEN_EXT) as z:
        return {k: z[k] for k in z.files}
