import math
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU; run on the gpurun box")


def label_tau(D: int) -> float:
    """Harness label band (L14): tau = H_b(1/(2D)), the binary entropy of the
    expected squared noise similarity far from all points.  A harness input
    passed identically to the oracle and to the library."""
    p = 1.0 / (2.0 * D)
    return -p * math.log2(p) - (1 - p) * math.log2(1 - p)


@pytest.fixture(scope="session")
def golden_dir():
    return os.path.join(ROOT, "tests", "golden")
