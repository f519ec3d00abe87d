import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) device")
    config.addinivalue_line("markers", "slow: long CPU test (exhaustive 2^32 sweeps); opt in with -m slow")


def read_golden(name):
    """Rows of a golden fixture file: whitespace-split fields, comments stripped."""
    rows = []
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            line = line.split("#", 1)[0].strip()
            if line:
                rows.append(line.split())
    return rows


@pytest.fixture
def golden():
    return read_golden


@pytest.fixture
def knob():
    """Select kernel variants through fp8_set_knob for one test; every knob is restored to the
    product default afterwards (the library never reads the process environment)."""
    from paper_2507_16099_b200 import ops
    ops.reset_knobs()
    yield ops.set_knob
    ops.reset_knobs()
