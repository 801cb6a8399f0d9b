import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


# The library tests a dense matrix for A = Aᵀ at set_matvec and, if it holds,
# takes the upper-triangle products (ccg.h CCG_STAT_SYMMETRIC).  Every test
# pins the path it exercises: the general kernels by default here (so the
# BASELINE configs 2 and 4 — symmetric — keep covering them), the
# symmetric ones explicitly in tests/test_gpu_sym.py (flag or CCG_SYM_DETECT=1).
os.environ.setdefault("CCG_SYM_DETECT", "0")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through libccg.so)")
    config.addinivalue_line("markers", "slow: long CPU test")


@pytest.fixture(scope="session")
def golden():
    import json
    with open(os.path.join(ROOT, "tests", "golden", "spec_examples.json")) as f:
        return json.load(f)
