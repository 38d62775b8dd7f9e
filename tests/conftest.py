import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
GOLD = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built CUDA library")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def orc():
    from oracle import oracle as O
    return O.restatement()


@pytest.fixture(scope="session")
def ref():
    from oracle import oracle as O
    if not O.LIB_REF.exists():
        try:
            O.build()
        except Exception:
            pass
    if not O.LIB_REF.exists():
        pytest.skip("reference build (oracle/_ref) unavailable")
    return O.reference()
