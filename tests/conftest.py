import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def ref():
    from ref import Ref  # oracle/ref.py — the checker
    return Ref()


@pytest.fixture(scope="session")
def orc():
    from ref import Orc
    return Orc()


@pytest.fixture(scope="session")
def ctx():
    import paper_1511_04515_b200 as ex
    from paper_1511_04515_b200.device import Context
    c = Context(0)
    yield c
    c.close()
