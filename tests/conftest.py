import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run with -m gpu)")
    config.addinivalue_line("markers", "slow: long-running")


REF_LIB = ROOT / "oracle" / "_ref" / "libfuseplan_ref.so"
REFERENCE = Path("/root/reference/proj")


@pytest.fixture(scope="session")
def sched():
    from paper_2409_13221_b200.sched import Sched
    return Sched()


@pytest.fixture(scope="session")
def ref_sched():
    from paper_2409_13221_b200.sched import Sched
    if not REF_LIB.exists():
        pytest.skip("oracle/_ref not built (needs /root/reference): make -C oracle")
    return Sched(str(REF_LIB))
