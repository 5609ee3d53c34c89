import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def oracle_mod():
    import oracle
    oracle.build()
    return oracle


# ---- parity record: every GPU parity check appends its k / flux errors here; the session
# writes them to gpurun_out/parity_r2.json (copied into profiles/ as evidence)
PARITY_LOG = []


@pytest.fixture(scope="session")
def parity_log():
    return PARITY_LOG


def pytest_sessionfinish(session, exitstatus):
    if not PARITY_LOG:
        return
    import json
    out = os.path.join(ROOT, "gpurun_out")
    os.makedirs(out, exist_ok=True)
    with open(os.path.join(out, "parity_r2.json"), "w") as f:
        json.dump(PARITY_LOG, f, indent=1)
