import json
import os
import sys

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, HERE)
sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) device")


def load_golden(name: str):
    with open(os.path.join(HERE, "golden", f"{name}.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def cpu_oracle():
    from oracles import CpuOracle, ORACLE_LIB
    if not os.path.exists(ORACLE_LIB):
        pytest.fail(f"{ORACLE_LIB} missing: run __graft_entry__.build()")
    return CpuOracle()


@pytest.fixture(scope="session")
def ref_oracle():
    from oracles import RefOracle, REF_LIB
    if not os.path.exists(REF_LIB):
        pytest.skip("reference oracle not built (needs /root/reference)")
    return RefOracle()


@pytest.fixture(scope="session")
def gpu():
    import paper_2604_02106_b200 as hg
    ctx = hg.GpuContext(0)  # raises (no fallback) without an sm_100 device
    yield ctx
    ctx.close()
