import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100) and libsirdgpu.so")


@pytest.fixture(scope="session")
def port():
    from oracle import oracle_py
    return oracle_py.load("port")


@pytest.fixture(scope="session")
def reference():
    from oracle import oracle_py
    if not oracle_py.reference_available():
        pytest.skip("reference build (oracle/_ref) not available")
    return oracle_py.load("reference")


@pytest.fixture(scope="session")
def ctx():
    import paper_2204_12346_b200 as eng
    c = eng.Context(0)
    yield c
    c.close()


@pytest.fixture(scope="session")
def poland():
    import numpy as np
    a = np.genfromtxt(GOLDEN / "poland_like.csv", delimiter=",", names=True)
    return {"I": a["infectious"], "R": a["recovered_cum"], "D": a["deaths_cum"], "new": a["new_cases"],
            "N": 38_000_000.0}
