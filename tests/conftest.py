import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built CUDA library")


@pytest.fixture(scope="session")
def orc():
    import oracle
    assert oracle.port is not None, "oracle/_build/libhsad_oracle.so missing: make -C oracle"
    return oracle


@pytest.fixture(scope="session")
def ref(orc):
    if orc.ref is None:
        pytest.skip("oracle/_ref not built (reference sources absent)")
    return orc.ref
