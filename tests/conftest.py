import json
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
for p in (str(ROOT), str(ROOT / "tests")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (run on the B200 box)")


@pytest.fixture(scope="session")
def golden():
    return json.loads((ROOT / "tests" / "golden" / "golden.json").read_text())


@pytest.fixture(scope="session")
def corc():
    """The plain-C oracle (built on demand with gcc)."""
    from oracle import c_oracle

    c_oracle.lib()
    return c_oracle


@pytest.fixture(scope="session")
def porc():
    """The Python/hashlib oracle."""
    from oracle import sentinel_oracle

    return sentinel_oracle
