import json
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
GOLDEN = Path(__file__).resolve().parent / "golden"
sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (run on the B200 box with -m gpu)")


@pytest.fixture(scope="session")
def golden():
    def load(name):
        path = GOLDEN / name
        if name.endswith(".json"):
            return json.loads(path.read_text())
        return path.read_text()
    return load


@pytest.fixture(scope="session", autouse=True)
def _built():
    """Build the native libraries once per session (no-op when they are up to date)."""
    from paper_1806_01430_b200 import build
    build.build_libmmx()
    build.build_libmmx_host()
    build.build_oracle()
