import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(Path(__file__).resolve().parent))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU; parity tests through the C ABI")


def _has_gpu():
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _has_gpu():
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


@pytest.fixture(scope="session", autouse=True)
def _built():
    """Builds the in-tree libraries once (no-op when up to date)."""
    from paper_2310_09259_b200 import build

    lib = build.LIB
    if not (lib.exists() and (ROOT / "oracle" / "build" / "libquik_oracle.so").exists()):
        if os.environ.get("QUIK_NO_BUILD"):
            pytest.exit("native libraries missing")
        build.build_all()
    yield
