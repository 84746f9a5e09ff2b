import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")

REF_SRC = Path("/root/reference/pkg/src")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libpbgk.so")
    config.addinivalue_line("markers", "slow: long-running parity case")


def have_reference() -> bool:
    return (REF_SRC / "parabgk" / "__init__.py").exists()


@pytest.fixture(scope="session")
def ref():
    """The unmodified reference package, when this container has it."""
    if not have_reference():
        pytest.skip("reference package not present (GPU box): golden vectors cover this")
    if str(REF_SRC) not in sys.path:
        sys.path.insert(0, str(REF_SRC))
    import parabgk
    return parabgk
