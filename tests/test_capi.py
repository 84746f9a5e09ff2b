"""The C-ABI library: built, loadable without a GPU, exports include/pbgk.h.

No compute calls here (this suite runs on CPU-only hosts).
"""

import ctypes
import re
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "pbgk.h"


def header_functions():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(pbgk_\w+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    from paper_2502_02704_b200 import _build, _lib
    _build.build()
    return _lib.load()


def test_header_declares_the_documented_entry_points():
    names = header_functions()
    for must in ("pbgk_ctx_create", "pbgk_lift", "pbgk_project", "pbgk_transport", "pbgk_relax",
                 "pbgk_propagate", "pbgk_fluid_propagate", "pbgk_parareal_correct"):
        assert must in names


def test_library_exports_every_declared_symbol(lib):
    from paper_2502_02704_b200 import _lib
    out = subprocess.run(["nm", "-D", "--defined-only", str(_lib.LIB_PATH)], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\bT (pbgk_\w+)", out))
    missing = [n for n in header_functions() if n not in exported]
    assert not missing, missing
    for n in header_functions():
        assert hasattr(lib, n)


def test_python_prototypes_cover_the_header():
    from paper_2502_02704_b200 import _lib
    assert set(header_functions()) == set(_lib.PROTOTYPES)


def test_calls_that_need_no_device(lib):
    assert lib.pbgk_version() == 1
    assert lib.pbgk_launch_count() >= 0
    # a null context is rejected with a message, never dereferenced
    assert lib.pbgk_profile_enable(None, 1) != 0
    assert b"null" in lib.pbgk_last_error()


def test_sm100a_code_in_library():
    from paper_2502_02704_b200 import _lib
    out = subprocess.run(["cuobjdump", "--list-elf", str(_lib.LIB_PATH)], capture_output=True,
                         text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout
    sass = subprocess.run(["cuobjdump", "-sass", str(_lib.LIB_PATH)], capture_output=True,
                          text=True).stdout
    # TMA tensor loads and 1-D bulk copies in the sweep kernel (B200_PROFILING.md)
    assert "UTMALDG" in sass
    assert "UBLKCP" in sass
