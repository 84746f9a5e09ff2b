"""ctypes binding of libpbgk.so, the C ABI declared in include/pbgk.h.

There is no CPU fallback: if the shared library is missing or no CUDA device
is visible, every solver entry point raises.
"""

from __future__ import annotations

import ctypes
from ctypes import POINTER, c_double, c_int, c_int32, c_longlong, c_size_t, c_void_p, c_char_p
from pathlib import Path

import os

LIB_PATH = Path(os.environ.get("PBGK_LIB") or Path(__file__).resolve().parent / "lib" / "libpbgk.so")


class GridDesc(ctypes.Structure):
    """struct pbgk_grid_desc (include/pbgk.h)."""

    _fields_ = [("nx", c_int32), ("nvx", c_int32), ("nvy", c_int32), ("nvz", c_int32),
                ("x_min", c_double), ("x_max", c_double), ("v_max", c_double),
                ("bc", c_int32), ("device", c_int32)]


_P = c_void_p
_D = c_double
_I = c_int
_CODE = POINTER(c_longlong)

# symbol -> (restype, argtypes); kept in the order of include/pbgk.h
PROTOTYPES = {
    "pbgk_version": (c_int, []),
    "pbgk_last_error": (c_char_p, []),
    "pbgk_ctx_create": (c_int, [POINTER(GridDesc), POINTER(c_void_p)]),
    "pbgk_ctx_destroy": (None, [_P]),
    "pbgk_ctx_workspace_bytes": (c_size_t, [_P]),
    "pbgk_lift": (c_int, [_P, _P, _I, _P, _P, _CODE]),
    "pbgk_project": (c_int, [_P, _P, _P, _P, _CODE]),
    "pbgk_transport": (c_int, [_P, _P, _P, _D, _P, _D, _P]),
    "pbgk_relax": (c_int, [_P, _P, _P, _D, _D, _D, _P, _P, _CODE]),
    "pbgk_propagate": (c_int, [_P, _P, _P, _P, _P, _I, _P, _I, POINTER(c_double), _D, _D, _P,
                               _D, _P, _CODE]),
    "pbgk_fluid_propagate": (c_int, [_P, _I, _P, _P, _P, POINTER(c_double), POINTER(c_double),
                                     _D, _D, _P, _P, _CODE]),
    "pbgk_check_finite": (c_int, [_P, _P, _I, _P, _CODE]),
    "pbgk_fluid_model": (c_int, [_P, _I, _D]),
    "pbgk_set_grid_reserve": (c_int, [_P, _I]),
    "pbgk_set_x_scheme": (c_int, [_P, _I]),
    "pbgk_set_fusion": (c_int, [_P, _I]),
    "pbgk_set_msweep": (c_int, [_P, _I, _I]),
    "pbgk_set_esweep": (c_int, [_P, _I]),
    "pbgk_esweep_levels": (c_int, [_P]),
    "pbgk_msweep_levels": (c_int, [_P]),
    "pbgk_set_batch_bytes": (c_int, [_P, _D]),
    "pbgk_table_len": (c_int, [_P]),
    "pbgk_propagate_windows": (c_int, [_P, _I, _P, _P, _P, _P, POINTER(c_int), POINTER(c_double),
                                       _D, _D, _P, _D, _P, POINTER(c_longlong)]),
    "pbgk_ctx_set_quadrature": (c_int, [_P, _I]),
    "pbgk_ctx_set_dx": (c_int, [_P, _D]),
    "pbgk_slab_tables": (c_int, [_P, _I, _P, _P, _P, _P]),
    "pbgk_slab_sweep": (c_int, [_P, _P, _P, _P, _D, _P, _D, _P]),
    "pbgk_slab_finalize": (c_int, [_P, _I, _I, _P, _P, _D, _D, _D, _I, _P, _P]),
    "pbgk_fluid_propagate_async": (c_int, [_P, _I, _P, _P, _P, _P, _P, _D, _D, _P, _P, _P]),
    "pbgk_parareal_correct_range": (c_int, [_P, _I, _I, _P, _P, _P, _P, _D, _D, _P, _P, _P, _P]),
    "pbgk_parareal_correct": (c_int, [_P, _I, _I, _P, _P, _P, POINTER(c_double), _D, _D, _P,
                                      _P, POINTER(c_double), _CODE]),
}



class Profile(ctypes.Structure):
    """struct pbgk_profile (include/pbgk.h)."""

    _fields_ = [("sweep_ms", c_double), ("sweep_bytes", c_double), ("sweeps", c_longlong),
                ("finalize_ms", c_double), ("finalizes", c_longlong),
                ("msweep_ms", c_double), ("msweep_bytes", c_double), ("msweeps", c_longlong),
                ("msweep_steps", c_longlong), ("marg_ms", c_double), ("margs", c_longlong)]


PROTOTYPES.update({
    "pbgk_launch_count": (c_longlong, []),
    "pbgk_ctx_describe": (c_int, [_P, ctypes.c_char_p, c_size_t]),
    "pbgk_profile_enable": (c_int, [_P, _I]),
    "pbgk_profile_read": (c_int, [_P, POINTER(Profile)]),
})

_lib = None


def load():
    """Load (once) and type the shared library; raises if it is not built."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise RuntimeError(
            "libpbgk.so is not built (%s); run `python -c 'import __graft_entry__ as g; "
            "g.build()'` — there is no CPU fallback" % LIB_PATH)
    lib = ctypes.CDLL(str(LIB_PATH))
    dev_override = bool(os.environ.get("PBGK_LIB"))  # A/B of older builds: tolerate gaps
    for name, (res, args) in PROTOTYPES.items():
        if dev_override and not hasattr(lib, name):
            continue
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(rc: int, what: str) -> None:
    if rc != 0:
        msg = load().pbgk_last_error()
        raise RuntimeError("%s failed: %s" % (what, msg.decode() if msg else "unknown"))
