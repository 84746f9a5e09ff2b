"""Device plumbing between the reference-shaped Python API and libpbgk.so.

* ``Ctx``: one ``pbgk_ctx`` (grid constants, tiling, device workspace) per
  (grid, boundary, device); cached.
* moment packing: a ``MomentField`` travels as a ``(5, nx)`` fp64 tensor
  (rho, u_x, u_y, u_z, theta) — the layout of include/pbgk.h.
* error keys from the C ABI are turned back into the reference's exceptions
  with the reference's context fields (``step``, ``slice_index``).

torch is used for device memory and streams only; every numeric operation on
the path runs in the kernels of libpbgk.so.
"""

from __future__ import annotations

import contextlib
import ctypes
import threading

import numpy as np
import torch

from . import _lib
from .errors import BlowUpError, CorrectionOvershootError, DegenerateStateError
from .grid import bc_code

# fine steps per pass of the multi-step path (the C default, pbgk_set_fusion:
# -1 = the per-shape choice)
DEFAULT_FUSION = -1

KIND_PROJECT, KIND_LIFT, KIND_NONFINITE, KIND_UNPHYSICAL, KIND_OVERSHOOT, KIND_SYNC, KIND_NONFINITE_MULTI = range(7)

_lock = threading.Lock()
_ctx_cache: dict = {}


def require_cuda() -> None:
    if not torch.cuda.is_available():
        raise RuntimeError("no CUDA device visible: this package runs its solver on the GPU "
                           "only (there is no CPU fallback)")


def current_device() -> torch.device:
    require_cuda()
    return torch.device("cuda", torch.cuda.current_device())


def stream_handle(device: torch.device | None = None) -> ctypes.c_void_p:
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def ptr(t: torch.Tensor | None) -> ctypes.c_void_p:
    return ctypes.c_void_p(0 if t is None else t.data_ptr())


class Ctx:
    """A libpbgk context bound to one grid, one x boundary and one device."""

    def __init__(self, shape, x_min, x_max, v_max, bc: int, device: torch.device):
        self.lib = _lib.load()
        self.shape = tuple(int(n) for n in shape)
        self.device = device
        self.bc = int(bc)
        self.periodic = self.bc == 1
        self.v_max = float(v_max)
        nx, nvx, nvy, nvz = self.shape
        self.dx = (x_max - x_min) / nx
        self.dv = tuple(2.0 * v_max / n for n in (nvx, nvy, nvz))
        desc = _lib.GridDesc(nx, nvx, nvy, nvz, float(x_min), float(x_max), float(v_max),
                             self.bc, device.index)
        h = ctypes.c_void_p()
        _lib.check(self.lib.pbgk_ctx_create(ctypes.byref(desc), ctypes.byref(h)),
                   "pbgk_ctx_create")
        self.h = h
        # f-sized scratch buffers reused across calls (allocated lazily)
        self._f_tmp = [None, None]

    def set_quadrature(self, q: int) -> None:
        _lib.check(self.lib.pbgk_ctx_set_quadrature(self.h, int(q)), "pbgk_ctx_set_quadrature")
        nv = self.shape[1:]
        self.dv = tuple(2.0 * self.v_max / ((n - 1) if q else n) for n in nv)
        self.quadrature = "trapezoid" if q else "midpoint"

    def set_fusion(self, levels: int) -> None:
        """Fine steps per pass over f on the multi-step path (include/pbgk.h
        pbgk_set_fusion; 0 = always the one-step path)."""
        _lib.check(self.lib.pbgk_set_fusion(self.h, int(levels)), "pbgk_set_fusion")
        self.fusion = int(levels)

    @contextlib.contextmanager
    def fusion_levels(self, levels: int):
        """Temporarily run this context with `levels` steps per pass."""
        old = getattr(self, "fusion", None)
        self.set_fusion(levels)
        try:
            yield self
        finally:
            if old is None:
                self.lib.pbgk_set_fusion(self.h, DEFAULT_FUSION)
                self.fusion = DEFAULT_FUSION
            else:
                self.set_fusion(old)

    def set_msweep(self, on: bool, levels: int = 0) -> None:
        """Pass kernel of the multi-step path (include/pbgk.h pbgk_set_msweep):
        the round-2 msweep kernel (default) or the round-1 fsweep kernel."""
        _lib.check(self.lib.pbgk_set_msweep(self.h, int(bool(on)), int(levels)), "pbgk_set_msweep")
        self.msweep = (bool(on), int(levels))

    @contextlib.contextmanager
    def msweep_mode(self, on: bool, levels: int = 0):
        """Temporarily select the multi-step pass kernel (tests / A-B)."""
        old = getattr(self, "msweep", (True, 0))
        self.set_msweep(on, levels)
        try:
            yield self
        finally:
            self.set_msweep(*old)

    def msweep_levels(self) -> int:
        return int(self.lib.pbgk_msweep_levels(self.h))

    def set_esweep(self, on: bool) -> None:
        """Field-term pass kernel of the multi-step path (include/pbgk.h
        pbgk_set_esweep): several steps per pass (default) or one."""
        _lib.check(self.lib.pbgk_set_esweep(self.h, int(bool(on))), "pbgk_set_esweep")
        self.esweep = bool(on)

    @contextlib.contextmanager
    def esweep_mode(self, on: bool):
        """Temporarily select the field-term pass kernel (tests / A-B)."""
        old = getattr(self, "esweep", True)
        self.set_esweep(on)
        try:
            yield self
        finally:
            self.set_esweep(old)

    def esweep_levels(self) -> int:
        return int(self.lib.pbgk_esweep_levels(self.h))

    def set_batch_bytes(self, nbytes: float) -> None:
        """Table budget of the multi-step path (include/pbgk.h pbgk_set_batch_bytes)."""
        _lib.check(self.lib.pbgk_set_batch_bytes(self.h, float(nbytes)), "pbgk_set_batch_bytes")

    def describe(self) -> str:
        buf = ctypes.create_string_buffer(1024)
        _lib.check(self.lib.pbgk_ctx_describe(self.h, buf, 1024), "pbgk_ctx_describe")
        return buf.value.decode()

    def __del__(self):
        try:
            if getattr(self, "h", None):
                self.lib.pbgk_ctx_destroy(self.h)
        except Exception:
            pass

    @property
    def nx(self):
        return self.shape[0]

    def empty_f(self) -> torch.Tensor:
        return torch.empty(self.shape, dtype=torch.float64, device=self.device)

    def f_scratch(self, k: int = 0) -> torch.Tensor:
        if self._f_tmp[k] is None:
            self._f_tmp[k] = self.empty_f()
        return self._f_tmp[k]

    def empty_moments(self, n: int | None = None) -> torch.Tensor:
        shape = (5, self.nx) if n is None else (n, 5, self.nx)
        return torch.empty(shape, dtype=torch.float64, device=self.device)


def ctx_for(grid, bc, device: torch.device | None = None) -> Ctx:
    """Cached context for a (phase grid, boundary, device) triple."""
    device = device or current_device()
    sp, vel = grid.space, grid.velocity
    nv = tuple(int(n) for n in vel.n_v)
    quad = getattr(vel, "quadrature", "midpoint")
    key = (float(sp.x_min), float(sp.x_max), int(sp.n_x), float(vel.v_max), nv,
           bc_code(bc), device.index, quad)
    with _lock:
        c = _ctx_cache.get(key)
        if c is None:
            c = Ctx((sp.n_x,) + nv, sp.x_min, sp.x_max, vel.v_max, bc_code(bc), device)
            if quad == "trapezoid":
                c.set_quadrature(1)
            _ctx_cache[key] = c
        return c


def release_contexts(device: torch.device | None = None) -> int:
    """Destroy the cached contexts (all, or those of one device): their device
    workspace -- the multi-step path's per-step tables, partial records and
    the f-sized scratch buffers (8.6 GB at config 4) -- goes back to the
    allocator.  Returns how many were released; later calls create new ones."""
    with _lock:
        keys = [k for k, c in _ctx_cache.items() if device is None or c.device == device]
        for k in keys:
            c = _ctx_cache.pop(k)
            c._f_tmp = [None, None]
            try:
                torch.cuda.synchronize(c.device)
                c.lib.pbgk_ctx_destroy(c.h)
            finally:
                c.h = None
    if keys:
        torch.cuda.empty_cache()
    return len(keys)


# ---------------------------------------------------------------------------
# moments <-> (5, nx) device tensors
# ---------------------------------------------------------------------------

def pack_moments_np(rho, u, theta) -> np.ndarray:
    nx = np.shape(rho)[0]
    out = np.empty((5, nx))
    out[0] = rho
    out[1:4] = np.asarray(u, dtype=float).T
    out[4] = theta
    return out


def to_device_moments(U, device: torch.device) -> torch.Tensor:
    return torch.from_numpy(pack_moments_np(U.rho, U.u, U.theta)).to(device)


def unpack_moments_np(m: np.ndarray):
    return m[0].copy(), np.ascontiguousarray(m[1:4].T), m[4].copy()


def to_device_field(force, device: torch.device, nx: int):
    if force is None:
        return None, 0.0
    E = np.array(np.broadcast_to(np.asarray(force, dtype=float), (nx,)), dtype=float)
    e_max = float(np.max(np.abs(force)))
    return torch.from_numpy(E).to(device), e_max


# ---------------------------------------------------------------------------
# solver status keys -> reference exceptions
# ---------------------------------------------------------------------------

def decode(code: int):
    """(unit, step, kind) of a status key (include/pbgk.h)."""
    return code >> 40, (code >> 8) & 0xFFFFFFFF, code & 0xFF


def raise_kinetic(code: int) -> None:
    """Kinetic-path status: same exception and step as the reference raises."""
    if code < 0:
        return
    _, step, kind = decode(code)
    if kind == KIND_PROJECT:
        raise DegenerateStateError("nonpositive density in projection")
    if kind == KIND_LIFT:
        raise DegenerateStateError("lift requires rho > 0 and theta > 0 in every cell")
    if kind == KIND_NONFINITE:
        raise BlowUpError("kinetic propagation lost finiteness at step %d" % step, step=step)
    if kind == KIND_SYNC:
        raise RuntimeError("internal: a multi-step pass timed out waiting for the concurrent "
                           "recursion (step %d)" % step)
    raise RuntimeError("unexpected kinetic status key %#x" % code)


def raise_fluid(code: int) -> None:
    """Coarse-path status (batched G or the correction sweep)."""
    if code < 0:
        return
    unit, step, kind = decode(code)
    if kind == KIND_OVERSHOOT:
        raise CorrectionOvershootError(
            "correction left the physical regime in window %d" % unit, slice_index=unit)
    if kind == KIND_LIFT:
        raise DegenerateStateError("nonpositive density or internal energy in conserved state")
    if kind == KIND_NONFINITE:
        raise BlowUpError("fluid propagation lost finiteness at step %d" % step, step=step)
    if kind == KIND_UNPHYSICAL:
        raise BlowUpError("fluid propagation left the physical regime at step %d" % step,
                          step=step)
    raise RuntimeError("unexpected fluid status key %#x" % code)
