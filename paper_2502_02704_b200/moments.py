"""Moment states and the projection P (GPU).

``project`` is one sweep of the fine-propagator kernel over f (marginals only)
plus the per-cell finalize kernel; it reproduces ref/moments.py:91-113 (three
marginals, folded first moment — exactly 0 for even data — and the two-pass
temperature).  ``MomentField`` / ``ConservedField`` and the primitive <->
conserved maps are small host-side value types, as in the reference
(ref/moments.py:29-77, 116-129); the GPU coarse solver performs the same maps
inside its kernel.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import runtime as rt
from .errors import DegenerateStateError

__all__ = ["MomentField", "ConservedField", "project", "primitive_to_conserved",
           "conserved_to_primitive"]


@dataclass
class MomentField:
    """Per-cell density (nx,), bulk velocity (nx, 3) and temperature (nx,)."""

    rho: np.ndarray
    u: np.ndarray
    theta: np.ndarray

    @property
    def n_x(self) -> int:
        return self.rho.shape[0]

    def copy(self) -> "MomentField":
        return MomentField(self.rho.copy(), self.u.copy(), self.theta.copy())

    def __add__(self, other: "MomentField") -> "MomentField":
        return MomentField(self.rho + other.rho, self.u + other.u, self.theta + other.theta)

    def __sub__(self, other: "MomentField") -> "MomentField":
        return MomentField(self.rho - other.rho, self.u - other.u, self.theta - other.theta)

    def sup_distance(self, other: "MomentField") -> float:
        """max over cells and components of |self - other| (ref/moments.py:48-52)."""
        return max(float(np.max(np.abs(self.rho - other.rho))),
                   float(np.max(np.abs(self.u - other.u))),
                   float(np.max(np.abs(self.theta - other.theta))))

    # device interchange -----------------------------------------------------
    def to_device(self, device):
        return rt.to_device_moments(self, device)

    @staticmethod
    def from_packed(m) -> "MomentField":
        """From a (5, nx) array/tensor (rho, u_x, u_y, u_z, theta)."""
        if hasattr(m, "detach"):
            m = m.detach().cpu().numpy()
        return MomentField(*rt.unpack_moments_np(np.asarray(m)))


@dataclass
class ConservedField:
    """Per-cell density, momentum (nx, 3) and total energy."""

    rho: np.ndarray
    mom: np.ndarray
    energy: np.ndarray

    def to_array(self) -> np.ndarray:
        v = np.empty((self.rho.shape[0], 5))
        v[:, 0], v[:, 1:4], v[:, 4] = self.rho, self.mom, self.energy
        return v

    @staticmethod
    def from_array(v: np.ndarray) -> "ConservedField":
        return ConservedField(v[:, 0].copy(), v[:, 1:4].copy(), v[:, 4].copy())


def primitive_to_conserved(U: MomentField) -> ConservedField:
    """E = rho |u|^2 / 2 + 3 rho theta / 2 (ref/moments.py:116-119)."""
    ke = 0.5 * U.rho * np.einsum("ij,ij->i", U.u, U.u)
    return ConservedField(U.rho.copy(), U.rho[:, None] * U.u, ke + 1.5 * U.rho * U.theta)


def conserved_to_primitive(V: ConservedField) -> MomentField:
    """Inverse map with the reference's degeneracy guards (ref/moments.py:122-129)."""
    if np.any(V.rho <= 0.0):
        raise DegenerateStateError("nonpositive density in conserved state")
    u = V.mom / V.rho[:, None]
    eint = V.energy - 0.5 * np.einsum("ij,ij->i", V.mom, u)
    if np.any(eint <= 0.0):
        raise DegenerateStateError("nonpositive internal energy in conserved state")
    return MomentField(V.rho.copy(), u, eint / (1.5 * V.rho))


def project(f, grid, bc=None) -> MomentField:
    """P: moments of a distribution, on the GPU (replaces ref/moments.py:91-113).

    ``bc`` is irrelevant to the quadrature; it only selects a cached context.
    """
    from .lifting import as_device_f
    import ctypes

    ctx = rt.ctx_for(grid, bc if bc is not None else "absorbing")
    fd = as_device_f(f, ctx)
    out = ctx.empty_moments()
    code = ctypes.c_longlong(-1)
    rt._lib.check(ctx.lib.pbgk_project(ctx.h, rt.ptr(fd), rt.ptr(out),
                                       rt.stream_handle(ctx.device), ctypes.byref(code)),
                  "pbgk_project")
    rt.raise_kinetic(code.value)
    return MomentField.from_packed(out)


def project_device(f_dev, ctx) -> "object":
    """Projection of a device tensor into a (5, nx) device tensor (no host copy)."""
    import ctypes

    out = ctx.empty_moments()
    code = ctypes.c_longlong(-1)
    rt._lib.check(ctx.lib.pbgk_project(ctx.h, rt.ptr(f_dev), rt.ptr(out),
                                       rt.stream_handle(ctx.device), ctypes.byref(code)),
                  "pbgk_project")
    rt.raise_kinetic(code.value)
    return out
