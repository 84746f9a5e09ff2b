"""Coarse propagator G: first-order Rusanov Euler solver with a force source.

``propagate_fluid`` runs on the GPU (``pbgk_fluid_propagate``: one CTA holds the
window's conserved state in shared memory and performs every step, CFL max
included, in the reference's operation order — bitwise the numpy result of
ref/fluid.py:91-125 on the same input).  The flux helpers ``euler_flux``,
``rusanov_flux`` and ``stable_dt_fluid`` are the reference's small pointwise
API (ref/fluid.py:45-75), kept as host functions of tiny arrays.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Optional

import numpy as np
import torch

from . import runtime as rt
from .errors import ConfigurationError
from .moments import ConservedField, MomentField

__all__ = ["FluidParams", "euler_flux", "rusanov_flux", "stable_dt_fluid", "propagate_fluid",
           "fluid_batch"]


@dataclass
class FluidParams:
    force: Optional[np.ndarray] = None  # per-cell E_i; None = no field
    cfl: float = 0.9


def _p(v):
    ke = 0.5 * (v[..., 1] ** 2 + v[..., 2] ** 2 + v[..., 3] ** 2) / v[..., 0]
    return (v[..., 4] - ke) / 1.5


def euler_flux(v) -> np.ndarray:
    """x flux of packed conserved states (..., 5) (ref/fluid.py:45-56)."""
    v = np.asarray(v, dtype=float)
    ux = v[..., 1] / v[..., 0]
    p = _p(v)
    return np.stack([v[..., 1], v[..., 1] * ux + p, v[..., 2] * ux, v[..., 3] * ux,
                     ux * (v[..., 4] + p)], axis=-1)


def rusanov_flux(vl, vr) -> np.ndarray:
    """Central flux with local max-speed dissipation (ref/fluid.py:59-66)."""
    vl = np.asarray(vl, dtype=float)
    vr = np.asarray(vr, dtype=float)
    s = np.maximum(np.abs(vl[..., 1] / vl[..., 0]) + np.sqrt(_p(vl) / vl[..., 0]),
                   np.abs(vr[..., 1] / vr[..., 0]) + np.sqrt(_p(vr) / vr[..., 0]))
    return 0.5 * (euler_flux(vl) + euler_flux(vr)) - 0.5 * s[..., None] * (vr - vl)


def stable_dt_fluid(V: ConservedField, grid, params: FluidParams) -> float:
    """cfl dx / max(|u_x| + sqrt(theta)) (ref/fluid.py:69-75)."""
    v = V.to_array()
    rate = float(np.max(np.abs(V.mom[:, 0] / V.rho) + np.sqrt(_p(v) / V.rho)))
    return params.cfl * grid.space.dx / rate


def fluid_batch(ctx, mom_in: torch.Tensor, mom_out: torch.Tensor, t0s, t1s, params: FluidParams,
                dt_max=None, minuend: torch.Tensor | None = None, force_dev=None) -> int:
    """G over nwin independent windows in one launch; returns the status key.

    mom_in / mom_out / minuend: (nwin, 5, nx) device tensors; with ``minuend``
    the output is ``minuend - G(mom_in)`` (the parareal jump).
    """
    nwin = mom_in.shape[0]
    if force_dev is None and params.force is not None:
        force_dev, _ = rt.to_device_field(params.force, ctx.device, ctx.nx)
    a0 = (ctypes.c_double * nwin)(*map(float, t0s))
    a1 = (ctypes.c_double * nwin)(*map(float, t1s))
    code = ctypes.c_longlong(-1)
    rt._lib.check(ctx.lib.pbgk_fluid_propagate(
        ctx.h, nwin, rt.ptr(mom_in), rt.ptr(mom_out), rt.ptr(minuend), a0, a1,
        -1.0 if dt_max is None else float(dt_max), float(params.cfl), rt.ptr(force_dev),
        rt.stream_handle(ctx.device), ctypes.byref(code)), "pbgk_fluid_propagate")
    return code.value


def propagate_fluid(U0: MomentField, t0: float, t1: float, grid, params: FluidParams, bc,
                    dt_max=None) -> MomentField:
    """Advance primitive moments from t0 to t1 on the GPU (ref/fluid.py:91-125)."""
    if t1 < t0:
        raise ConfigurationError("need t1 >= t0, got [%r, %r]" % (t0, t1))
    if t1 - t0 == 0.0:
        return U0
    ctx = rt.ctx_for(grid, bc)
    m = rt.to_device_moments(U0, ctx.device).unsqueeze(0)
    out = torch.empty_like(m)
    code = fluid_batch(ctx, m, out, [t0], [t1], params, dt_max)
    rt.raise_fluid(code)
    return MomentField.from_packed(out[0])
