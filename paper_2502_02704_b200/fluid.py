"""Coarse propagator G: first-order Rusanov Euler solver with a force source,
or (extension) the drift-diffusion solver of the diffusive scaling.

``propagate_fluid`` runs on the GPU (``pbgk_fluid_propagate``: one CTA holds the
window's conserved state in shared memory and performs every step, CFL max
included, in the reference's operation order — bitwise the numpy result of
ref/fluid.py:91-125 on the same input).  The flux helpers ``euler_flux``,
``rusanov_flux`` and ``stable_dt_fluid`` are the reference's small pointwise
API (ref/fluid.py:45-75), kept as host functions of tiny arrays.

``FluidParams(model="drift_diffusion")`` selects the EXTENSION G for the
diffusive scaling alpha = 1 (BASELINE.json config 3; the reference has none,
SPEC:8): PAPER eq. (DDbis) ``d_t rho = D d_x(d_x rho - E rho)`` with u = 0,
theta = 1, discretised by the explicit central scheme PAPER:351 names
(``fluid.cu`` ``g_advance_dd``; checker: ``oracle/bgk.py`` ``dd_propagate``).
``D`` defaults to m2 / tau = the v_x second moment of the discrete unit
Maxwellian (tau = 1).
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
           "fluid_batch", "drift_diffusion_m2", "stable_dt_drift_diffusion"]

G_MODELS = ("euler", "drift_diffusion")


@dataclass
class FluidParams:
    force: Optional[np.ndarray] = None  # per-cell E_i; None = no field
    cfl: float = 0.9
    model: str = "euler"                # "drift_diffusion": extension G (alpha = 1)
    diffusivity: Optional[float] = None  # drift-diffusion D; None = m2 of the grid

    def __post_init__(self):
        if self.model not in G_MODELS:
            raise ConfigurationError("unknown coarse model %r (expected one of %s)"
                                     % (self.model, ", ".join(G_MODELS)))
        if self.diffusivity is not None and not self.diffusivity > 0.0:
            raise ConfigurationError("need diffusivity > 0, got %r" % (self.diffusivity,))


def drift_diffusion_m2(v_max: float, n_vx: int) -> float:
    """m2 of PAPER eq. (DDbis): sum c^2 w / sum w, w = exp(-c^2/2) on the v_x centres."""
    from .grid import _centres
    c = _centres(v_max, n_vx)
    w = np.exp(-(c * c) * 0.5)
    return float(np.sum(c * c * w) / np.sum(w))


def _diffusivity(ctx, params: FluidParams) -> float:
    if params.diffusivity is not None:
        return float(params.diffusivity)
    return drift_diffusion_m2(ctx.v_max, ctx.shape[1])


def select_model(ctx, params: FluidParams) -> None:
    """Point the context's G (pbgk_fluid_model) at params.model."""
    if params.model == "euler":
        rt._lib.check(ctx.lib.pbgk_fluid_model(ctx.h, 0, 1.0), "pbgk_fluid_model")
    else:
        rt._lib.check(ctx.lib.pbgk_fluid_model(ctx.h, 1, _diffusivity(ctx, params)),
                      "pbgk_fluid_model")


def stable_dt_drift_diffusion(grid, params: FluidParams) -> float:
    """cfl dx^2 / (D (2 + dx e_max)): the explicit central scheme's step bound."""
    dx = grid.space.dx
    D = params.diffusivity if params.diffusivity is not None else \
        drift_diffusion_m2(grid.velocity.v_max, grid.velocity.n_v[0])
    e = 0.0 if params.force is None else float(np.max(np.abs(params.force)))
    return params.cfl * dx * dx / (D * (2.0 + dx * e))


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
    select_model(ctx, params)
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
