"""Fine propagator F on the GPU: upwind transport + implicit BGK relaxation.

Same API as ref/kinetic.py:42-161.  The step loop of ``propagate_kinetic`` —
``dt = min(cap, dt_max, remaining)`` while ``remaining > 1e-12 span``
(ref/kinetic.py:146-160) — is evaluated here in Python floats, exactly as the
reference does, and the whole schedule is handed to ``pbgk_propagate``: one
fused sweep kernel per fine step (one read + one write of f) plus one tiny
per-cell finalize kernel, with f resident on the device throughout.  Errors
come back as the reference's exceptions with the reference's step index.

A collision frequency ``tau`` that is ``constant_tau`` / ``ConstantTau`` (the
reference's defaults, also when imported from the reference package) is
evaluated on the device.  Any other callable is honoured through a slower
step-by-step path that evaluates ``tau(rho, theta)`` on the host each step.

``KineticParams(alpha=1)`` is the diffusive scaling of PAPER eq. (1) (an
EXTENSION; the reference implements alpha = 0 only): transport at rate
1/eps and relaxation at 1/eps^2.  A physical step d is the reference's
alpha = 0 step with the scaled step d/eps (transport d/(eps dx),
lambda = (d/eps) tau/eps), and the CFL cap is eps times the alpha = 0 cap;
checker: ``oracle/bgk.py`` ``fine_propagate(alpha=1)``.

``KineticParams(scheme="muscl")`` replaces the first-order upwind x flux by a
MUSCL reconstruction with the minmod limiter (EXTENSION: BASELINE north_star
"upwind/MUSCL", the paper's flux limiters; checker ``oracle/bgk.py``
``transport_muscl``).  It has no v_x field term (E must be None).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Callable, Optional

import numpy as np
import torch

from . import runtime as rt
from .errors import ConfigurationError
from .lifting import Distribution, as_device_f

__all__ = ["constant_tau", "ConstantTau", "KineticParams", "stable_dt_kinetic",
           "transport_update", "bgk_relax", "propagate_kinetic", "fine_schedule",
           "propagate_window", "propagate_windows"]

SPAN_GUARD = 1e-12  # ref/kinetic.py:39


def constant_tau(rho, theta):
    """Unit collision frequency (ref/kinetic.py:42-44)."""
    return 1.0


@dataclass(frozen=True)
class ConstantTau:
    """Picklable constant collision frequency (ref/kinetic.py:47-54)."""

    value: float

    def __call__(self, rho, theta):
        return self.value


@dataclass
class KineticParams:
    """epsilon, tau(rho, theta), per-cell field E (or None), Courant factor."""

    epsilon: float
    tau: Callable = constant_tau
    force: Optional[np.ndarray] = None
    cfl: float = 0.5
    alpha: int = 0  # 0 hydrodynamic (reference); 1 diffusive scaling (extension)
    scheme: str = "upwind"  # x flux: "upwind" (reference) or "muscl" (extension)

    def __post_init__(self):
        if self.alpha not in (0, 1):
            raise ConfigurationError("alpha must be 0 or 1, got %r" % (self.alpha,))
        if self.scheme not in ("upwind", "muscl"):
            raise ConfigurationError("unknown x scheme %r (upwind | muscl)" % (self.scheme,))
        if self.scheme == "muscl" and self.force is not None and np.max(np.abs(self.force)) > 0:
            raise ConfigurationError("the MUSCL x scheme has no v_x field term; use scheme='upwind'")


def _check_grid(grid, params) -> None:
    """Combinations the extensions do not define."""
    if getattr(grid.velocity, "quadrature", "midpoint") == "trapezoid" and \
            params.force is not None and np.max(np.abs(params.force)) > 0:
        raise ConfigurationError("the v_x field term is defined on midpoint velocity cells only "
                                 "(trapezoidal quadrature needs force=None)")


def _scheme(ctx, params) -> None:
    """Point the context's sweeps at params.scheme (pbgk_set_x_scheme)."""
    code = 1 if getattr(params, "scheme", "upwind") == "muscl" else 0
    rt._lib.check(ctx.lib.pbgk_set_x_scheme(ctx.h, code), "pbgk_set_x_scheme")


def _kdt(dt: float, params) -> float:
    """The step the alpha = 0 kernels take for a physical step dt."""
    return dt / params.epsilon if getattr(params, "alpha", 0) == 1 else dt


def tau_constant(tau) -> Optional[float]:
    """The constant value of a reference-style constant tau, else None."""
    if tau is constant_tau:
        return 1.0
    if isinstance(tau, ConstantTau):
        return float(tau.value)
    name = getattr(tau, "__name__", None) or type(tau).__name__
    mod = getattr(tau, "__module__", "") or type(tau).__module__
    if mod.endswith("kinetic") and name == "constant_tau":
        return 1.0
    if mod.endswith("kinetic") and type(tau).__name__ == "ConstantTau":
        return float(tau.value)
    return None


def _e_max(params) -> float:
    return 0.0 if params.force is None else float(np.max(np.abs(params.force)))


def stable_dt_kinetic(grid, params) -> float:
    """cfl / (v_max/dx + E_max/dv_x) with the cube bound v_max (ref/kinetic.py:77-83)."""
    rate = grid.velocity.v_max / grid.space.dx
    e = _e_max(params)
    if e > 0.0:
        rate += e / grid.velocity.dv[0]
    cap = params.cfl / rate
    return cap * params.epsilon if getattr(params, "alpha", 0) == 1 else cap


def fine_schedule(span: float, cap: float) -> list:
    """The reference's dt sequence for one propagation (ref/kinetic.py:150-160)."""
    out = []
    done = 0.0
    while span - done > SPAN_GUARD * span:
        d = min(cap, span - done)
        out.append(d)
        done += d
    return out


def transport_update(f, dt: float, grid, params, bc) -> Distribution:
    """One explicit transport step on the GPU (ref/kinetic.py:86-124)."""
    _check_grid(grid, params)
    ctx = rt.ctx_for(grid, bc)
    _scheme(ctx, params)
    fd = as_device_f(f, ctx)
    E, e_max = rt.to_device_field(params.force, ctx.device, ctx.nx)
    out = ctx.empty_f()
    rt._lib.check(ctx.lib.pbgk_transport(ctx.h, rt.ptr(fd), rt.ptr(out), float(_kdt(dt, params)),
                                         rt.ptr(E), e_max, rt.stream_handle(ctx.device)),
                  "pbgk_transport")
    return Distribution(out)


def _relax_dev(ctx, fd, dt, params, out, tau_cells=None):
    tc = tau_constant(params.tau)
    if tc is None and tau_cells is None:
        # general callable: tau needs the moments of f first (one projection)
        from .moments import project_device, MomentField
        U = MomentField.from_packed(project_device(fd, ctx))
        tau = np.broadcast_to(np.asarray(params.tau(U.rho, U.theta), dtype=float), U.rho.shape)
        tau_cells = torch.from_numpy(np.array(tau, dtype=float)).to(ctx.device)
    code = ctypes.c_longlong(-1)
    rt._lib.check(ctx.lib.pbgk_relax(ctx.h, rt.ptr(fd), rt.ptr(out), float(dt),
                                     float(params.epsilon), 1.0 if tc is None else tc,
                                     rt.ptr(tau_cells), rt.stream_handle(ctx.device),
                                     ctypes.byref(code)), "pbgk_relax")
    rt.raise_kinetic(code.value)
    return out


def bgk_relax(f, dt: float, grid, params, bc=None) -> Distribution:
    """Implicit relaxation toward the Maxwellian of f's moments (ref/kinetic.py:127-134)."""
    ctx = rt.ctx_for(grid, bc if bc is not None else "absorbing")
    fd = as_device_f(f, ctx)
    return Distribution(_relax_dev(ctx, fd, _kdt(dt, params), params, ctx.empty_f()))


def _run_schedule(ctx, f0, mom0, dts, params, out, want_f=True, mom_out=None):
    """pbgk_propagate over a fixed schedule; returns the status key."""
    tc = tau_constant(params.tau)
    _scheme(ctx, params)
    E, e_max = rt.to_device_field(params.force, ctx.device, ctx.nx)
    arr = (ctypes.c_double * max(len(dts), 1))(*[_kdt(d, params) for d in dts])
    code = ctypes.c_longlong(-1)
    rt._lib.check(ctx.lib.pbgk_propagate(
        ctx.h, rt.ptr(f0), rt.ptr(mom0), rt.ptr(out), rt.ptr(ctx.f_scratch(0)),
        1 if want_f else 0, rt.ptr(mom_out), len(dts), arr, float(params.epsilon), tc,
        rt.ptr(E), e_max, rt.stream_handle(ctx.device), ctypes.byref(code)), "pbgk_propagate")
    return code.value


def _step_by_step(ctx, fd, dts, params):
    """Slow path for a non-constant tau callable: transport, host tau, relax."""
    _scheme(ctx, params)
    E, e_max = rt.to_device_field(params.force, ctx.device, ctx.nx)
    cur = fd
    for s, dt in enumerate(dts, start=1):
        dt = _kdt(dt, params)
        mid = ctx.empty_f()
        rt._lib.check(ctx.lib.pbgk_transport(ctx.h, rt.ptr(cur), rt.ptr(mid), float(dt), rt.ptr(E),
                                             e_max, rt.stream_handle(ctx.device)), "pbgk_transport")
        cur = _relax_dev(ctx, mid, dt, params, ctx.empty_f())
        code = ctypes.c_longlong(-1)
        rt._lib.check(ctx.lib.pbgk_check_finite(ctx.h, rt.ptr(cur), s, rt.stream_handle(ctx.device),
                                                ctypes.byref(code)), "pbgk_check_finite")
        rt.raise_kinetic(code.value)
    return cur


def propagate_kinetic(f0, t0: float, t1: float, grid, params, bc, dt_max=None) -> Distribution:
    """Advance f0 from t0 to t1 (ref/kinetic.py:137-161), on the GPU."""
    if t1 < t0:
        raise ConfigurationError("need t1 >= t0, got [%r, %r]" % (t0, t1))
    _check_grid(grid, params)
    span = t1 - t0
    if span == 0.0:
        return f0
    cap = stable_dt_kinetic(grid, params)
    if dt_max is not None:
        cap = min(cap, dt_max)
    dts = fine_schedule(span, cap)
    ctx = rt.ctx_for(grid, bc)
    fd = as_device_f(f0, ctx)
    if tau_constant(params.tau) is None:
        return Distribution(_step_by_step(ctx, fd, dts, params))
    out = ctx.empty_f()
    code = _run_schedule(ctx, fd, None, dts, params, out)
    rt.raise_kinetic(code)
    return Distribution(out)


def propagate_window(ctx, mom0: torch.Tensor, t0: float, t1: float, grid, params, dt_max,
                     mom_out: torch.Tensor) -> int:
    """P(F(L(U))) of one window, moments in and out on the device.

    Neither L(U) nor f_S is materialised: the first sweep synthesises the lift
    from the moment tables and the last one only projects.  Returns the
    status key (-1 clean) without raising, so callers can order failures.
    """
    _check_grid(grid, params)
    span = t1 - t0
    cap = stable_dt_kinetic(grid, params)
    if dt_max is not None:
        cap = min(cap, dt_max)
    dts = fine_schedule(span, cap) if span > 0.0 else []
    if not dts:
        mom_out.copy_(mom0)
        return -1
    if tau_constant(params.tau) is None:
        from .lifting import lift
        from .moments import MomentField, project_device
        f = lift(MomentField.from_packed(mom0), grid, bc=("absorbing", "periodic", "outflow")[ctx.bc])
        f = _step_by_step(ctx, f.device_tensor(ctx.device), dts, params)
        mom_out.copy_(project_device(f, ctx))
        return -1
    return _run_schedule(ctx, None, mom0, dts, params, ctx.f_scratch(1), want_f=False,
                         mom_out=mom_out)


def propagate_windows(ctx, mom_in: torch.Tensor, spans, grid, params, dt_max,
                      mom_out: torch.Tensor) -> list:
    """P(F(L(U_w))) for every window w of a batch in one library call
    (``pbgk_propagate_windows``: one host synchronisation for the batch).

    mom_in / mom_out: (nwin, 5, nx) device tensors; spans[w] = t1 - t0 of
    window w.  Returns the status keys (-1 clean).  Constant tau only; the
    schedule of each window is that of ``propagate_window``."""
    _check_grid(grid, params)
    tc = tau_constant(params.tau)
    if tc is None:
        raise ConfigurationError("propagate_windows needs a constant tau")
    cap = stable_dt_kinetic(grid, params)
    if dt_max is not None:
        cap = min(cap, dt_max)
    nwin = len(spans)
    # the batch's schedules are the same in every parareal iteration: keep the
    # marshalled arrays of the last few (spans, cap, scaling) on the context
    key = (tuple(float(x) for x in spans), float(cap), float(params.epsilon), getattr(params, "alpha", 0))
    cache = ctx.__dict__.setdefault("_schedule_cache", {})
    hit = cache.get(key)
    if hit is None:
        counts, dts, per_span = [], [], {}
        for span in key[0]:
            d = per_span.get(span)
            if d is None:
                d = [_kdt(x, params) for x in fine_schedule(span, cap)] if span > 0.0 else []
                per_span[span] = d
            counts.append(len(d))
            dts += d
        hit = ((ctypes.c_int * max(nwin, 1))(*counts), (ctypes.c_double * max(len(dts), 1))(*dts))
        if len(cache) >= 8:
            cache.clear()
        cache[key] = hit
    c_counts, c_dts = hit
    _scheme(ctx, params)
    E, e_max = rt.to_device_field(params.force, ctx.device, ctx.nx)
    codes = (ctypes.c_longlong * max(nwin, 1))()
    rt._lib.check(ctx.lib.pbgk_propagate_windows(
        ctx.h, nwin, rt.ptr(mom_in), rt.ptr(mom_out), rt.ptr(ctx.f_scratch(0)),
        rt.ptr(ctx.f_scratch(1)), c_counts, c_dts, float(params.epsilon), tc, rt.ptr(E), e_max,
        rt.stream_handle(ctx.device), codes), "pbgk_propagate_windows")
    return [codes[w] for w in range(nwin)]

