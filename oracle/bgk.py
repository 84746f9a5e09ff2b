"""Numpy restatement of the reference hot path (TEST INFRASTRUCTURE ONLY).

This module is the CPU checker for the CUDA path in ``paper_2502_02704_b200``.
It restates, operation for operation, the arithmetic of the reference package
``parabgk`` (``/root/reference/pkg/src/parabgk``; abbreviated ``ref/`` below)
so that on the same inputs it reproduces the reference bit for bit.  The pin is
``tests/test_oracle.py`` (reference imported where present, golden vectors in
``tests/golden/`` everywhere else).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs may
use it.  The product never imports it and has no CPU fallback.

Conventions: a distribution is an ``(nx, nvx, nvy, nvz)`` float64 C-order
array; a moment state is the triple ``(rho (nx,), u (nx, 3), theta (nx,))``.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Callable, Optional, Sequence

import numpy as np

GUARD = 1e-12  # ref/kinetic.py:39 and ref/fluid.py:30 (span guard)


class OracleError(Exception):
    """Base of the oracle's failure signals (mirrors ref/errors.py:4-29)."""


class OracleConfigError(OracleError):
    pass


class OracleDegenerate(OracleError):
    pass


class OracleBlowUp(OracleError):
    def __init__(self, msg, step=None):
        super().__init__(msg)
        self.step = step


class OracleOvershoot(OracleError):
    def __init__(self, msg, slice_index=None):
        super().__init__(msg)
        self.slice_index = slice_index


# --------------------------------------------------------------------------
# meshes (ref/grid.py:89-127)
# --------------------------------------------------------------------------

@dataclass
class Mesh:
    """Phase-space mesh: x cells plus a per-axis velocity cube."""

    x_min: float
    x_max: float
    nx: int
    v_max: float
    nv: tuple
    quadrature: str = "midpoint"

    def __post_init__(self):
        self.nv = tuple(int(n) for n in self.nv)
        # ref/grid.py:95-96
        self.dx = (self.x_max - self.x_min) / self.nx
        self.xc = self.x_min + (np.arange(self.nx) + 0.5) * self.dx
        if self.quadrature == "trapezoid":
            # ORACLE EXTENSION (BASELINE config 0's "trapezoidal quadrature"; the
            # reference has midpoint only): n nodes on
            # [-v_max, v_max] including the ends, dv = 2 v_max/(n-1), weights
            # dv * (1/2 at the two end nodes, 1 elsewhere) on every velocity sum
            if min(self.nv) < 2:
                raise OracleConfigError("trapezoidal quadrature needs >= 2 nodes per axis")
            self.dv = tuple(2.0 * self.v_max / (n - 1) for n in self.nv)
            self.vc = tuple((np.arange(n) - (n - 1) / 2.0) * (2.0 * self.v_max / (n - 1))
                            for n in self.nv)
            self.wq = tuple(np.where((np.arange(n) == 0) | (np.arange(n) == n - 1), 0.5, 1.0)
                            for n in self.nv)
        else:
            # ref/grid.py:100-103, 114-115
            self.dv = tuple(2.0 * self.v_max / n for n in self.nv)
            self.vc = tuple((np.arange(n) - (n - 1) / 2.0) * (2.0 * self.v_max / n)
                            for n in self.nv)
            self.wq = None
        # ref/grid.py:57-59
        self.dvol = self.dv[0] * self.dv[1] * self.dv[2]


def coarse_grid(t_final: float, n_g: int, n_f: int):
    """(times, dt_g, dt_f) of ref/grid.py:119-127."""
    return np.linspace(0.0, t_final, n_g + 1), t_final / n_g, t_final / n_f


# --------------------------------------------------------------------------
# moments: P (ref/moments.py:80-129)
# --------------------------------------------------------------------------

def marginals(f: np.ndarray, mesh: Optional[Mesh] = None):
    """Three per-cell velocity marginals (ref/moments.py:100).  Trapezoidal
    meshes weight the two summed axes (exact: the weights are 1/2 or 1)."""
    if mesh is None or mesh.wq is None:
        return (np.add.reduce(f, axis=(2, 3)), np.add.reduce(f, axis=(1, 3)),
                np.add.reduce(f, axis=(1, 2)))
    wx, wy, wz = mesh.wq
    return (np.add.reduce(f * (wy[:, None] * wz[None, :])[None, None], axis=(2, 3)),
            np.add.reduce(f * (wx[:, None] * wz[None, :])[None, :, None, :], axis=(1, 3)),
            np.add.reduce(f * (wx[:, None] * wy[None, :])[None, :, :, None], axis=(1, 2)))


def _mirror_weighted(m: np.ndarray, c: np.ndarray) -> np.ndarray:
    # ref/moments.py:80-88: mirrored pairs are differenced before weighting.
    n = c.size
    k = n // 2
    return np.matmul(m[:, :k] - m[:, : n - k - 1: -1], c[:k])


def moments_of(margs, mesh: Mesh):
    """(rho, u, theta) from marginals (ref/moments.py:101-113)."""
    w = mesh.dvol
    q = mesh.wq  # trapezoid: the remaining axis is weighted here
    m0 = margs[0] if q is None else margs[0] * q[0]
    rho = np.add.reduce(m0, axis=1) * w
    if np.any(rho <= 0.0):
        raise OracleDegenerate("rho <= 0 in projection at cell %d"
                               % int(np.argmax(rho <= 0.0)))
    ru = np.stack([_mirror_weighted(margs[a], mesh.vc[a] if q is None else mesh.vc[a] * q[a])
                   for a in range(3)], axis=1) * w
    u = ru / rho[:, None]
    acc = np.zeros_like(rho)
    for a in range(3):
        d = mesh.vc[a][None, :] - u[:, a, None]
        acc += np.einsum("ij,ij->i", d * d, margs[a] if q is None else margs[a] * q[a])
    theta = acc * w / (3.0 * rho)
    return rho, u, theta


def project(f: np.ndarray, mesh: Mesh):
    """P: ref/moments.py:91-113."""
    return moments_of(marginals(f, mesh), mesh)


# --------------------------------------------------------------------------
# lifting: L (ref/lifting.py:36-58)
# --------------------------------------------------------------------------

def maxwell_factors(rho, u, theta, mesh: Mesh):
    """Separable Maxwellian factors (gx*amp, gy, gz) of ref/lifting.py:44-50."""
    if np.any(rho <= 0.0) or np.any(theta <= 0.0):
        raise OracleDegenerate("lift needs rho > 0 and theta > 0")
    h = 1.0 / (2.0 * theta)
    g = []
    for a in range(3):
        d = mesh.vc[a][None, :] - u[:, a, None]
        g.append(np.exp(-(d * d) * h[:, None]))
    amp = rho / (2.0 * np.pi * theta) ** 1.5
    return g[0] * amp[:, None], g[1], g[2]


def lift(rho, u, theta, mesh: Mesh, normalize: bool = False) -> np.ndarray:
    """L: ref/lifting.py:36-58 (outer product, optional per-cell mass fix)."""
    gxa, gy, gz = maxwell_factors(rho, u, theta, mesh)
    f = gxa[:, :, None, None] * gy[:, None, :, None] * gz[:, None, None, :]
    if normalize:
        fw = f if mesh.wq is None else f * (mesh.wq[0][:, None, None] * mesh.wq[1][None, :, None]
                                             * mesh.wq[2][None, None, :])[None]
        mass = np.add.reduce(fw, axis=(1, 2, 3)) * mesh.dvol
        f *= (rho / mass)[:, None, None, None]
    return f


def maxwellian_point(rho, u, theta, v):
    """Scalar Maxwellian (ref/lifting.py:26-33)."""
    if theta <= 0.0:
        raise OracleDegenerate("theta <= 0")
    q = np.sum((np.asarray(v, float) - np.asarray(u, float)) ** 2)
    return float(rho / (2.0 * np.pi * theta) ** 1.5 * np.exp(-q / (2.0 * theta)))


# --------------------------------------------------------------------------
# fine propagator F (ref/kinetic.py:77-161)
# --------------------------------------------------------------------------

def field_bound(force) -> float:
    """max |E| (ref/kinetic.py:71-74)."""
    return 0.0 if force is None else float(np.max(np.abs(force)))


def fine_cap(mesh: Mesh, cfl: float, force=None) -> float:
    """CFL cap of ref/kinetic.py:77-83 (cube bound v_max, not the last centre)."""
    rate = mesh.v_max / mesh.dx
    e = field_bound(force)
    if e > 0.0:
        rate += e / mesh.dv[0]
    return cfl / rate


def bc_kind(bc) -> str:
    """'periodic' | 'absorbing' | 'outflow' from a bool (True = periodic) or a name."""
    if isinstance(bc, str):
        return bc
    return "periodic" if bc else "absorbing"


def transport(f: np.ndarray, dt: float, mesh: Mesh, periodic, force=None) -> np.ndarray:
    """Explicit upwind-x + Rusanov-v_x step (ref/kinetic.py:86-124).

    ``periodic``: True / False (the reference's PERIODIC / ABSORBING) or one of
    'periodic', 'absorbing', 'outflow'.  'outflow' is an ORACLE EXTENSION
    (BASELINE.json configs 0/4 ask for zero-gradient boundaries; the reference
    has only the zero-inflow ghost): ghost planes copy the edge planes, i.e.
    ref/kinetic.py:106-108 with ``ghosted[0] = vals[0]``, ``ghosted[-1] = vals[-1]``.
    """
    kind = bc_kind(periodic)
    nx = f.shape[0]
    c = mesh.vc[0]
    cpos = np.maximum(c, 0.0)[None, :, None, None]
    cneg = np.minimum(c, 0.0)[None, :, None, None]
    g = np.empty((nx + 2,) + f.shape[1:])
    g[1:-1] = f
    if kind == "periodic":
        g[0], g[-1] = f[-1], f[0]
    elif kind == "outflow":
        g[0], g[-1] = f[0], f[-1]
    else:
        g[0], g[-1] = 0.0, 0.0
    fl = cpos * g[:-1] + cneg * g[1:]
    out = f - (dt / mesh.dx) * (fl[1:] - fl[:-1])
    e = field_bound(force)
    if e > 0.0:
        E = force[:, None, None, None]
        a, b = f[:, :-1], f[:, 1:]
        G = 0.5 * E * (a + b) - 0.5 * e * (b - a)
        r = dt / mesh.dv[0]
        out[:, 0] -= r * G[:, 0]
        out[:, 1:-1] -= r * (G[:, 1:] - G[:, :-1])
        out[:, -1] -= r * (-G[:, -1])
    return out


def minmod(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """0 where a, b differ in sign (or one is 0), else the smaller magnitude with their sign."""
    return np.where(a * b > 0.0, np.sign(a) * np.minimum(np.abs(a), np.abs(b)), 0.0)


def transport_muscl(f: np.ndarray, dt: float, mesh: Mesh, periodic) -> np.ndarray:
    """Second-order x transport (ORACLE EXTENSION; BASELINE north_star's
    "upwind/MUSCL", PAPER's flux limiters): MUSCL reconstruction with the
    minmod limiter, upwind face states, forward Euler, on the reference's
    flux form (ref/kinetic.py:110-112 with g -> reconstructed face states):
        s_j = minmod(g_j - g_{j-1}, g_{j+1} - g_j),
        F_{j+1/2} = max(c,0) (g_j + s_j/2) + min(c,0) (g_{j+1} - s_{j+1}/2),
        f* = f - (dt/dx)(F_{i+1/2} - F_{i-1/2}).
    Two ghost planes per side: periodic wrap, zero (absorbing) or copies of
    the edge plane (outflow).  No v_x field term (upwind only)."""
    kind = bc_kind(periodic)
    nx = f.shape[0]
    c = mesh.vc[0]
    cpos = np.maximum(c, 0.0)[None, :, None, None]
    cneg = np.minimum(c, 0.0)[None, :, None, None]
    g = np.empty((nx + 4,) + f.shape[1:])
    g[2:-2] = f
    if kind == "periodic":
        g[0], g[1], g[-2], g[-1] = f[-2], f[-1], f[0], f[1]
    elif kind == "outflow":
        g[0], g[1], g[-2], g[-1] = f[0], f[0], f[-1], f[-1]
    else:
        g[0] = g[1] = g[-2] = g[-1] = 0.0
    sl = minmod(g[1:-1] - g[:-2], g[2:] - g[1:-1])  # slopes of g[1..nx+2]
    gL = g[1:-2] + 0.5 * sl[:-1]  # left state of faces g[1]|g[2] .. g[nx+1]|g[nx+2]
    gR = g[2:-1] - 0.5 * sl[1:]   # right state of the same faces
    fl = cpos * gL + cneg * gR
    return f - (dt / mesh.dx) * (fl[1:] - fl[:-1])


def unit_tau(rho, theta):
    """Default collision frequency (ref/kinetic.py:42-44)."""
    return 1.0


def relax(fs: np.ndarray, dt: float, mesh: Mesh, eps: float,
          tau: Callable = unit_tau) -> np.ndarray:
    """Implicit BGK blend (ref/kinetic.py:127-134)."""
    rho, u, theta = project(fs, mesh)
    lam = dt * np.asarray(tau(rho, theta), dtype=float) / eps
    lam = np.broadcast_to(lam, rho.shape)[:, None, None, None]
    M = lift(rho, u, theta, mesh, normalize=True)
    return (fs + lam * M) / (1.0 + lam)


def fine_schedule(t0: float, t1: float, cap: float) -> list:
    """The dt sequence of ref/kinetic.py:146-160 (Python-float arithmetic)."""
    span = t1 - t0
    out = []
    done = 0.0
    while span - done > GUARD * span:
        d = min(cap, span - done)
        out.append(d)
        done += d
    return out


def scaled_cap(mesh: Mesh, cfl: float, force, eps: float, alpha: int) -> float:
    """CFL cap in physical time.  ORACLE EXTENSION for alpha = 1 (diffusive
    scaling, PAPER eq. (1): transport rate 1/eps, relaxation 1/eps^2): the
    alpha = 0 cap times eps."""
    cap = fine_cap(mesh, cfl, force)
    return cap * eps if alpha == 1 else cap


def fine_propagate(f0: np.ndarray, t0: float, t1: float, mesh: Mesh,
                   eps: float, periodic: bool, force=None, dt_max=None,
                   cfl: float = 0.5, tau: Callable = unit_tau, alpha: int = 0,
                   scheme: str = "upwind") -> np.ndarray:
    """F over [t0, t1] (ref/kinetic.py:137-161).

    ``alpha = 1`` is an ORACLE EXTENSION (unpinned; the reference has only
    alpha = 0): a physical step d runs the reference's transport and relax
    with the scaled step d / eps, i.e. transport rate d/(eps dx) and
    lambda = (d/eps) tau / eps = d tau / eps^2."""
    if t1 < t0:
        raise OracleConfigError("t1 < t0")
    if t1 - t0 == 0.0:
        return f0
    cap = scaled_cap(mesh, cfl, force, eps, alpha)
    if dt_max is not None:
        cap = min(cap, dt_max)
    f = f0
    for s, d in enumerate(fine_schedule(t0, t1, cap), start=1):
        if alpha == 1:
            d = d / eps
        if scheme == "muscl":
            if field_bound(force) > 0.0:
                raise OracleConfigError("MUSCL x transport has no field term")
            f = transport_muscl(f, d, mesh, periodic)
        else:
            f = transport(f, d, mesh, periodic, force)
        f = relax(f, d, mesh, eps, tau)
        if not np.all(np.isfinite(f)):
            raise OracleBlowUp("non-finite at step %d" % s, step=s)
    return f


# --------------------------------------------------------------------------
# coarse propagator G (ref/fluid.py:39-125, ref/moments.py:116-129)
# --------------------------------------------------------------------------

def to_conserved(rho, u, theta) -> np.ndarray:
    """Packed (nx, 5) conserved state (ref/moments.py:116-119, 59-72)."""
    out = np.empty((rho.shape[0], 5))
    out[:, 0] = rho
    out[:, 1:4] = rho[:, None] * u
    out[:, 4] = 0.5 * rho * np.einsum("ij,ij->i", u, u) + 1.5 * rho * theta
    return out


def to_primitive(v: np.ndarray):
    """ref/moments.py:122-129 on a packed state."""
    rho = v[:, 0].copy()
    mom = v[:, 1:4].copy()
    en = v[:, 4].copy()
    if np.any(rho <= 0.0):
        raise OracleDegenerate("rho <= 0 in conserved state")
    u = mom / rho[:, None]
    eint = en - 0.5 * np.einsum("ij,ij->i", mom, u)
    if np.any(eint <= 0.0):
        raise OracleDegenerate("internal energy <= 0")
    return rho, u, eint / (1.5 * rho)


def pressure(v: np.ndarray) -> np.ndarray:
    """ref/fluid.py:39-42."""
    ke = 0.5 * (v[..., 1] ** 2 + v[..., 2] ** 2 + v[..., 3] ** 2) / v[..., 0]
    return (v[..., 4] - ke) / 1.5


def euler_flux(v: np.ndarray) -> np.ndarray:
    """ref/fluid.py:45-56."""
    v = np.asarray(v, dtype=float)
    ux = v[..., 1] / v[..., 0]
    p = pressure(v)
    h = np.empty_like(v)
    h[..., 0] = v[..., 1]
    h[..., 1] = v[..., 1] * ux + p
    h[..., 2] = v[..., 2] * ux
    h[..., 3] = v[..., 3] * ux
    h[..., 4] = ux * (v[..., 4] + p)
    return h


def rusanov(vl: np.ndarray, vr: np.ndarray) -> np.ndarray:
    """ref/fluid.py:59-66."""
    vl = np.asarray(vl, dtype=float)
    vr = np.asarray(vr, dtype=float)
    sl = np.abs(vl[..., 1] / vl[..., 0]) + np.sqrt(pressure(vl) / vl[..., 0])
    sr = np.abs(vr[..., 1] / vr[..., 0]) + np.sqrt(pressure(vr) / vr[..., 0])
    s = np.maximum(sl, sr)
    return 0.5 * (euler_flux(vl) + euler_flux(vr)) - 0.5 * s[..., None] * (vr - vl)


def coarse_cap(v: np.ndarray, dx: float, cfl: float) -> float:
    """ref/fluid.py:69-75 on a packed state."""
    ux = v[:, 1] / v[:, 0]
    th = pressure(v) / v[:, 0]
    return cfl * dx / float(np.max(np.abs(ux) + np.sqrt(th)))


def coarse_propagate(rho, u, theta, t0, t1, mesh: Mesh, periodic: bool,
                     force=None, dt_max=None, cfl: float = 0.9):
    """G over [t0, t1] (ref/fluid.py:91-125); returns (rho, u, theta)."""
    if t1 < t0:
        raise OracleConfigError("t1 < t0")
    span = t1 - t0
    if span == 0.0:
        return rho, u, theta
    v = to_conserved(rho, u, theta)
    done = 0.0
    step = 0
    while span - done > GUARD * span:
        d = coarse_cap(v, mesh.dx, cfl)
        if dt_max is not None:
            d = min(d, dt_max)
        d = min(d, span - done)
        g = np.empty((v.shape[0] + 2, 5))
        g[1:-1] = v
        if bc_kind(periodic) == "periodic":
            g[0], g[-1] = v[-1], v[0]
        else:  # transmissive copy (ref/fluid.py:84-87); also for 'outflow'
            g[0], g[-1] = v[0], v[-1]
        H = rusanov(g[:-1], g[1:])
        nv = v - (d / mesh.dx) * (H[1:] - H[:-1])
        if force is not None:
            nv[:, 1] += d * v[:, 0] * force
            nv[:, 4] += d * v[:, 1] * force
        step += 1
        if not np.all(np.isfinite(nv)):
            raise OracleBlowUp("fluid non-finite at step %d" % step, step=step)
        if np.any(nv[:, 0] <= 0.0) or np.any(pressure(nv) <= 0.0):
            raise OracleBlowUp("fluid unphysical at step %d" % step, step=step)
        v = nv
        done += d
    return to_primitive(v)


# --------------------------------------------------------------------------
# drift-diffusion coarse propagator -- ORACLE EXTENSION (unpinned)
# --------------------------------------------------------------------------
# PAPER eq. (DDbis): d_t rho - m2 d_x J = 0, J = d_x rho - E rho, with u = 0,
# theta = 1; discretised by the central finite-difference scheme the paper
# names, explicit in time.  The reference has no diffusive G
# (SPEC:8); this is the builder's restatement, the checker of the CUDA G.
# Conservative face fluxes J_{i+1/2} = (rho_{i+1}-rho_i)/dx
# - 0.5 (E_i rho_i + E_{i+1} rho_{i+1}); rho_i += (dt D / dx)(J_{i+1/2} - J_{i-1/2}).
# Ghosts: periodic wrap, else zero-gradient copies of rho and E.

def dd_m2(mesh: Mesh) -> float:
    """Second moment of the discrete unit Maxwellian along v_x (m2 of DDbis)."""
    c = mesh.vc[0]
    w = np.exp(-(c * c) * 0.5)
    return float(np.sum(c * c * w) / np.sum(w))


def dd_cap(dx: float, D: float, e_max: float, cfl: float) -> float:
    """Explicit stability bound cfl dx^2 / (D (2 + dx e_max))."""
    return cfl * dx * dx / (D * (2.0 + dx * e_max))


def dd_propagate(rho, t0, t1, mesh: Mesh, periodic, force=None, dt_max=None,
                 cfl: float = 0.9, D: float = 1.0):
    """G over [t0, t1] for the drift-diffusion model; returns (rho, u=0, theta=1)."""
    if t1 < t0:
        raise OracleConfigError("t1 < t0")
    nx = rho.shape[0]
    span = t1 - t0
    if span == 0.0:
        return rho, np.zeros((nx, 3)), np.ones(nx)
    E = np.zeros(nx) if force is None else np.asarray(force, dtype=float)
    cap = dd_cap(mesh.dx, D, field_bound(force), cfl)
    if dt_max is not None:
        cap = min(cap, dt_max)
    r = np.array(rho, dtype=float, copy=True)
    done = 0.0
    step = 0
    g = np.empty(nx + 2)
    e = np.empty(nx + 2)
    e[1:-1] = E
    if bc_kind(periodic) == "periodic":
        e[0], e[-1] = E[-1], E[0]
    else:
        e[0], e[-1] = E[0], E[-1]
    while span - done > GUARD * span:
        d = min(cap, span - done)
        g[1:-1] = r
        if bc_kind(periodic) == "periodic":
            g[0], g[-1] = r[-1], r[0]
        else:
            g[0], g[-1] = r[0], r[-1]
        J = (g[1:] - g[:-1]) / mesh.dx - 0.5 * (e[:-1] * g[:-1] + e[1:] * g[1:])
        coef = d * D / mesh.dx
        nr = r + coef * (J[1:] - J[:-1])
        step += 1
        if not np.all(np.isfinite(nr)):
            raise OracleBlowUp("drift-diffusion non-finite at step %d" % step, step=step)
        if np.any(nr <= 0.0):
            raise OracleBlowUp("drift-diffusion unphysical at step %d" % step, step=step)
        r = nr
        done += d
    return r, np.zeros((nx, 3)), np.ones(nx)


# --------------------------------------------------------------------------
# parareal slice loop (ref/parareal.py:109-314)
# --------------------------------------------------------------------------

@dataclass
class Problem:
    """Everything one parareal run fixes (mesh, time grid, physics)."""

    mesh: Mesh
    t_final: float
    n_g: int
    n_f: int
    eps: float
    periodic: bool
    force: Optional[np.ndarray] = None
    cfl_kin: float = 0.5
    cfl_fluid: float = 0.9
    tau: Callable = unit_tau
    alpha: int = 0                 # 1: diffusive scaling (ORACLE EXTENSION)
    g_model: str = "euler"         # "drift_diffusion": dd_propagate (ORACLE EXTENSION)
    scheme: str = "upwind"         # "muscl": transport_muscl (ORACLE EXTENSION)
    diffusivity: Optional[float] = None  # D of the drift-diffusion G (default m2 / 1)

    @property
    def times(self):
        return coarse_grid(self.t_final, self.n_g, self.n_f)[0]

    @property
    def dt_g(self):
        return self.t_final / self.n_g

    @property
    def dt_f(self):
        return self.t_final / self.n_f


def G(prob: Problem, U, n: int):
    """Coarse solve over window n (1-based)."""
    t = prob.times
    if prob.g_model == "drift_diffusion":
        D = prob.diffusivity if prob.diffusivity is not None else dd_m2(prob.mesh)
        return dd_propagate(U[0], float(t[n - 1]), float(t[n]), prob.mesh, prob.periodic,
                            prob.force, prob.dt_g, prob.cfl_fluid, D)
    return coarse_propagate(*U, float(t[n - 1]), float(t[n]), prob.mesh,
                            prob.periodic, prob.force, prob.dt_g, prob.cfl_fluid)


def PFL(prob: Problem, U, n: int):
    """Fine solve of window n from moments U: P(F(L(U))) (ref/parareal.py:123-142)."""
    t = prob.times
    f = lift(*U, prob.mesh, normalize=False)
    f = fine_propagate(f, float(t[n - 1]), float(t[n]), prob.mesh, prob.eps,
                       prob.periodic, prob.force, prob.dt_f, prob.cfl_kin,
                       prob.tau, prob.alpha, prob.scheme)
    return project(f, prob.mesh)


def _sub(a, b):
    return tuple(x - y for x, y in zip(a, b))


def _add(a, b):
    return tuple(x + y for x, y in zip(a, b))


def sup_gap(a, b) -> float:
    """ref/moments.py:48-52."""
    return max(float(np.max(np.abs(x - y))) for x, y in zip(a, b))


def window_jump(prob: Problem, U, n: int):
    """Delta^n = P F L (U) - G (U) (ref/parareal.py:123-142)."""
    return _sub(PFL(prob, U, n), G(prob, U, n))


def parareal(prob: Problem, U0, k_max: int, tol: float, frozen: bool = True,
             jump_fn=None):
    """Outer iteration (ref/parareal.py:109-120, 179-278).

    Returns (snapshots, errors).  ``jump_fn(prob, U, n)`` may replace the
    serial window jump (tests use it to inject distributed variants).
    """
    jump_fn = jump_fn or window_jump
    snaps = [tuple(np.array(x, copy=True) for x in U0)]
    for n in range(1, prob.n_g + 1):
        snaps.append(G(prob, snaps[-1], n))
    jumps = [None] * prob.n_g
    errors = []
    for k in range(1, k_max + 1):
        start = k if frozen else 1
        for n in range(start, prob.n_g + 1):
            jumps[n - 1] = jump_fn(prob, snaps[n - 1], n)
        new = list(snaps)
        err = 0.0
        for n in range(start, prob.n_g + 1):
            cor = _add(G(prob, new[n - 1], n), jumps[n - 1])
            ok = all(np.all(np.isfinite(x)) for x in cor)
            if not ok or np.any(cor[0] <= 0.0) or np.any(cor[2] <= 0.0):
                raise OracleOvershoot("overshoot in window %d" % n, slice_index=n)
            err = max(err, sup_gap(cor, snaps[n]))
            new[n] = cor
        snaps = new
        errors.append(err)
        if err < tol:
            break
    return snaps, errors


def fine_chain(prob: Problem, U0):
    """Window-wise serial fine reference (ref/parareal.py:281-295)."""
    out = [tuple(np.array(x, copy=True) for x in U0)]
    for n in range(1, prob.n_g + 1):
        out.append(PFL(prob, out[-1], n))
    return out


def work_range(work: int, n_p: int, rank: int):
    """(start, end, end-start, size) of ref/parareal.py:298-314."""
    if n_p < 1 or not 0 <= rank < n_p or work < 0:
        raise OracleConfigError("bad partition request")
    q, r = divmod(work, n_p)
    s = rank * q + min(r, rank) + 1
    e = (rank + 1) * q + min(r, rank + 1)
    return s, e, e - s, max(0, e - s + 1)


# --------------------------------------------------------------------------
# synthetic problem builders for the BASELINE.json configs
# --------------------------------------------------------------------------

def two_state(mesh: Mesh, edge: float, left, right):
    """Piecewise (rho, u_x, theta) classified by cell centre (ref/cases.py:29-42)."""
    x = mesh.xc
    m = x < edge
    rho = np.where(m, left[0], right[0]).astype(float)
    u = np.zeros((mesh.nx, 3))
    u[:, 0] = np.where(m, left[1], right[1])
    theta = np.where(m, left[2], right[2]).astype(float)
    return rho, u, theta
