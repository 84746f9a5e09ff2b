"""Shared builders and the normwise parity metric."""

from __future__ import annotations

import numpy as np

from oracle import bgk as O


def rel_inf(a, b) -> float:
    """||a - b||_inf / ||b||_inf (0 if both are zero)."""
    a = np.asarray(a, dtype=float)
    b = np.asarray(b, dtype=float)
    den = float(np.max(np.abs(b))) if b.size else 0.0
    num = float(np.max(np.abs(a - b))) if b.size else 0.0
    if den == 0.0:
        return num
    return num / den


def moment_gap(a, b) -> float:
    """Parity metric on (rho, u, theta): relative for rho/theta, u scaled by
    max(|u|, sqrt(theta))."""
    ra, ua, ta = a
    rb, ub, tb = b
    scale_u = max(float(np.max(np.abs(ub))), float(np.sqrt(np.max(np.abs(tb)))))
    return max(rel_inf(ra, rb), rel_inf(ta, tb),
               float(np.max(np.abs(np.asarray(ua) - np.asarray(ub)))) / scale_u)


def mf(U):
    """(rho, u, theta) of a MomentField-like object."""
    return (np.asarray(U.rho), np.asarray(U.u), np.asarray(U.theta))


def random_moments(nx, rng, rho=(0.5, 1.5), u=0.4, theta=(0.5, 1.5)):
    return (rng.uniform(*rho, nx), rng.uniform(-u, u, (nx, 3)), rng.uniform(*theta, nx))


def pkg_grids(P, x_min, x_max, nx, v_max, nv):
    return P.PhaseGrid(P.build_spatial_grid(x_min, x_max, nx), P.build_velocity_grid(v_max, nv))
