"""Exact solution of the 1-D Euler Riemann problem (ideal gas, gamma = 5/3).

Independent checker for the coarse solver's shock-tube behaviour (the
reference's acceptance criterion 7 uses an exact-Riemann L1 bound).  Textbook
construction: Newton iteration on the star-region pressure, then sampling of
the self-similar wave fan at speeds xi = x / t.  States are (rho, u, p).
"""

from __future__ import annotations

import math

import numpy as np

G = 5.0 / 3.0


def _f_and_df(p, rho, pk):
    """Velocity jump across one wave and its derivative w.r.t. star pressure."""
    a = math.sqrt(G * pk / rho)
    if p > pk:  # shock
        A = 2.0 / ((G + 1.0) * rho)
        B = (G - 1.0) / (G + 1.0) * pk
        s = math.sqrt(A / (p + B))
        return (p - pk) * s, s * (1.0 - 0.5 * (p - pk) / (p + B))
    e = (G - 1.0) / (2.0 * G)
    return (2.0 * a / (G - 1.0)) * ((p / pk) ** e - 1.0), (p / pk) ** (-(G + 1.0) / (2.0 * G)) / (rho * a)


def star(left, right):
    (rl, ul, pl), (rr, ur, pr) = left, right
    al, ar = math.sqrt(G * pl / rl), math.sqrt(G * pr / rr)
    e = (G - 1.0) / (2.0 * G)
    p = ((al + ar - 0.5 * (G - 1.0) * (ur - ul)) / (al / pl ** e + ar / pr ** e)) ** (1.0 / e)
    for _ in range(100):
        fl, dl = _f_and_df(p, rl, pl)
        fr, dr = _f_and_df(p, rr, pr)
        step = (fl + fr + ur - ul) / (dl + dr)
        p = max(p - step, 1e-14)
        if abs(step) <= 1e-15 * p:
            break
    fl, _ = _f_and_df(p, rl, pl)
    fr, _ = _f_and_df(p, rr, pr)
    return p, 0.5 * (ul + ur) + 0.5 * (fr - fl)


def density(left, right, xi):
    ps, us = star(left, right)
    out = np.empty(len(xi))
    for n, s in enumerate(xi):
        side, sgn = (left, -1.0) if s <= us else (right, 1.0)
        rk, uk, pk = side
        ak = math.sqrt(G * pk / rk)
        if ps > pk:  # shock on this side
            sh = uk + sgn * ak * math.sqrt((G + 1.0) / (2.0 * G) * ps / pk + (G - 1.0) / (2.0 * G))
            if sgn * (s - sh) > 0.0:
                out[n] = rk
            else:
                q = (G - 1.0) / (G + 1.0)
                out[n] = rk * (ps / pk + q) / (q * ps / pk + 1.0)
        else:  # rarefaction
            head = uk + sgn * ak
            tail = us + sgn * ak * (ps / pk) ** ((G - 1.0) / (2.0 * G))
            if sgn * (s - head) > 0.0:
                out[n] = rk
            elif sgn * (s - tail) < 0.0:
                out[n] = rk * (ps / pk) ** (1.0 / G)
            else:
                out[n] = rk * (2.0 / (G + 1.0) - sgn * (G - 1.0) / ((G + 1.0) * ak) * (uk - s)) ** \
                    (2.0 / (G - 1.0))
    return out
