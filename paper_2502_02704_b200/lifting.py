"""Distributions and the Maxwellian lift L (GPU).

``Distribution`` keeps the reference's ``values`` attribute (an
``(nx, nvx, nvy, nvz)`` fp64 array, ref/lifting.py:16-23) but lives on the
device: solver results are CUDA tensors and ``values`` copies them to the host
on first access.  After such an access the host array is the authoritative
copy (it may be mutated in place, as the reference's own tests do), and the
next GPU call uploads it again.  Code that wants to stay on the device uses
``device_tensor()`` / ``Distribution.on_device``.

``lift`` builds three per-cell 1-D exponential tables in the finalize kernel
and writes ``f = ((gx amp) gy) gz`` (optionally times rho/mass) in one sweep,
following ref/lifting.py:36-58.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import runtime as rt
from .errors import DegenerateStateError

__all__ = ["Distribution", "maxwellian", "lift", "as_device_f"]


class Distribution:
    """Discrete distribution f[i, jx, jy, jz] (host- or device-resident)."""

    __slots__ = ("_host", "_dev")

    def __init__(self, values):
        self._host = None
        self._dev = None
        if isinstance(values, torch.Tensor):
            if values.is_cuda:
                self._dev = values
            else:
                self._host = values.numpy()
        else:
            self._host = values

    @classmethod
    def on_device(cls, t: torch.Tensor) -> "Distribution":
        return cls(t)

    @property
    def values(self):
        if self._host is None:
            # through a (cached) pinned block: DMA at full PCIe rate, no page
            # faults on a fresh pageable allocation (the numpy view keeps the
            # pinned tensor alive)
            h = torch.empty(tuple(self._dev.shape), dtype=self._dev.dtype, pin_memory=True)
            h.copy_(self._dev)
            self._host = h.numpy()
        self._dev = None  # the host copy may now be mutated in place
        return self._host

    @values.setter
    def values(self, v):
        self._dev = None
        self._host = None
        if isinstance(v, torch.Tensor) and v.is_cuda:
            self._dev = v
        else:
            self._host = v

    @property
    def shape(self):
        return tuple(self._dev.shape) if self._dev is not None else np.shape(self._host)

    @property
    def is_device(self) -> bool:
        return self._dev is not None

    def device_tensor(self, device=None) -> torch.Tensor:
        """fp64 C-contiguous CUDA tensor of f (uploads a host array)."""
        device = device or rt.current_device()
        if self._dev is not None:
            t = self._dev
            if t.device != device:
                t = t.to(device)
            if t.dtype != torch.float64:
                t = t.double()
            return t.contiguous()
        arr = np.ascontiguousarray(self._host, dtype=np.float64)
        return torch.from_numpy(arr).to(device, non_blocking=False)

    def copy(self) -> "Distribution":
        if self._dev is not None:
            return Distribution(self._dev.clone())
        return Distribution(np.array(self._host, copy=True))


def as_device_f(f, ctx) -> torch.Tensor:
    if isinstance(f, Distribution):
        t = f.device_tensor(ctx.device)
    elif isinstance(f, torch.Tensor):
        t = f.to(ctx.device, torch.float64).contiguous()
    else:  # a reference Distribution or a bare array
        vals = getattr(f, "values", f)
        t = torch.from_numpy(np.ascontiguousarray(vals, dtype=np.float64)).to(ctx.device)
    if tuple(t.shape) != ctx.shape:
        raise ValueError("distribution shape %s does not match grid %s" % (tuple(t.shape), ctx.shape))
    return t


def maxwellian(rho: float, u, theta: float, v) -> float:
    """Point value of one Maxwellian (ref/lifting.py:26-33); scalar host helper."""
    if theta <= 0.0:
        raise DegenerateStateError("need theta > 0, got %r" % (theta,))
    d = np.asarray(v, dtype=float) - np.asarray(u, dtype=float)
    return float(rho / (2.0 * np.pi * theta) ** 1.5 * np.exp(-np.sum(d ** 2) / (2.0 * theta)))


def lift(U, grid, normalize_mass: bool = False, bc=None) -> Distribution:
    """L: cell-local Maxwellians on the velocity centres, on the GPU."""
    if np.any(np.asarray(U.rho) <= 0.0) or np.any(np.asarray(U.theta) <= 0.0):
        raise DegenerateStateError("lift requires rho > 0 and theta > 0 in every cell")
    ctx = rt.ctx_for(grid, bc if bc is not None else "absorbing")
    mom = rt.to_device_moments(U, ctx.device)
    out = ctx.empty_f()
    code = ctypes.c_longlong(-1)
    rt._lib.check(ctx.lib.pbgk_lift(ctx.h, rt.ptr(mom), 1 if normalize_mass else 0, rt.ptr(out),
                                    rt.stream_handle(ctx.device), ctypes.byref(code)),
                  "pbgk_lift")
    rt.raise_kinetic(code.value)
    return Distribution(out)
