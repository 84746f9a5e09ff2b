"""x-sharded fine propagator F over ranks (an extension).

The reference parallelises only over parareal windows; a single fine
propagation (config 1's fine-only run, the serial fine reference of
``run_fine_mode``) is one process.  Here the x cells of one propagation are
split into contiguous slabs, one per rank (``work_distribution``), and every
fine step is the unsharded step restricted to the slab:

* each rank owns a slab context (``bc = 3``) whose f and table buffers are
  padded by one plane / row per side;
* after every step (sweep -> f*_s, finalize -> R_s tables) the ranks swap
  their boundary planes f*_s and table rows R_s with their x neighbours
  (1 plane = nvx*nvy*nvz*8 bytes per side; config 4: 2 MiB) -- over NCCL
  point-to-point (NVLink) when the group is NCCL, host-staged over gloo;
* at the global x ends the halos are filled locally: zeros (absorbing),
  the edge itself (outflow), the far slab (periodic).

Each cell's arithmetic and velocity reductions stay within its own plane, so
the sharded F is bitwise the single-GPU F (tested with 2 and 3 ranks).
Failure keys are min-reduced over ranks at the end, so every rank raises
the same exception with the reference's step index.
"""

from __future__ import annotations

import ctypes
from typing import Optional

import numpy as np
import torch

from . import runtime as rt
from .errors import ConfigurationError
from .grid import bc_code
from .kinetic import _kdt, _scheme, fine_schedule, stable_dt_kinetic, tau_constant
from .parareal import work_distribution

__all__ = ["SlabFine"]


class SlabFine:
    """One rank's slab of an x-sharded fine propagation on ``grid``."""

    def __init__(self, grid, bc, params, device: Optional[torch.device] = None, group=None):
        dist = torch.distributed
        self.group = group
        self.world = dist.get_world_size(group) if (dist.is_available() and dist.is_initialized()) else 1
        self.rank = dist.get_rank(group) if self.world > 1 else 0
        self.params = params
        if tau_constant(params.tau) is None:
            raise ConfigurationError("the x-sharded F needs a constant tau")
        if getattr(params, "scheme", "upwind") != "upwind":
            raise ConfigurationError("the x-sharded F supports the upwind x scheme only")
        self.grid = grid
        self.bc = bc_code(bc)
        nx = grid.space.n_x
        r = work_distribution(nx, self.world, self.rank)
        if r.size < 1:
            raise ConfigurationError("x-sharding %d cells over %d ranks leaves a rank empty"
                                     % (nx, self.world))
        self.x0, self.n = r.start - 1, r.size
        self.device = device or rt.current_device()
        nv = tuple(int(v) for v in grid.velocity.n_v)
        dx = grid.space.dx
        self.ctx = rt.Ctx((self.n,) + nv, grid.space.x_min + self.x0 * dx,
                          grid.space.x_min + (self.x0 + self.n) * dx, grid.velocity.v_max, 3,
                          self.device)
        lib, h = self.ctx.lib, self.ctx.h
        rt._lib.check(lib.pbgk_ctx_set_dx(h, float(dx)), "pbgk_ctx_set_dx")
        if getattr(grid.velocity, "quadrature", "midpoint") == "trapezoid":
            self.ctx.set_quadrature(1)
        _scheme(self.ctx, params)
        self.TL = lib.pbgk_table_len(h)
        shp = (self.n + 2,) + nv
        f64 = dict(dtype=torch.float64, device=self.device)
        self.f = [torch.zeros(shp, **f64), torch.zeros(shp, **f64)]
        self.t = [torch.zeros((self.n + 2, self.TL), **f64), torch.zeros((self.n + 2, self.TL), **f64)]
        E = params.force
        self.e_max = 0.0 if E is None else float(np.max(np.abs(E)))
        self.E = None
        if E is not None and self.e_max > 0.0:
            self.E = torch.from_numpy(np.ascontiguousarray(
                np.asarray(E, dtype=float)[self.x0:self.x0 + self.n])).to(self.device)
        self.nccl = self.world > 1 and dist.get_backend(group) == "nccl"
        periodic = self.bc == 1
        self.left = (self.rank - 1) % self.world if (self.rank > 0 or periodic) else None
        self.right = (self.rank + 1) % self.world if (self.rank < self.world - 1 or periodic) else None

    # -- halo exchange ---------------------------------------------------------------
    def _halos(self, f: Optional[torch.Tensor], tab: torch.Tensor) -> None:
        """Fill plane / row 0 and n+1 of (f, tab) from the neighbours or the x boundary."""
        n = self.n
        pairs = [(tab, 1, n)] if f is None else [(f, 1, n), (tab, 1, n)]
        if self.world == 1 or (self.left is None and self.right is None):
            for buf, lo, hi in pairs:
                self._edge(buf, 0, lo, hi)
                self._edge(buf, n + 1, lo, hi)
            return
        dist = torch.distributed
        ops, stage = [], []
        for q, (buf, lo, hi) in enumerate(pairs):
            # left-bound message: my first interior plane -> left neighbour's
            # right halo; right-bound: my last -> right neighbour's left halo
            for peer, src, dst, tag in ((self.left, lo, n + 1, 2 * q), (self.right, hi, 0, 2 * q + 1)):
                if peer is None:
                    continue
                out = buf[src] if self.nccl else buf[src].cpu()
                ops.append(dist.P2POp(dist.isend, out.contiguous(), peer, self.group, tag))
            for peer, dst, tag in ((self.right, n + 1, 2 * q), (self.left, 0, 2 * q + 1)):
                if peer is None:
                    continue
                into = buf[dst] if self.nccl else torch.empty(buf[dst].shape, dtype=buf.dtype)
                ops.append(dist.P2POp(dist.irecv, into, peer, self.group, tag))
                stage.append((buf, dst, into))
        for w in dist.batch_isend_irecv(ops):
            w.wait()
        if not self.nccl:
            for buf, dst, into in stage:
                buf[dst].copy_(into)
        for buf, lo, hi in pairs:
            if self.left is None:
                self._edge(buf, 0, lo, hi)
            if self.right is None:
                self._edge(buf, n + 1, lo, hi)

    def _edge(self, buf, dst, lo, hi):
        """A global-boundary halo: absorbing 0, outflow = the edge, periodic (one slab) = wrap."""
        if self.bc == 0:
            buf[dst].zero_()
        elif self.bc == 2:
            buf[dst].copy_(buf[lo if dst == 0 else hi])
        else:
            buf[dst].copy_(buf[hi if dst == 0 else lo])

    # -- propagation ------------------------------------------------------------------
    def propagate(self, t0: float, t1: float, f0: Optional[torch.Tensor] = None,
                  mom0: Optional[torch.Tensor] = None, dt_max=None, want_f: bool = True,
                  want_moments: bool = False):
        """F over [t0, t1] of this slab, from its planes f0 (n, nv...) or from
        its moments mom0 (5, n) (the lift is synthesised).  Returns
        (f (n, nv...) or None, moments (5, n) or None)."""
        if t1 < t0:
            raise ConfigurationError("need t1 >= t0, got [%r, %r]" % (t0, t1))
        p = self.params
        lib, h = self.ctx.lib, self.ctx.h
        st = rt.stream_handle(self.device)
        cap = stable_dt_kinetic(self.grid, p)
        if dt_max is not None:
            cap = min(cap, dt_max)
        dts = fine_schedule(t1 - t0, cap) if t1 > t0 else []
        tau = tau_constant(p.tau)
        keys = []
        code = ctypes.c_longlong(-1)
        fa, fb = self.f
        ta, tb = self.t
        if f0 is not None:
            fa[1:self.n + 1].copy_(f0)
            rt._lib.check(lib.pbgk_slab_tables(h, 0, None, rt.ptr(ta), st, ctypes.byref(code)),
                          "pbgk_slab_tables")
            self._halos(fa, ta)
            cur = fa
        else:
            rt._lib.check(lib.pbgk_slab_tables(h, 1, rt.ptr(mom0.contiguous()), rt.ptr(ta), st,
                                               ctypes.byref(code)), "pbgk_slab_tables")
            keys.append(code.value)
            self._halos(None, ta)
            cur = None
        field = self.E is not None
        for s, dt in enumerate(dts, start=1):
            d = _kdt(dt, p)
            rt._lib.check(lib.pbgk_slab_sweep(h, rt.ptr(cur), rt.ptr(ta), rt.ptr(fb), float(d),
                                              rt.ptr(self.E), self.e_max, st), "pbgk_slab_sweep")
            rt._lib.check(lib.pbgk_slab_finalize(h, 0, 1 if field else 0, rt.ptr(tb), None, float(d),
                                                 float(p.epsilon), tau, s, st, None),
                          "pbgk_slab_finalize")
            self._halos(fb, tb)
            cur = fb
            fa, fb = fb, fa
            ta, tb = tb, ta
        # final pass: relax R_S only (no transport); with no steps it returns
        # f0 (identity tables) or the synthesised lift
        out_f = mom = None
        S = len(dts)
        rt._lib.check(lib.pbgk_slab_sweep(h, rt.ptr(cur), rt.ptr(ta), rt.ptr(fb) if want_f else None,
                                          0.0, None, 0.0, st), "pbgk_slab_sweep")
        mom = torch.empty((5, self.n), dtype=torch.float64, device=self.device)
        # the projection also reads back the failure key of the whole run
        rt._lib.check(lib.pbgk_slab_finalize(h, 1, 0, None, rt.ptr(mom), 0.0, 1.0, 1.0, S + 1,
                                             st, ctypes.byref(code)), "pbgk_slab_finalize")
        keys.append(code.value)
        if not want_moments:
            mom = None
        if want_f:
            out_f = fb[1:self.n + 1].clone()
        self._raise_agreed(keys)
        return out_f, mom

    def _raise_agreed(self, keys):
        bad = [k for k in keys if k >= 0]
        key = min(bad) if bad else (1 << 62)
        if self.world > 1:
            t = torch.tensor([key], dtype=torch.int64,
                             device=self.device if self.nccl else torch.device("cpu"))
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MIN, group=self.group)
            key = int(t.item())
        if key < (1 << 62):
            rt.raise_kinetic(key)

    def gather(self, local: torch.Tensor, axis: int = 0) -> torch.Tensor:
        """Concatenate every rank's slab of a per-cell tensor along `axis` (x)."""
        if self.world == 1:
            return local
        dist = torch.distributed
        nx = self.grid.space.n_x
        parts = []
        sizes = [work_distribution(nx, self.world, q).size for q in range(self.world)]
        mx = max(sizes)
        loc = local.movedim(axis, 0).contiguous()
        pad = torch.zeros((mx,) + tuple(loc.shape[1:]), dtype=loc.dtype, device=loc.device)
        pad[:loc.shape[0]] = loc
        src = pad if self.nccl else pad.cpu()
        flat = torch.empty((self.world * src.numel(),), dtype=src.dtype, device=src.device)
        dist.all_gather_into_tensor(flat, src.reshape(-1), group=self.group)
        g = flat.view((self.world,) + tuple(src.shape))
        for q in range(self.world):
            parts.append(g[q, :sizes[q]])
        return torch.cat(parts, 0).to(local.device).movedim(0, axis)
