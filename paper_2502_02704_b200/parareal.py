"""Parareal slice loop on the GPU, optionally sharded over ranks (one GPU each).

Same API and semantics as ref/parareal.py:49-333.  The state of a run lives
on the device as three tensors — snapshots ``(n_g+1, 5, nx)``, the previous
iterate and jumps ``(n_g, 5, nx)`` — and iteration k is

* fine stage (parallel over windows n = k..n_g, ref/parareal.py:179-214):
  ``P(F(L(U^{k-1}_{n-1})))`` per window by ``pbgk_propagate`` (f never leaves
  the device, the lift and the projection are fused into the first and last
  sweeps), then one batched G launch that writes ``fine - G(U)`` = the jump;
* sequential correction (ref/parareal.py:217-248): one single-CTA kernel for
  the whole sweep ``U_n = G(U_{n-1}) + jump_n``, overshoot guard and the sup
  error.

With ``torch.distributed`` initialised (world > 1) the windows of each
iteration are dealt to ranks with ``work_distribution`` (the reference's
Appendix-A partition, ref/parareal.py:298-314); the only exchange is one
all-gather of the jumps (5*nx fp64 per window, plus a status word) per
iteration, after which every rank runs the cheap deterministic correction
itself, so snapshots are bitwise identical on all ranks and for any rank
count.  The distribution f never crosses NVLink.
"""

from __future__ import annotations

import ctypes
import math
import time
from dataclasses import dataclass
from typing import Callable, List, NamedTuple, Optional

import numpy as np
import torch

from . import runtime as rt
from .errors import ConfigurationError
from .fluid import FluidParams, fluid_batch, select_model
from .kinetic import KineticParams, propagate_window, propagate_windows, tau_constant
from .moments import MomentField

__all__ = ["PararealConfig", "ConvergenceRecord", "ParTrajectory", "WorkRange",
           "initial_coarse_sweep", "compute_jumps", "sequential_correction", "run_parareal",
           "fine_moment_chain", "work_distribution", "parareal_cost", "estimate_k_opt",
           "make_executor", "GpuBackend", "ShardedRun", "PipelinedRun"]


@dataclass
class PararealConfig:
    """k_max, tol, frozen-prefix switch, workers (ref/parareal.py:49-65).

    ``workers`` = parallel fine solvers, here GPU ranks: under
    torch.distributed it must equal the world size (or be 1); without it, a
    value > 1 runs on this process's GPU with a RuntimeWarning.
    """

    k_max: int
    tol: float
    use_frozen_prefix: bool = True
    workers: int = 1
    pipelined: bool = False  # extension: overlap G / correction with the fine windows

    def __post_init__(self):
        if self.k_max < 1:
            raise ConfigurationError("need k_max >= 1, got %r" % (self.k_max,))
        if not self.tol > 0.0:
            raise ConfigurationError("need tol > 0, got %r" % (self.tol,))
        if self.workers < 1:
            raise ConfigurationError("need workers >= 1, got %r" % (self.workers,))


@dataclass
class ConvergenceRecord:
    k: int
    error: float
    seconds: float


@dataclass
class ParTrajectory:
    """snapshots[n] ~ U(T^n); previous = iterate before the last correction;
    jumps[n-1] = fine-minus-coarse defect of window n (ref/parareal.py:74-88)."""

    snapshots: List[MomentField]
    previous: List[MomentField]
    jumps: List[MomentField]
    iteration: int = 0
    frozen_upto: int = 0


class WorkRange(NamedTuple):
    start: int
    end: int
    my_chunk: int
    size: int


def work_distribution(work: int, n_p: int, rank: int) -> WorkRange:
    """Contiguous 1-based inclusive window ranges (ref/parareal.py:298-314)."""
    if n_p < 1:
        raise ConfigurationError("need n_p >= 1, got %r" % (n_p,))
    if not 0 <= rank < n_p:
        raise ConfigurationError("need 0 <= rank < n_p, got rank %r" % (rank,))
    if work < 0:
        raise ConfigurationError("need work >= 0, got %r" % (work,))
    q, r = divmod(work, n_p)
    start = rank * q + min(r, rank) + 1
    end = (rank + 1) * q + min(r, rank + 1)
    return WorkRange(start, end, end - start, max(0, end - start + 1))


def parareal_cost(k, t_kin, t_fluid, t_lift, t_proj, n_g, n_p) -> float:
    """Modelled wall time of k iterations on n_p workers (ref/parareal.py:317-321)."""
    per = (t_lift + t_proj + t_kin + t_fluid) / n_p + t_fluid
    return t_fluid + n_g * k * per


def estimate_k_opt(t_kin, t_fluid, t_lift, t_proj, n_g, n_p) -> int:
    """Break-even iteration count, at least 1 (ref/parareal.py:324-333)."""
    per = (t_lift + t_proj + t_kin + t_fluid) / n_p + t_fluid
    return max(1, math.ceil((n_g * t_kin - t_fluid) / (n_g * per)))


class _DeviceExecutor:
    """What ``make_executor`` returns: the reference's process pool
    (ref/parareal.py:161-170) becomes the device itself -- the fine stage of
    an iteration is one batched launch sequence on this rank's GPU, and the
    windows are dealt to ranks (one per GPU) when torch.distributed is
    initialised."""

    def __init__(self, workers: int = 1):
        self.workers = workers

    def shutdown(self, wait: bool = True):
        return None


def make_executor(workers, disc, kinetic, fluid):
    """ref/parareal.py:161-170: the parallel stage of this implementation (see
    _DeviceExecutor); `workers` is checked against the rank count."""
    _check_workers(workers)
    return _DeviceExecutor(workers)


def _world() -> int:
    dist = torch.distributed
    return dist.get_world_size() if (dist.is_available() and dist.is_initialized()) else 1


def _check_workers(workers: int) -> None:
    """``workers`` (ref PararealConfig.workers) means parallel fine solvers:
    here GPU ranks.  Under torch.distributed it must match the world size;
    without it, a request for several workers runs on this process's GPU and
    says so (never silently)."""
    world = _world()
    if world > 1 and workers not in (1, world):
        raise ConfigurationError("workers=%d but torch.distributed runs %d ranks (one GPU each)"
                                 % (workers, world))
    if world == 1 and workers > 1:
        import warnings
        warnings.warn("workers=%d: the fine stage of every iteration runs batched on this "
                      "process's GPU; launch %d ranks with torchrun (one per GPU) to shard the "
                      "windows over GPUs" % (workers, workers), RuntimeWarning, stacklevel=3)


def _check_executor(executor) -> None:
    if executor is not None and not isinstance(executor, _DeviceExecutor):
        raise ConfigurationError(
            "compute_jumps: the fine stage runs on the GPU (windows dealt to torch.distributed "
            "ranks, one per GPU); a host executor (%s) cannot run it -- pass executor=None or "
            "the object make_executor() returns" % type(executor).__name__)


# ---------------------------------------------------------------------------
# backend: the per-rank numerical work of one iteration
# ---------------------------------------------------------------------------

class GpuBackend:
    """Window jumps, coarse sweeps and corrections through libpbgk.so."""

    def __init__(self, disc, kinetic: KineticParams, fluid: FluidParams, device=None):
        self.disc = disc
        self.kinetic = kinetic
        self.fluid = fluid
        self.ctx = rt.ctx_for(disc.phase, disc.bc, device)
        self.device = self.ctx.device
        self.nx = self.ctx.nx
        self.times = [float(t) for t in disc.time.coarse_times]
        self.force_dev = None
        if fluid.force is not None:
            self.force_dev, _ = rt.to_device_field(fluid.force, self.device, self.nx)
        self.t_kin = 0.0
        self.t_fluid = 0.0

    def empty(self, n):
        return torch.empty((n, 5, self.nx), dtype=torch.float64, device=self.device)

    def jumps(self, snaps: torch.Tensor, windows: List[int], out: torch.Tensor):
        """out[w] = P F L(snaps[n-1]) - G(snaps[n-1]) for n = windows[w]; status per window."""
        codes = []
        t = self.times
        src = None
        if windows:
            # a rank's windows are consecutive (work_distribution): their start
            # states are a view of the snapshots, no gather
            if windows == list(range(windows[0], windows[0] + len(windows))):
                src = snaps[windows[0] - 1:windows[0] - 1 + len(windows)]
            else:
                src = snaps[torch.tensor([n - 1 for n in windows], device=self.device)]
        if windows and tau_constant(self.kinetic.tau) is not None:
            # the whole fine stage in one library call (one host sync)
            tic = time.perf_counter()
            codes = propagate_windows(self.ctx, src, [t[n] - t[n - 1] for n in windows],
                                      self.disc.phase, self.kinetic, self.disc.time.dt_f,
                                      out[:len(windows)])
            self.t_kin = max(self.t_kin, (time.perf_counter() - tic) / len(windows))
        else:
            for w, n in enumerate(windows):
                tic = time.perf_counter()
                c = propagate_window(self.ctx, snaps[n - 1], t[n - 1], t[n], self.disc.phase,
                                     self.kinetic, self.disc.time.dt_f, out[w])
                self.t_kin = max(self.t_kin, time.perf_counter() - tic)
                codes.append(c)
        if windows:
            tic = time.perf_counter()
            gc = fluid_batch(self.ctx, src, out[:len(windows)], [t[n - 1] for n in windows],
                             [t[n] for n in windows], self.fluid, self.disc.time.dt_g,
                             minuend=out[:len(windows)], force_dev=self.force_dev)  # in place: each entry is read, then written, by one thread
            self.t_fluid = max(self.t_fluid, (time.perf_counter() - tic) / len(windows))
            if gc >= 0:
                # the failing window of the batch (unit = batch index)
                unit, _, _ = rt.decode(gc)
                codes[unit] = codes[unit] if codes[unit] >= 0 else ("G", gc)
        return codes

    def correct(self, snaps: torch.Tensor, old: torch.Tensor, jumps: torch.Tensor, start: int):
        e = ctypes.c_double(0.0)
        code = ctypes.c_longlong(-1)
        n_g = len(self.times) - 1
        tarr = (ctypes.c_double * (n_g + 1))(*self.times)
        select_model(self.ctx, self.fluid)
        rt._lib.check(self.ctx.lib.pbgk_parareal_correct(
            self.ctx.h, n_g, start, rt.ptr(snaps), rt.ptr(old), rt.ptr(jumps), tarr,
            float(self.disc.time.dt_g), float(self.fluid.cfl), rt.ptr(self.force_dev),
            rt.stream_handle(self.device), ctypes.byref(e), ctypes.byref(code)),
            "pbgk_parareal_correct")
        return e.value, code.value

    # -- pipelined mode (PipelinedRun): F on the current stream, the G jumps
    # and the correction on a side stream that trails the fine windows --------
    def fine_into(self, src: torch.Tensor, n: int, out: torch.Tensor) -> int:
        """out = P F L(src) of window n on the current stream; returns the status key."""
        t = self.times
        tic = time.perf_counter()
        c = propagate_window(self.ctx, src, t[n - 1], t[n], self.disc.phase, self.kinetic,
                             self.disc.time.dt_f, out)
        self.t_kin = max(self.t_kin, time.perf_counter() - tic)
        return c

    def side_begin(self, snaps: torch.Tensor) -> torch.Tensor:
        """Start an iteration: old = snaps (main stream); side stream state reset."""
        if getattr(self, "_side", None) is None:
            self._side = torch.cuda.Stream(self.device, priority=-1)
            self._dtimes = torch.tensor(self.times, dtype=torch.float64, device=self.device)
            n_g = len(self.times) - 1
            self._gstat = torch.empty(n_g, dtype=torch.int64, device=self.device)
            self._cstat = torch.empty(1, dtype=torch.int64, device=self.device)
            self._emax = torch.empty(1, dtype=torch.float64, device=self.device)
            self._ring = [None, None]
            self._free = [None, None]
        main = torch.cuda.current_stream(self.device)
        old = snaps.clone()
        self._side.wait_stream(main)
        with torch.cuda.stream(self._side):
            self._gstat.fill_(-1)
            self._cstat.fill_(-1)
            self._emax.zero_()
        rt._lib.check(self.ctx.lib.pbgk_set_grid_reserve(self.ctx.h, 1), "pbgk_set_grid_reserve")
        select_model(self.ctx, self.fluid)
        return old

    def round_slot(self, r: int, nslots: int) -> torch.Tensor:
        """Buffer for the fine outputs of round r (ring of two; waits until the
        side stream has consumed the round that used it before)."""
        i = r & 1
        buf = self._ring[i]
        if buf is None or buf.shape[0] < nslots:
            buf = self._ring[i] = torch.empty((nslots, 5, self.nx), dtype=torch.float64,
                                              device=self.device)
        if self._free[i] is not None:
            torch.cuda.current_stream(self.device).wait_event(self._free[i])
        return buf

    def side_round(self, r: int, fine: torch.Tensor, windows: List[int], snaps, old, jumps):
        """Side stream, after everything queued so far on the main stream:
        jumps[n-1] = fine[q] - G(old[n-1]) for each window n = windows[q], then
        the correction U_n = G(U_{n-1}) + jumps[n-1] over the round's windows."""
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream(self.device))
        side = self._side
        side.wait_event(ev)
        lib, h = self.ctx.lib, self.ctx.h
        sh = side.cuda_stream
        dt_g, cfl = float(self.disc.time.dt_g), float(self.fluid.cfl)
        force = rt.ptr(self.force_dev)
        dt = self._dtimes
        for q, n in enumerate(windows):
            rt._lib.check(lib.pbgk_fluid_propagate_async(
                h, 1, rt.ptr(old[n - 1]), rt.ptr(jumps[n - 1]), rt.ptr(fine[q]),
                rt.ptr(dt[n - 1:]), rt.ptr(dt[n:]), dt_g, cfl, force, ctypes.c_void_p(sh),
                rt.ptr(self._gstat[n - 1:])), "pbgk_fluid_propagate_async")
        if windows:
            rt._lib.check(lib.pbgk_parareal_correct_range(
                h, windows[0], windows[-1], rt.ptr(snaps), rt.ptr(old), rt.ptr(jumps), rt.ptr(dt),
                dt_g, cfl, force, ctypes.c_void_p(sh), rt.ptr(self._emax), rt.ptr(self._cstat)),
                "pbgk_parareal_correct_range")
        free = torch.cuda.Event()
        free.record(side)
        self._free[r & 1] = free

    def side_finish(self):
        """Wait for the side stream; (sup error, G-jump keys per window, correction key)."""
        self._side.synchronize()
        torch.cuda.current_stream(self.device).wait_stream(self._side)
        rt._lib.check(self.ctx.lib.pbgk_set_grid_reserve(self.ctx.h, 0), "pbgk_set_grid_reserve")
        return (float(self._emax.item()), self._gstat.cpu().tolist(), int(self._cstat.item()))


def _raise_window_status(status):
    """Raise the reference's exception for the first failing window."""
    for c in status:
        if isinstance(c, tuple):
            rt.raise_fluid(c[1])
        elif c >= 0:
            rt.raise_kinetic(c)


class ShardedRun:
    """One parareal run: device state + the (optional) rank decomposition."""

    def __init__(self, backend, group=None):
        self.b = backend
        self.n_g = len(backend.times) - 1
        self.group = group
        dist = torch.distributed
        self.world = dist.get_world_size(group) if (dist.is_available() and dist.is_initialized()) else 1
        self.rank = dist.get_rank(group) if self.world > 1 else 0

    # -- iteration 0 -------------------------------------------------------------
    def coarse_sweep(self, U0: torch.Tensor) -> torch.Tensor:
        snaps = self.b.empty(self.n_g + 1)
        snaps[0] = U0
        zero = torch.zeros((self.n_g, 5, self.b.nx), dtype=torch.float64, device=self.b.device)
        # U_n = G(U_{n-1}) + 0 is the coarse sweep (x + 0.0 == x)
        old = snaps.clone()
        _, code = self.b.correct(snaps, old, zero, 1)
        rt.raise_fluid(code)
        return snaps

    # -- parallel fine stage -------------------------------------------------------
    def jumps(self, snaps: torch.Tensor, jumps: torch.Tensor, start: int) -> None:
        work = self.n_g - start + 1
        if self.world == 1:
            windows = list(range(start, self.n_g + 1))
            # the jumps land in place; a failing window raises before anything reads them
            status = self.b.jumps(snaps, windows, jumps[start - 1:])
            _raise_window_status(status)
            return
        dist = torch.distributed
        chunk = -(-work // self.world)  # ceil
        r = work_distribution(work, self.world, self.rank)
        windows = list(range(start - 1 + r.start, start - 1 + r.end + 1))
        out = self.b.empty(max(chunk, 1))
        out.zero_()
        status = self.b.jumps(snaps, windows, out) if windows else []
        # status word per slot: -1 clean, kinetic key, or G key (+ 2**62 tag)
        words = torch.full((max(chunk, 1),), -1, dtype=torch.int64)
        for w, c in enumerate(status):
            if isinstance(c, tuple):
                words[w] = c[1] | (1 << 62)
            else:
                words[w] = c
        payload = torch.cat([out.reshape(-1), words.to(out.device).view(torch.float64)])
        flat = torch.empty(self.world * payload.numel(), dtype=torch.float64,
                           device=payload.device)
        dist.all_gather_into_tensor(flat, payload, group=self.group)
        gathered = flat.view(self.world, payload.numel())
        nj = max(chunk, 1) * 5 * self.b.nx
        all_status = []
        for q in range(self.world):
            rq = work_distribution(work, self.world, q)
            if rq.size == 0:
                continue
            blk = gathered[q, :nj].view(max(chunk, 1), 5, self.b.nx)
            wq = gathered[q, nj:].view(torch.int64).cpu()
            a = start - 1 + rq.start
            jumps[a - 1:a - 1 + rq.size] = blk[:rq.size]
            for w in range(rq.size):
                v = int(wq[w])
                all_status.append(("G", v & ~(1 << 62)) if v >= 0 and (v >> 62) & 1 else v)
        _raise_window_status(all_status)

    # -- sequential correction -------------------------------------------------------
    def correct(self, snaps, jumps, start):
        old = snaps.clone()
        err, code = self.b.correct(snaps, old, jumps, start)
        rt.raise_fluid(code)
        return old, err


class PipelinedRun(ShardedRun):
    """Iteration k with the coarse work trailing the fine windows (SURVEY.md
    8(f) rank 1).  Windows k..n_g are dealt CYCLICALLY to the ranks, one per
    rank per round; after each round the fine outputs are all-gathered and
    every rank queues, on a side stream, the round's G jumps and the
    correction of those windows -- which needs only the previous windows'
    corrections and the round's jumps -- while its next fine window runs.
    Only the last round's coarse work is exposed.  Every value is computed
    from the same inputs by the same kernels as in the phased ShardedRun, so
    trajectories are bitwise identical; no work is speculative (iteration
    k+1 starts after the correction of iteration k, as the reference's stop
    test requires).  Failure precedence is the phased one: the first failing
    window of the fine stage (F, then its G jump), then the correction.
    """

    def iterate(self, snaps: torch.Tensor, jumps: torch.Tensor, start: int):
        b = self.b
        N = self.world
        old = b.side_begin(snaps)
        windows = list(range(start, self.n_g + 1))
        rounds = [windows[i:i + N] for i in range(0, len(windows), N)]
        fstat = {}
        dist = torch.distributed
        for r, wr in enumerate(rounds):
            mine = wr[self.rank] if self.rank < len(wr) else None
            if N == 1:
                buf = b.round_slot(r, 1)
                fstat[mine] = b.fine_into(old[mine - 1], mine, buf[0])
                b.side_round(r, buf, wr, snaps, old, jumps)
                continue
            local = b.empty(1)
            code = -1
            if mine is not None:
                code = b.fine_into(old[mine - 1], mine, local[0])
            else:
                local.zero_()
            word = torch.tensor([code], dtype=torch.int64).to(local.device).view(torch.float64)
            payload = torch.cat([local.reshape(-1), word])
            flat = torch.empty(N * payload.numel(), dtype=torch.float64, device=payload.device)
            dist.all_gather_into_tensor(flat, payload, group=self.group)
            g = flat.view(N, payload.numel())
            nj = 5 * b.nx
            buf = b.round_slot(r, N)
            buf[:N].copy_(g[:, :nj].view(N, 5, b.nx))
            words = g[:, nj:].contiguous().view(torch.int64).cpu().tolist()
            for q, n in enumerate(wr):
                fstat[n] = words[q][0]
            b.side_round(r, buf, wr, snaps, old, jumps)
        err, gstat, cstat = b.side_finish()
        status = []
        for n in windows:
            c = fstat[n]
            if c < 0 and gstat[n - 1] >= 0:
                c = ("G", gstat[n - 1] & ~(0xFFFFFF << 40))  # unit: the batch index 0
            status.append(c)
        _raise_window_status(status)
        rt.raise_fluid(cstat)
        return old, err


def _stack(fields: List[MomentField], device) -> torch.Tensor:
    return torch.stack([rt.to_device_moments(U, device) for U in fields])


def _unstack(t: torch.Tensor) -> List[MomentField]:
    h = t.detach().cpu().numpy()
    return [MomentField(*rt.unpack_moments_np(h[i])) for i in range(h.shape[0])]


# ---------------------------------------------------------------------------
# reference-shaped API
# ---------------------------------------------------------------------------

def initial_coarse_sweep(U0: MomentField, disc, fluid: FluidParams) -> ParTrajectory:
    """Iteration 0: serial G over all windows (ref/parareal.py:109-120)."""
    run = ShardedRun(GpuBackend(disc, KineticParams(epsilon=1.0), fluid))
    snaps = _unstack(run.coarse_sweep(rt.to_device_moments(U0, run.b.device)))
    snaps[0] = U0.copy()
    zero = [MomentField(np.zeros_like(U0.rho), np.zeros_like(U0.u), np.zeros_like(U0.theta))
            for _ in range(disc.time.n_g)]
    return ParTrajectory(snaps, [s.copy() for s in snaps], zero)


def compute_jumps(traj: ParTrajectory, k: int, disc, kinetic, fluid,
                  use_frozen_prefix: bool = True, executor=None, timing=None) -> None:
    """Fill traj.jumps[k-1:] (or all) in place (ref/parareal.py:179-214)."""
    _check_executor(executor)
    start = k if use_frozen_prefix else 1
    n_g = disc.time.n_g
    if start > n_g:
        return
    b = GpuBackend(disc, kinetic, fluid)
    run = ShardedRun(b)
    snaps = _stack(traj.snapshots, b.device)
    jumps = b.empty(n_g)
    jumps.zero_()
    run.jumps(snaps, jumps, start)
    host = jumps.cpu().numpy()
    for n in range(start, n_g + 1):
        slot = traj.jumps[n - 1]
        rho, u, th = rt.unpack_moments_np(host[n - 1])
        slot.rho[:] = rho
        slot.u[:] = u
        slot.theta[:] = th
    if timing is not None:
        for key, val in (("t_lift", 0.0), ("t_kin", b.t_kin), ("t_proj", 0.0),
                         ("t_fluid", b.t_fluid)):
            timing[key] = max(timing.get(key, 0.0), val)


def sequential_correction(traj: ParTrajectory, k: int, disc, fluid: FluidParams,
                          use_frozen_prefix: bool = True) -> float:
    """U_n = G(U_{n-1}) + jump_n, overshoot guard, sup error (ref/parareal.py:217-248)."""
    start = k if use_frozen_prefix else 1
    b = GpuBackend(disc, KineticParams(epsilon=1.0), fluid)
    run = ShardedRun(b)
    snaps = _stack(traj.snapshots, b.device)
    jumps = _stack(traj.jumps, b.device)
    if start <= disc.time.n_g:
        _, err = run.correct(snaps, jumps, start)
    else:
        err = 0.0
    old = traj.snapshots
    new = _unstack(snaps)
    for n in range(0, min(start, len(new))):
        new[n] = old[n].copy()
    traj.previous = old
    traj.snapshots = new
    traj.iteration = k
    traj.frozen_upto = min(k, disc.time.n_g)
    return err


def run_parareal(U0: MomentField, config: PararealConfig, disc, kinetic: KineticParams,
                 fluid: FluidParams, sink: Optional[Callable] = None, timing: dict | None = None,
                 backend=None, group=None):
    """Full outer iteration on the device (ref/parareal.py:251-278).

    Returns ``(ParTrajectory, [ConvergenceRecord])``.  Under torch.distributed
    every rank must call it with the same arguments; all ranks return the same
    (bitwise) trajectory.
    """
    if group is None:
        _check_workers(config.workers)
    b = backend or GpuBackend(disc, kinetic, fluid)
    run = (PipelinedRun if config.pipelined else ShardedRun)(b, group)
    n_g = disc.time.n_g
    U0d = rt.to_device_moments(U0, b.device) if b.device.type == "cuda" else \
        torch.from_numpy(rt.pack_moments_np(U0.rho, U0.u, U0.theta))
    snaps = run.coarse_sweep(U0d)
    prev = snaps.clone()
    jumps = b.empty(n_g)
    jumps.zero_()
    records: List[ConvergenceRecord] = []
    it = 0
    for k in range(1, config.k_max + 1):
        tic = time.perf_counter()
        start = k if config.use_frozen_prefix else 1
        if start <= n_g and config.pipelined:
            prev, err = run.iterate(snaps, jumps, start)
        elif start <= n_g:
            run.jumps(snaps, jumps, start)
            prev, err = run.correct(snaps, jumps, start)
        else:
            prev, err = snaps.clone(), 0.0
        it = k
        rec = ConvergenceRecord(k, err, time.perf_counter() - tic)
        records.append(rec)
        if sink is not None:
            sink(rec)
        if err < config.tol:
            break
    if timing is not None:
        for key, val in (("t_lift", 0.0), ("t_kin", getattr(b, "t_kin", 0.0)), ("t_proj", 0.0),
                         ("t_fluid", getattr(b, "t_fluid", 0.0))):
            timing[key] = max(timing.get(key, 0.0), val)
    snap_l = _unstack(snaps)
    snap_l[0] = U0.copy()
    traj = ParTrajectory(snap_l, _unstack(prev), _unstack(jumps), it, min(it, n_g))
    traj.previous[0] = U0.copy()
    return traj, records


def fine_moment_chain(U0: MomentField, disc, kinetic: KineticParams) -> List[MomentField]:
    """Window-wise serial fine reference L -> F -> P (ref/parareal.py:281-295)."""
    ctx = rt.ctx_for(disc.phase, disc.bc)
    t = [float(x) for x in disc.time.coarse_times]
    cur = rt.to_device_moments(U0, ctx.device)
    out = [U0.copy()]
    for n in range(1, disc.time.n_g + 1):
        nxt = ctx.empty_moments()
        code = propagate_window(ctx, cur, t[n - 1], t[n], disc.phase, kinetic, disc.time.dt_f, nxt)
        rt.raise_kinetic(code)
        out.append(MomentField.from_packed(nxt))
        cur = nxt
    return out
