"""CPU baseline timing of the oracle port (TEST / BENCH INFRASTRUCTURE ONLY).

Used by ``bench.py`` for the ``cpu_baseline`` object and the
``--impl reference`` arm: the reference algorithm -- this numpy restatement
of ``parabgk``, bit-identical to the reference (tests/test_oracle.py) -- is
timed on the host's cores the way the reference itself runs it:

* parareal workloads: the reference parallelises the fine stage over windows
  with a process pool (ref/parareal.py:145-170, 200-211), one window per
  task, each task the whole ``_window_jump`` -- lift, F over the window, P and
  G (ref/parareal.py:123-142).  Here every core runs one such window on an
  x-slab of the workload (same velocity grid, dx, dt, boundary, window step
  count; the slab centred on the Sod interface): a full window at config 4
  needs ~26 GB and ~15 min per core, the slab keeps one bench step to
  seconds.  Cell-updates are counted for the fine steps only.
* fine-only workloads (config 1): ONE core -- the reference has no
  intra-propagator parallelism -- advancing an x-slab of the
  periodic wave for a bounded number of the workload's fine steps.
"""

from __future__ import annotations

import multiprocessing as mp
import os
import time
from dataclasses import replace

import numpy as np

from . import bgk as O


def _limit_threads():
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    try:
        from threadpoolctl import threadpool_limits
        threadpool_limits(1)
    except Exception:
        pass


def slab_workload(w, nx_slab: int):
    """The workload restricted to nx_slab cells (same dx), centred at x = 0.5."""
    dx = (w.x_max - w.x_min) / w.nx
    nx_slab = min(nx_slab, w.nx)
    x0 = w.x_min + dx * ((w.nx - nx_slab) // 2)
    return replace(w, nx=nx_slab, x_min=x0, x_max=x0 + nx_slab * dx)


def _problem(ws):
    mesh = O.Mesh(ws.x_min, ws.x_max, ws.nx, ws.v_max, ws.nv, quadrature=ws.quadrature)
    prob = O.Problem(mesh, ws.t_final, ws.n_g, ws.n_f, ws.eps, ws.bc, ws.force(), alpha=ws.alpha,
                     g_model=ws.g_model)
    return mesh, prob


def _window_worker(ws):
    """One ``_window_jump`` of window 1 (ref/parareal.py:123-142) on the slab."""
    _limit_threads()
    mesh, prob = _problem(ws)
    U = O.project(O.lift(*ws.raw_moments(), mesh), mesh)
    tic = time.perf_counter()
    O.window_jump(prob, U, 1)
    return time.perf_counter() - tic


def _fine_worker(args):
    ws, steps = args
    _limit_threads()
    mesh, prob = _problem(ws)
    f0 = O.lift(*ws.raw_moments(), mesh)
    cap = O.scaled_cap(mesh, 0.5, ws.force(), ws.eps, ws.alpha)
    tic = time.perf_counter()
    O.fine_propagate(f0, 0.0, (steps - 0.5) * cap, mesh, ws.eps, ws.bc, ws.force(), alpha=ws.alpha)
    return time.perf_counter() - tic


def window_rate(w, nx_slab: int, workers: int | None = None) -> dict:
    """Cell-updates/s of `workers` concurrent full-window jumps on x-slabs."""
    workers = workers or len(os.sched_getaffinity(0))
    ws = slab_workload(w, nx_slab)
    steps = w.window_steps()
    cells = ws.nx * int(np.prod(w.nv))
    ctx = mp.get_context("fork")
    with ctx.Pool(workers) as pool:
        secs = pool.map(_window_worker, [ws] * workers)
    total = workers * cells * steps
    return {"value": total / max(secs), "cores": workers, "seconds": float(max(secs)),
            "cell_updates": total,
            "sample": "%d concurrent processes (the reference's window pool, ref/parareal.py:"
                      "161-170), each one whole window jump (lift, %d fine steps, project, G; "
                      "ref/parareal.py:123-142) on a %d-cell x-slab of %s (%d cells x %s)"
                      % (workers, steps, ws.nx, w.name, w.nx, "x".join(map(str, w.nv)))}


def fine_rate(w, nx_slab: int, steps: int) -> dict:
    """Cell-updates/s of one core advancing an x-slab `steps` fine steps."""
    ws = slab_workload(w, nx_slab)
    cells = ws.nx * int(np.prod(w.nv))
    ctx = mp.get_context("fork")
    with ctx.Pool(1) as pool:
        sec = pool.map(_fine_worker, [(ws, steps)])[0]
    total = cells * steps
    return {"value": total / sec, "cores": 1, "seconds": sec, "cell_updates": total,
            "sample": "1 process (the reference cannot split one propagation, SPEC:262): %d fine "
                      "steps of propagate_kinetic on a %d-cell x-slab of %s (%d cells x %s)"
                      % (steps, ws.nx, w.name, w.nx, "x".join(map(str, w.nv)))}


def workload_rate(w, budget_cells: float = 1.4e8) -> dict:
    """The CPU baseline of a BASELINE workload: about `budget_cells`
    cell-updates per core (a few seconds of numpy)."""
    plane = int(np.prod(w.nv))
    if w.mode == "parareal":
        steps = w.window_steps()
        nx_slab = max(4, int(budget_cells // (plane * steps)))
        return window_rate(w, nx_slab)
    steps = 40
    nx_slab = max(4, int(budget_cells // (plane * steps)))
    return fine_rate(w, nx_slab, steps)
