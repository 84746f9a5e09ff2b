"""CPU baseline timing of the oracle port (TEST / BENCH INFRASTRUCTURE ONLY).

Used by ``bench.py`` for the ``cpu_baseline`` object and the
``--impl reference`` arm: the reference algorithm (this numpy restatement of
ref/kinetic.py, bit-identical to the reference) is timed on the host's cores,
one process per core, each advancing an independent x-slab of the workload
(same velocity grid, same dx, so the same per-cell work) for a few fine steps.
The reference itself parallelises only over windows (process pool,
ref/parareal.py:145-170) and a full window of the large configs needs ~26 GB
and ~15 min per core, so a bounded slab sample is what fits a bench run.
"""

from __future__ import annotations

import multiprocessing as mp
import os
import time

import numpy as np

from . import bgk as O


def _slab_worker(args):
    nx_slab, dx, nv, v_max, eps, steps, alpha = args
    try:
        from threadpoolctl import threadpool_limits
        threadpool_limits(1)
    except Exception:
        pass
    mesh = O.Mesh(0.0, nx_slab * dx, nx_slab, v_max, nv)
    x = mesh.xc / (nx_slab * dx)
    rho = np.where(x < 0.5, 1.0, 0.125)
    u = np.zeros((nx_slab, 3))
    theta = np.where(x < 0.5, 1.0, 0.8)
    f = O.lift(rho, u, theta, mesh)
    cap = O.scaled_cap(mesh, 0.5, None, eps, alpha)
    tic = time.perf_counter()
    O.fine_propagate(f, 0.0, steps * cap, mesh, eps, True, alpha=alpha)
    return time.perf_counter() - tic


def slab_rate(nx_full: int, nv, v_max: float, eps: float, nx_slab: int, steps: int,
              workers: int | None = None, alpha: int = 0) -> dict:
    """Aggregate cell-updates/s of `workers` concurrent oracle slab solves."""
    workers = workers or len(os.sched_getaffinity(0))
    dx = 1.0 / nx_full
    cells = nx_slab * int(np.prod(nv))
    ctx = mp.get_context("fork")
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    tic = time.perf_counter()
    with ctx.Pool(workers) as pool:
        secs = pool.map(_slab_worker, [(nx_slab, dx, tuple(nv), v_max, eps, steps, alpha)] * workers)
    wall = time.perf_counter() - tic
    total = workers * cells * steps
    # rate over the slowest worker's compute time (pool start-up excluded)
    return {"value": total / max(secs), "cores": workers, "wall_s": wall,
            "per_core_s": float(np.mean(secs)), "cell_updates": total,
            "sample": "%d independent x-slabs (%d cells x %s) x %d fine steps of the oracle F, "
                      "one process per core" % (workers, nx_slab, "x".join(map(str, nv)), steps)}
