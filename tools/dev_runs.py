"""Development: full parareal runs of the BASELINE configs on the GPU."""
import sys, time
from dataclasses import replace
sys.path.insert(0, ".")
import numpy as np
import bench
from paper_2502_02704_b200.configs import config
import paper_2502_02704_b200 as P

for idx, eps, bc in [(2, 1.0, None), (2, 0.1, None)]:
    w = config(idx, eps)
    if bc == "absorbing":
        w = replace(w, outflow=False)
    P_, phase, bcx, disc, kin, flu = bench.build_problem(w)
    U0 = P.project(P.lift(P.MomentField(*w.raw_moments()), phase, bc=bcx), phase, bc=bcx)
    tic = time.time()
    try:
        traj, rec = P.run_parareal(U0, P.PararealConfig(w.k_max, w.tol), disc, kin, flu)
        print(w.name, w.bc, "eps", w.eps, "K", len(rec), ["%.3e" % r.error for r in rec], "%.2fs" % (time.time() - tic), flush=True)
    except P.SolverError as e:
        print(w.name, w.bc, "eps", w.eps, type(e).__name__, getattr(e, "slice_index", None), getattr(e, "step", None), "%.2fs" % (time.time() - tic), flush=True)
