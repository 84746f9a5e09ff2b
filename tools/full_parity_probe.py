"""Per-iteration parity of a full-size parareal run against its fixture
(tests/golden/full_*.npz): snapshot gap and error difference per iteration,
on the default multi-step path and on the one-step path.
usage: python tools/full_parity_probe.py cfg3a|cfg2_e1|cfg2_e0.1"""
import sys
import numpy as np
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import paper_2502_02704_b200 as P
from paper_2502_02704_b200 import runtime as rt
from paper_2502_02704_b200.configs import config
from helpers import moment_gap

name = sys.argv[1]
fx = np.load("tests/golden/full_%s.npz" % name)
w = config(3) if name == "cfg3a" else config(2, float(name.split("_e")[1]))
g = P.PhaseGrid(P.build_spatial_grid(w.x_min, w.x_max, w.nx), P.build_velocity_grid(w.v_max, w.nv))
bc = P.BoundaryKind(w.bc)
d = P.Discretization(g, P.build_time_grids(w.t_final, w.n_g, w.n_f), bc)
E = w.force()
kin, flu = P.KineticParams(w.eps, force=E), P.FluidParams(force=E)
U0 = P.project(P.lift(P.MomentField(*w.raw_moments()), g, bc=bc), g, bc=bc)
errs = list(fx["errors"])
for L in (-1, 0):
    with rt.ctx_for(g, bc).fusion_levels(L):
        for k in range(1, len(errs) + 1):
            traj, rec = P.run_parareal(U0, P.PararealConfig(k, 1e-300), d, kin, flu)
            gap = max(moment_gap((S.rho, S.u, S.theta), (fx["snap_rho"][n], fx["snap_u"][n], fx["snap_theta"][n]))
                      for n, S in enumerate(traj.snapshots)) if k == len(errs) else float("nan")
            print("fusion %d k %d error %.17g ref %.17g diff %.3e %s" % (
                L, k, rec[-1].error, errs[k - 1], abs(rec[-1].error - errs[k - 1]),
                "final snapshot gap %.3e" % gap if k == len(errs) else ""))
