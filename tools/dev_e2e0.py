"""Development: median wall time of run_parareal(k_max=1) on config 0 (the bench's e2e leg)."""
import sys, time
import numpy as np, torch
sys.path.insert(0, ".")
import paper_2502_02704_b200 as P
from paper_2502_02704_b200.configs import config
w = config(0)
g = P.PhaseGrid(P.build_spatial_grid(w.x_min, w.x_max, w.nx), P.build_velocity_grid(w.v_max, w.nv))
bc = P.BoundaryKind(w.bc)
d = P.Discretization(g, P.build_time_grids(w.t_final, w.n_g, w.n_f), bc)
U0 = P.project(P.lift(P.MomentField(*w.raw_moments()), g, bc=bc), g, bc=bc)
cfg = P.PararealConfig(k_max=1, tol=1e-300)
ts = []
for r in range(40):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    traj, rec = P.run_parareal(U0, cfg, d, P.KineticParams(w.eps), P.FluidParams())
    torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
ts = np.array(ts[5:]) * 1e6
print("run_parareal(k_max=1) config 0: median %.0f us  min %.0f  p90 %.0f" % (np.median(ts), ts.min(), np.percentile(ts, 90)))
