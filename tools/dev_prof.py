"""Profiling driver (development): one fine window on a chosen config.

usage: python tests/dev_prof.py CFG [NSTEPS]; CFG in 1, 2, 3 (periodic, no field),
3a (periodic, E = 0.5 sin 2 pi x: the field sweep), 4."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2502_02704_b200 as P
from paper_2502_02704_b200 import runtime as rt
from paper_2502_02704_b200.kinetic import propagate_window, stable_dt_kinetic

cfg = sys.argv[1] if len(sys.argv) > 1 else "4"
nsteps = int(sys.argv[2]) if len(sys.argv) > 2 else 6
nx, nv, vm, per = {"4": (2048, (64,) * 3, 8.0, False), "2": (512, (48,) * 3, 10.0, False),
                   "3": (1024, (32,) * 3, 8.0, True), "3a": (1024, (32,) * 3, 8.0, True),
                   "1": (256, (32,) * 3, 8.0, True)}[cfg]
grid = P.PhaseGrid(P.build_spatial_grid(0.0, 1.0, nx), P.build_velocity_grid(vm, nv))
ctx = rt.ctx_for(grid, P.BoundaryKind.PERIODIC if per else P.BoundaryKind.ABSORBING)
x = grid.space.centers
force = 0.5 * np.sin(2 * np.pi * x) if cfg == "3a" else None
kp = P.KineticParams(1e-2, force=force)
U = P.MomentField(np.where(x < 0.5, 1.0, 0.125), np.zeros((nx, 3)), np.where(x < 0.5, 1.0, 0.8))
m0 = rt.to_device_moments(U, ctx.device)
mo = ctx.empty_moments()
code = propagate_window(ctx, m0, 0.0, nsteps * stable_dt_kinetic(grid, kp), grid, kp, None, mo)
torch.cuda.synchronize()
print("done", code, ctx.describe())
