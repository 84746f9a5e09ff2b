"""Development: time of the batched moment recursion alone (config 0 / config 1 shapes)."""
import sys, time
import numpy as np, torch
sys.path.insert(0, ".")
import paper_2502_02704_b200 as P
from paper_2502_02704_b200 import runtime as rt, _lib
from paper_2502_02704_b200.kinetic import propagate_windows, stable_dt_kinetic
for nx, nv, nwin, steps in ((64, (16,) * 3, 8, 13), (256, (32,) * 3, 1, 200)):
    grid = P.PhaseGrid(P.build_spatial_grid(0.0, 1.0, nx), P.build_velocity_grid(8.0, nv))
    ctx = rt.ctx_for(grid, P.BoundaryKind.PERIODIC)
    kp = P.KineticParams(1e-2)
    x = grid.space.centers
    U = P.MomentField(1.0 + 0.3 * np.sin(2 * np.pi * x), np.zeros((nx, 3)), np.ones(nx))
    m0 = torch.stack([rt.to_device_moments(U, ctx.device)] * nwin)
    out = ctx.empty_moments(nwin)
    span = (steps - 0.5) * stable_dt_kinetic(grid, kp)
    lib = _lib.load()
    for r in range(4):
        lib.pbgk_profile_enable(ctx.h, 1)
        codes = propagate_windows(ctx, m0, [span] * nwin, grid, kp, None, out)
        torch.cuda.synchronize()
        prof = _lib.Profile(); lib.pbgk_profile_read(ctx.h, prof)
        if r:
            print("nx %d nv %d windows %d steps %d: recursion %.1f us (%.2f us per step)  passes %.1f us" % (
                nx, nv[0], nwin, steps, prof.marg_ms * 1e3, prof.marg_ms * 1e3 / steps, prof.msweep_ms * 1e3))
