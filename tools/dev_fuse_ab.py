"""A/B of multi-step builds (development): PBGK_LIB=<so> python tests/dev_fuse_ab.py
-- default-level window times of the BASELINE shapes."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2502_02704_b200 as P
from paper_2502_02704_b200 import runtime as rt
from paper_2502_02704_b200.kinetic import propagate_window, stable_dt_kinetic

B = P.BoundaryKind
for nx, nv, vm, S, bc in ((2048, 64, 8.0, 32, B.OUTFLOW), (512, 48, 10.0, 32, B.OUTFLOW),
                         (1024, 32, 8.0, 26, B.PERIODIC)):
    grid = P.PhaseGrid(P.build_spatial_grid(0.0, 1.0, nx), P.build_velocity_grid(vm, (nv,) * 3))
    ctx = rt.ctx_for(grid, bc)
    kp = P.KineticParams(1e-2)
    x = grid.space.centers
    U = P.MomentField(np.where(x < 0.5, 1.0, 0.125), np.zeros((nx, 3)), np.where(x < 0.5, 1.0, 0.8))
    m0 = rt.to_device_moments(U, ctx.device)
    mo = ctx.empty_moments()
    t1 = S * stable_dt_kinetic(grid, kp) * 0.999
    best = 1e30
    for r in range(5):
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record()
        propagate_window(ctx, m0, 0.0, t1, grid, kp, None, mo)
        b.record(); torch.cuda.synchronize()
        if r: best = min(best, a.elapsed_time(b))
    print(f"{nx}x{nv}^3 x{S}: {best:7.2f} ms  {nx * nv ** 3 * S / best / 1e9:.3e} cell-upd/s", flush=True)
