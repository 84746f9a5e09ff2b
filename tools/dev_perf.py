"""Ad-hoc perf probe (development only, not collected by pytest)."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2502_02704_b200 as P
from paper_2502_02704_b200 import runtime as rt
from paper_2502_02704_b200.kinetic import propagate_window, fine_schedule, stable_dt_kinetic

def run(nx, nv, vm, nsteps, periodic, reps=3):
    grid = P.PhaseGrid(P.build_spatial_grid(0.0, 1.0, nx), P.build_velocity_grid(vm, nv))
    bc = P.BoundaryKind.PERIODIC if periodic else P.BoundaryKind.ABSORBING
    ctx = rt.ctx_for(grid, bc)
    kp = P.KineticParams(1e-2)
    cap = stable_dt_kinetic(grid, kp)
    x = grid.space.centers
    U = P.MomentField(np.where(x < 0.5, 1.0, 0.125), np.zeros((nx, 3)), np.where(x < 0.5, 1.0, 0.8))
    m0 = rt.to_device_moments(U, ctx.device)
    mo = ctx.empty_moments()
    t1 = nsteps * cap
    for r in range(reps + 1):
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record()
        code = propagate_window(ctx, m0, 0.0, t1, grid, kp, None, mo)
        b.record(); torch.cuda.synchronize()
        ms = a.elapsed_time(b)
        cells = nx * np.prod(nv) * nsteps
        if r > 0:
            print(f"{nx}x{nv} steps={nsteps}: {ms:.2f} ms  {cells/ms*1e3:.3e} cell-upd/s  {16*cells/ms*1e3/1e9:.0f} GB/s  code={code}")

run(2048, (64,64,64), 8.0, 32, False)
run(512, (48,48,48), 10.0, 32, False)
run(1024, (32,32,32), 8.0, 26, True)
run(256, (32,32,32), 8.0, 100, True)
