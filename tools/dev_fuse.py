"""Multi-step path check + timing (development): window moments with
pbgk_set_fusion(0..3) against the one-step path, and their window times."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2502_02704_b200 as P
from paper_2502_02704_b200 import runtime as rt
from paper_2502_02704_b200.kinetic import propagate_window, stable_dt_kinetic


def run(nx, nv, vm, nsteps, bc, reps=3, quad="midpoint"):
    vg = P.build_velocity_grid(vm, nv) if quad == "midpoint" else P.build_velocity_grid(vm, nv, quadrature=quad)
    grid = P.PhaseGrid(P.build_spatial_grid(0.0, 1.0, nx), vg)
    ctx = rt.ctx_for(grid, bc)
    kp = P.KineticParams(1e-2)
    x = grid.space.centers
    rng = np.random.default_rng(1)
    U = P.MomentField(np.where(x < 0.5, 1.0, 0.125) * (1 + 0.01 * rng.random(nx)),
                      np.stack([0.1 * np.sin(2 * np.pi * x), 0.05 * np.cos(2 * np.pi * x), 0 * x], 1),
                      np.where(x < 0.5, 1.0, 0.8))
    m0 = rt.to_device_moments(U, ctx.device)
    t1 = nsteps * stable_dt_kinetic(grid, kp) * 0.97
    res = {}
    for L in (0, 2, 3, 4):
        ctx.lib.pbgk_set_fusion(ctx.h, L)
        mo = ctx.empty_moments()
        best = 1e30
        for r in range(reps + 1):
            torch.cuda.synchronize()
            a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
            a.record()
            code = propagate_window(ctx, m0, 0.0, t1, grid, kp, None, mo)
            b.record(); torch.cuda.synchronize()
            if r: best = min(best, a.elapsed_time(b))
        res[L] = (mo.cpu().numpy().copy(), best, code)
    ref = res[0][0]
    cells = nx * np.prod(nv) * nsteps
    line = f"{nx}x{nv[0]}^3 {bc.name[:4]} {quad[:4]} x{nsteps}:"
    for L in (0, 2, 3, 4):
        m, ms, code = res[L]
        err = max(np.max(np.abs(m[k] - ref[k])) / max(np.max(np.abs(ref[k])), 1e-300) for k in range(5))
        line += f" | L{L} {ms:7.2f} ms {cells / ms / 1e6:.3e}/s err {err:.1e} c{code}"
    print(line, flush=True)


B = P.BoundaryKind
if len(sys.argv) > 1 and sys.argv[1] == "quick":
    for bc in (B.ABSORBING, B.PERIODIC, B.OUTFLOW):
        run(64, (16,) * 3, 8.0, 13, bc)
        run(96, (8,) * 3, 8.0, 7, bc)
        run(64, (16,) * 3, 8.0, 13, bc, quad="trapezoid")
elif len(sys.argv) == 1:
    run(2048, (64,) * 3, 8.0, 32, B.OUTFLOW)
    run(512, (48,) * 3, 10.0, 32, B.OUTFLOW)
    run(1024, (32,) * 3, 8.0, 26, B.PERIODIC)
    run(256, (32,) * 3, 8.0, 100, B.PERIODIC)
    run(64, (16,) * 3, 8.0, 13, B.OUTFLOW)

if len(sys.argv) > 1 and sys.argv[1] == "prof":  # one 64^3 window at L = argv[2]
    grid = P.PhaseGrid(P.build_spatial_grid(0.0, 1.0, 2048), P.build_velocity_grid(8.0, (64,) * 3))
    ctx = rt.ctx_for(grid, B.OUTFLOW)
    ctx.lib.pbgk_set_fusion(ctx.h, int(sys.argv[2]))
    kp = P.KineticParams(1e-2)
    x = grid.space.centers
    U = P.MomentField(np.where(x < 0.5, 1.0, 0.125), np.zeros((2048, 3)), np.where(x < 0.5, 1.0, 0.8))
    m0 = rt.to_device_moments(U, ctx.device)
    mo = ctx.empty_moments()
    propagate_window(ctx, m0, 0.0, 8 * stable_dt_kinetic(grid, kp), grid, kp, None, mo)
    torch.cuda.synchronize()
    print("done")
