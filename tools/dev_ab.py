"""A/B timing of library variants (development only): PBGK_LIB=<so> python tests/dev_ab.py.

Prints whole-window time and the profiled sweep / finalize split."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2502_02704_b200 as P
from paper_2502_02704_b200 import runtime as rt, _lib
from paper_2502_02704_b200.kinetic import propagate_window, stable_dt_kinetic


def run(nx, nv, vm, nsteps, periodic, reps=3, field=False, scheme="upwind"):
    grid = P.PhaseGrid(P.build_spatial_grid(0.0, 1.0, nx), P.build_velocity_grid(vm, nv))
    bc = P.BoundaryKind.PERIODIC if periodic else P.BoundaryKind.OUTFLOW
    ctx = rt.ctx_for(grid, bc)
    E = 0.5 * np.sin(2 * np.pi * grid.space.centers) if field else None
    kp = P.KineticParams(1e-2, force=E, scheme=scheme)
    x = grid.space.centers
    U = P.MomentField(np.where(x < 0.5, 1.0, 0.125), np.zeros((nx, 3)), np.where(x < 0.5, 1.0, 0.8))
    m0 = rt.to_device_moments(U, ctx.device)
    mo = ctx.empty_moments()
    t1 = nsteps * stable_dt_kinetic(grid, kp)
    lib = _lib.load()
    best = 1e30
    for r in range(reps + 1):
        if r == reps:
            lib.pbgk_profile_enable(ctx.h, 1)
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record()
        propagate_window(ctx, m0, 0.0, t1, grid, kp, None, mo)
        b.record(); torch.cuda.synchronize()
        if r and r < reps:
            best = min(best, a.elapsed_time(b))
    prof = _lib.Profile()
    lib.pbgk_profile_read(ctx.h, prof)
    lib.pbgk_profile_enable(ctx.h, 0)
    cells = nx * np.prod(nv) * nsteps
    print(f"{nx}x{nv[0]}^3{' E' if field else ''}{' M' if scheme == 'muscl' else ''} x{nsteps}: {best:7.2f} ms {16*cells/best/1e6:6.0f} GB/s | sweep "
          f"{prof.sweep_bytes/prof.sweep_ms/1e6:6.0f} GB/s fin {prof.finalize_ms/max(prof.finalizes,1)*1e3:6.1f} us"
          f" ({prof.finalize_ms/(prof.sweep_ms+prof.finalize_ms):.3f})")


if len(sys.argv) > 1 and sys.argv[1] == "one":  # one case: nx nv steps [field]
    nx, nv, st = int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
    run(nx, (nv,) * 3, 10.0 if nv == 48 else 8.0, st, True, field=len(sys.argv) > 5)
elif len(sys.argv) > 1 and sys.argv[1] == "muscl":
    for sch in ("upwind", "muscl"):
        run(2048, (64, 64, 64), 8.0, 16, False, scheme=sch)
        run(512, (48, 48, 48), 10.0, 16, False, scheme=sch)
        run(1024, (32, 32, 32), 8.0, 26, True, scheme=sch)
elif len(sys.argv) > 1 and sys.argv[1] == "field":
    run(1024, (32, 32, 32), 8.0, 26, True)
    run(1024, (32, 32, 32), 8.0, 26, True, field=True)
    run(2048, (64, 64, 64), 8.0, 8, True, field=True)
    run(512, (48, 48, 48), 10.0, 16, True, field=True)
else:
    run(2048, (64, 64, 64), 8.0, 32, False)
    run(512, (48, 48, 48), 10.0, 32, False)
    run(1024, (32, 32, 32), 8.0, 26, True)
