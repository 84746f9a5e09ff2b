"""Same-box A/B of library builds (development): PBGK_LIB=<so> python tests/dev_abrev.py.
Times pbgk_propagate directly (no profiling events), window from moments."""
import ctypes, sys
import numpy as np, torch
sys.path.insert(0, ".")
import paper_2502_02704_b200 as P
from paper_2502_02704_b200 import runtime as rt
from paper_2502_02704_b200.kinetic import fine_schedule, stable_dt_kinetic
for nx, nv, S, vm in ((2048, 64, 32, 8.0), (512, 48, 32, 10.0), (1024, 32, 26, 8.0), (256, 32, 200, 8.0)):
    g = P.PhaseGrid(P.build_spatial_grid(0, 1, nx), P.build_velocity_grid(vm, nv))
    kp = P.KineticParams(1e-2)
    ctx = rt.ctx_for(g, P.BoundaryKind.OUTFLOW)
    x = g.space.centers
    U = P.MomentField(np.where(x < 0.5, 1.0, 0.125), np.zeros((nx, 3)), np.where(x < 0.5, 1.0, 0.8))
    m0 = rt.to_device_moments(U, ctx.device)
    mo = ctx.empty_moments()
    dts = fine_schedule(S * stable_dt_kinetic(g, kp), stable_dt_kinetic(g, kp))
    arr = (ctypes.c_double * len(dts))(*dts)
    code = ctypes.c_longlong(-1)
    f1, f2 = ctx.f_scratch(0), ctx.f_scratch(1)
    best = 1e9
    for r in range(5):
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record()
        ctx.lib.pbgk_propagate(ctx.h, None, rt.ptr(m0), rt.ptr(f2), rt.ptr(f1), 0, rt.ptr(mo), len(dts),
                               arr, 1e-2, 1.0, None, 0.0, rt.stream_handle(ctx.device), ctypes.byref(code))
        b.record(); torch.cuda.synchronize()
        if r: best = min(best, a.elapsed_time(b))
    print(f"{nx}x{nv}^3 x{len(dts)}: {best:8.3f} ms  {16*nx*nv**3*len(dts)/best/1e6:6.0f} GB/s")
