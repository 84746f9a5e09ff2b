"""PDL A/B on config 1 (no profiling events in the timed region)."""
import sys, numpy as np, torch
sys.path.insert(0, ".")
import paper_2502_02704_b200 as P
from paper_2502_02704_b200 import runtime as rt
from paper_2502_02704_b200.kinetic import _run_schedule, fine_schedule, stable_dt_kinetic
for nx, nv, T in ((256, 32, 0.2), (1024, 32, 26 * 6.1e-5), (2048, 64, 32 * 3.0517578125e-5)):
    g = P.PhaseGrid(P.build_spatial_grid(0, 1, nx), P.build_velocity_grid(8.0, nv))
    kp = P.KineticParams(1e-3)
    ctx = rt.ctx_for(g, P.BoundaryKind.PERIODIC)
    x = g.space.centers
    f0 = P.lift(P.MomentField(1 + 0.5 * np.sin(2 * np.pi * x), np.zeros((nx, 3)), np.ones(nx)), g).device_tensor(ctx.device)
    dts = fine_schedule(T, stable_dt_kinetic(g, kp))
    out = ctx.empty_f()
    best = 1e9
    for r in range(4):
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); _run_schedule(ctx, f0, None, dts, kp, out); b.record(); torch.cuda.synchronize()
        if r: best = min(best, a.elapsed_time(b))
    print(f"{nx}x{nv}^3 {len(dts)} steps: {best:.2f} ms  {best/len(dts)*1e3:.1f} us/step")
