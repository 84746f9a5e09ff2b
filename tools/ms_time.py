"""Development timing of one config-4 window (32 steps) on the multi-step path:
python tools/ms_time.py [reps]; env knobs of capi.cu select the variant."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2502_02704_b200 as P
from paper_2502_02704_b200 import runtime as rt, _lib
from paper_2502_02704_b200.kinetic import propagate_window, stable_dt_kinetic

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
cfg = sys.argv[2] if len(sys.argv) > 2 else "4"
nx, nv, vm = {"4": (2048, (64,) * 3, 8.0), "2": (512, (48,) * 3, 10.0), "1": (256, (32,) * 3, 8.0)}[cfg]
grid = P.PhaseGrid(P.build_spatial_grid(0.0, 1.0, nx), P.build_velocity_grid(vm, nv))
ctx = rt.ctx_for(grid, P.BoundaryKind.OUTFLOW)
x = grid.space.centers
kp = P.KineticParams(1e-2)
U = P.MomentField(np.where(x < 0.5, 1.0, 0.125), np.zeros((nx, 3)), np.where(x < 0.5, 1.0, 0.8))
m0 = rt.to_device_moments(U, ctx.device)
mo = ctx.empty_moments()
span = 32 * stable_dt_kinetic(grid, kp)
lib = _lib.load()
for r in range(reps + 1):
    lib.pbgk_profile_enable(ctx.h, 1)
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record()
    code = propagate_window(ctx, m0, 0.0, span, grid, kp, None, mo)
    b.record(); torch.cuda.synchronize()
    prof = _lib.Profile(); lib.pbgk_profile_read(ctx.h, prof)
    if r:
        print("window %.3f ms  passes %d: %.3f ms (%.3f per pass, %.2f TB/s)  rec %.3f ms  fin %.3f ms  code %d" % (
            a.elapsed_time(b), prof.msweeps, prof.msweep_ms, prof.msweep_ms / max(prof.msweeps, 1),
            prof.msweep_bytes / max(prof.msweep_ms, 1e-9) / 1e9, prof.marg_ms, prof.finalize_ms, code))
