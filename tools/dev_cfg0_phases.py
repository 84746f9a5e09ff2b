"""Development: host-side phase times of one config-0 parareal iteration."""
import sys, time
import torch
sys.path.insert(0, ".")
import paper_2502_02704_b200 as P
from paper_2502_02704_b200 import runtime as rt
from paper_2502_02704_b200.configs import config
from paper_2502_02704_b200.parareal import GpuBackend, ShardedRun
w = config(0)
g = P.PhaseGrid(P.build_spatial_grid(w.x_min, w.x_max, w.nx), P.build_velocity_grid(w.v_max, w.nv))
bc = P.BoundaryKind(w.bc)
d = P.Discretization(g, P.build_time_grids(w.t_final, w.n_g, w.n_f), bc)
U0 = P.project(P.lift(P.MomentField(*w.raw_moments()), g, bc=bc), g, bc=bc)
b = GpuBackend(d, P.KineticParams(w.eps), P.FluidParams())
run = ShardedRun(b)
snaps = run.coarse_sweep(rt.to_device_moments(U0, b.device))
jumps = b.empty(w.n_g); jumps.zero_()
def sync(): torch.cuda.synchronize()
for rep in range(6):
    sync(); t0 = time.perf_counter()
    run.jumps(snaps.clone(), jumps, 1); sync(); t1 = time.perf_counter()
    run.correct(snaps.clone(), jumps, 1); sync(); t2 = time.perf_counter()
    # inside jumps
    windows = list(range(1, w.n_g + 1)); out = b.empty(len(windows))
    from paper_2502_02704_b200.kinetic import propagate_windows
    from paper_2502_02704_b200.fluid import fluid_batch
    t = b.times
    sync(); a0 = time.perf_counter()
    src = snaps[0:w.n_g]
    codes = propagate_windows(b.ctx, src, [t[n] - t[n - 1] for n in windows], d.phase, b.kinetic, d.time.dt_f, out)
    a1 = time.perf_counter()
    gc = fluid_batch(b.ctx, src, out, [t[n - 1] for n in windows], [t[n] for n in windows], b.fluid, d.time.dt_g, minuend=out, force_dev=None)
    a2 = time.perf_counter()
    if rep:
        print("jumps %.0f us  correct %.0f us | propagate_windows %.0f us  fluid_batch %.0f us" % (
            (t1 - t0) * 1e6, (t2 - t1) * 1e6, (a1 - a0) * 1e6, (a2 - a1) * 1e6))
