"""Time the coarse work of one parareal iteration (batched jump G and the
sequential correction) for configs 4 and 3b (development)."""
import sys, time, torch
sys.path.insert(0, ".")
import bench
import paper_2502_02704_b200 as P
from paper_2502_02704_b200 import runtime as rt
from paper_2502_02704_b200.configs import config
from paper_2502_02704_b200.fluid import fluid_batch
from paper_2502_02704_b200.parareal import GpuBackend, ShardedRun
for idx in sys.argv[1:] or ["4", "3b"]:
    w = config(idx)
    _, phase, bc, disc, kin, flu = bench.build_problem(w)
    U0 = P.project(P.lift(P.MomentField(*w.raw_moments()), phase, bc=bc), phase, bc=bc)
    b = GpuBackend(disc, kin, flu)
    run = ShardedRun(b)
    snaps = run.coarse_sweep(rt.to_device_moments(U0, b.device))
    jumps = b.empty(w.n_g); jumps.zero_()
    for rep in range(3):
        s = snaps.clone()
        torch.cuda.synchronize(); t0 = time.perf_counter()
        run.correct(s, jumps, 1)
        torch.cuda.synchronize(); t1 = time.perf_counter()
        src = snaps[:w.n_g].contiguous(); out = b.empty(w.n_g)
        fluid_batch(b.ctx, src, out, b.times[:-1], b.times[1:], flu, disc.time.dt_g, minuend=out.clone(),
                    force_dev=b.force_dev)
        torch.cuda.synchronize(); t2 = time.perf_counter()
    print(f"{w.name}: correction {1e3*(t1-t0):.2f} ms, batched G ({w.n_g} windows) {1e3*(t2-t1):.2f} ms")
