"""Where config 1's end-to-end time goes (development): propagate_kinetic with
a pinned host f vs a device f, and the bare copies."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
import bench
from paper_2502_02704_b200.configs import config

w = config(1)
P, phase, bc, disc, kin, flu = bench.build_problem(w)
f_init = P.lift(P.MomentField(*w.raw_moments()), phase, bc=bc)
dev = torch.device("cuda", 0)
host = f_init.values.copy()
pinned = torch.from_numpy(host).pin_memory()


def tm(name, fn, reps=4):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    print("%-40s %8.2f ms" % (name, 1e3 * np.median(ts)))


fd = pinned.to(dev)
tm("h2d pinned", lambda: pinned.to(dev, non_blocking=True))
tm("d2h to pinned", lambda: torch.empty(pinned.shape, dtype=torch.float64, pin_memory=True).copy_(fd))
tm("propagate device f", lambda: P.propagate_kinetic(P.Distribution(fd), 0.0, w.t_final, phase, kin, bc))
tm("propagate pinned host f (values)", lambda: P.propagate_kinetic(P.Distribution(pinned), 0.0, w.t_final, phase, kin, bc).values)
tm("propagate numpy host f (values)", lambda: P.propagate_kinetic(P.Distribution(host), 0.0, w.t_final, phase, kin, bc).values)
import cProfile, pstats
pr = cProfile.Profile()
pr.enable()
P.propagate_kinetic(P.Distribution(pinned), 0.0, w.t_final, phase, kin, bc).values
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(18)
