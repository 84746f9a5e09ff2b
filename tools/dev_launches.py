"""Launch-list driver for ncu (development): one short parareal iteration of
config 4 restricted to 2 windows, so ncu's per-launch list stays small."""
import sys
from dataclasses import replace
sys.path.insert(0, ".")
import bench
import paper_2502_02704_b200 as P
from paper_2502_02704_b200.configs import config

w = replace(config(4), n_g=64)
P_, phase, bc, disc, kin, flu = bench.build_problem(w)
U0 = P.project(P.lift(P.MomentField(*w.raw_moments()), phase, bc=bc), phase, bc=bc)
from paper_2502_02704_b200 import runtime as rt
from paper_2502_02704_b200.parareal import GpuBackend, ShardedRun
b = GpuBackend(disc, kin, flu)
run = ShardedRun(b)
snaps = run.coarse_sweep(rt.to_device_moments(U0, b.device))
jumps = b.empty(w.n_g)
jumps.zero_()
# windows 63..64 only (k = 63): 2 fine windows + batched G + correction
run.jumps(snaps, jumps, 63)
run.correct(snaps, jumps, 63)
import torch; torch.cuda.synchronize()
print("ok", b.ctx.describe())
