"""One window of configs 2 and 3a through the bench's problem builder (for ncu)."""
import sys
sys.path.insert(0, ".")
import bench
import paper_2502_02704_b200 as P
from paper_2502_02704_b200 import runtime as rt
from paper_2502_02704_b200.configs import config
from paper_2502_02704_b200.parareal import GpuBackend
for idx in sys.argv[1:] or ["2", "3"]:
    w = config(idx)
    P_, phase, bc, disc, kin, flu = bench.build_problem(w)
    U0 = P.project(P.lift(P.MomentField(*w.raw_moments()), phase, bc=bc), phase, bc=bc)
    b = GpuBackend(disc, kin, flu)
    m0 = rt.to_device_moments(U0, b.device)
    out = b.empty(1)
    print(w.name, b.fine_into(m0, 1, out[0]), b.ctx.describe())
