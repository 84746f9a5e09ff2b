"""Ad-hoc probe used during development (not collected by pytest)."""
import sys
import numpy as np
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import paper_2502_02704_b200 as P
from oracle import bgk as O
import torch

what = sys.argv[1]
nx = int(sys.argv[2])
nv = tuple(int(x) for x in sys.argv[3].split(","))
vm = 8.0
grid = P.PhaseGrid(P.build_spatial_grid(0.0, 1.0, nx), P.build_velocity_grid(vm, nv))
mesh = O.Mesh(0.0, 1.0, nx, vm, nv)
rng = np.random.default_rng(0)
U = (rng.uniform(0.5, 1.5, nx), rng.uniform(-0.4, 0.4, (nx, 3)), rng.uniform(0.5, 1.5, nx))
f = O.lift(*U, mesh)
if what == "transport":
    got = P.transport_update(P.Distribution(f), 1e-3, grid, P.KineticParams(1.0), P.BoundaryKind.PERIODIC).values
    want = O.transport(f, 1e-3, mesh, True)
    print(what, np.max(np.abs(got - want)))
elif what == "project":
    got = P.project(P.Distribution(f), grid)
    want = O.project(f, mesh)
    print(what, np.max(np.abs(got.rho - want[0])), np.max(np.abs(got.u - want[1])), np.max(np.abs(got.theta - want[2])))
