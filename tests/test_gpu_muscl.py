"""MUSCL-minmod x transport on the GPU (north_star
"upwind/MUSCL") against the builder's ORACLE EXTENSION
``oracle/bgk.py transport_muscl`` (self-pinned; the reference has only the
first-order upwind flux).  Transport bitwise on every tile configuration and
x boundary; multi-step F <= 1e-12; parareal <= 1e-10, equal iteration counts."""

import numpy as np
import pytest

from oracle import bgk as O
from helpers import mf, moment_gap, random_moments, rel_inf

pytestmark = pytest.mark.gpu
P = pytest.importorskip("paper_2502_02704_b200")

SHAPES = [
    (12, (8, 8, 8), 8.0),
    (10, (16, 16, 16), 8.0),
    (9, (32, 32, 32), 8.0),
    (7, (48, 48, 48), 10.0),
    (5, (64, 64, 64), 8.0),
    (8, (16, 8, 6), 5.0),
    (5, (9, 5, 7), 6.0),
    (40, (8, 8, 8), 8.0),
    (3, (16, 16, 16), 8.0),
]
BCS = ["periodic", "absorbing", "outflow"]


def _grids(nx, nv, vm):
    return (P.PhaseGrid(P.build_spatial_grid(0.0, 1.0, nx), P.build_velocity_grid(vm, nv)),
            O.Mesh(0.0, 1.0, nx, vm, nv))


def _f(mesh, seed):
    rng = np.random.default_rng(seed)
    f = O.lift(*random_moments(mesh.nx, rng), mesh)
    return f * rng.uniform(0.7, 1.3, f.shape)


@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: "x".join(map(str, (s[0],) + s[1])))
@pytest.mark.parametrize("bc", BCS)
def test_muscl_transport_bitwise(shape, bc):
    nx, nv, vm = shape
    grid, mesh = _grids(nx, nv, vm)
    f = _f(mesh, nx)
    dt = 0.45 * O.fine_cap(mesh, 1.0)
    kp = P.KineticParams(1e-2, scheme="muscl")
    got = P.transport_update(P.Distribution(f), dt, grid, kp, P.BoundaryKind(bc)).values
    want = O.transport_muscl(f, dt, mesh, bc)
    assert np.array_equal(got, want), rel_inf(got, want)


@pytest.mark.parametrize("shape", SHAPES[:5], ids=lambda s: "x".join(map(str, (s[0],) + s[1])))
@pytest.mark.parametrize("bc", BCS)
def test_muscl_propagate_matches_oracle(shape, bc):
    nx, nv, vm = shape
    grid, mesh = _grids(nx, nv, vm)
    f = _f(mesh, 3)
    cap = O.fine_cap(mesh, 0.5)
    t1 = 5.5 * cap
    kp = P.KineticParams(1e-2, scheme="muscl")
    got = P.propagate_kinetic(P.Distribution(f), 0.0, t1, grid, kp, P.BoundaryKind(bc))
    want = O.fine_propagate(f, 0.0, t1, mesh, 1e-2, bc, scheme="muscl")
    assert rel_inf(got.values, want) <= 1e-12
    # and it is not the upwind result
    up = O.fine_propagate(f, 0.0, t1, mesh, 1e-2, bc)
    assert rel_inf(up, want) > 1e-6


def test_muscl_parareal_matches_oracle():
    mesh = O.Mesh(0.0, 1.0, 32, 8.0, (8, 8, 8))
    prob = O.Problem(mesh, 0.05, 4, 16, 1e-2, "outflow", scheme="muscl")
    U0 = O.two_state(mesh, 0.5, (1.0, 0.0, 1.0), (0.125, 0.0, 0.8))
    want_s, want_e = O.parareal(prob, U0, 3, 1e-300)
    disc = P.Discretization(P.PhaseGrid(P.build_spatial_grid(0.0, 1.0, 32), P.build_velocity_grid(8.0, 8)),
                            P.build_time_grids(0.05, 4, 16), P.BoundaryKind.OUTFLOW)
    traj, rec = P.run_parareal(P.MomentField(*U0), P.PararealConfig(3, 1e-300), disc,
                               P.KineticParams(1e-2, scheme="muscl"), P.FluidParams())
    assert len(rec) == len(want_e)
    for a, b in zip(traj.snapshots, want_s):
        assert moment_gap(mf(a), b) <= 1e-10
    for e1, e2 in zip([r.error for r in rec], want_e):
        assert abs(e1 - e2) <= 1e-10 * max(1.0, abs(e2))


def test_muscl_rejects_field():
    with pytest.raises(P.ConfigurationError):
        P.KineticParams(1e-2, force=np.ones(4), scheme="muscl")
