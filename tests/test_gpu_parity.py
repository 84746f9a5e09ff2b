"""GPU (libpbgk.so) vs the CPU oracle on the same seeded inputs.

Tolerances: the x transport and G are evaluated in the reference's operation
order and must match bit for bit (the v_x field flux is reassociated: 1e-14); projections/lifts differ from numpy only in the
summation order of the marginals and in exp/pow (<= a few ulp), so they are
held to 1e-13 relative; multi-step runs to 1e-12; parareal to the north-star
bound 1e-10 (normwise).
"""

import numpy as np
import pytest

from oracle import bgk as O
from helpers import mf, moment_gap, random_moments, rel_inf

pytestmark = pytest.mark.gpu

P = pytest.importorskip("paper_2502_02704_b200")

# (nx, nv, v_max): one per tile configuration of the sweep (see capi.cu)
SHAPES = [
    (12, (8, 8, 8), 8.0),
    (10, (16, 16, 16), 8.0),
    (9, (32, 32, 32), 8.0),
    (7, (48, 48, 48), 10.0),
    (5, (64, 64, 64), 8.0),
    (8, (16, 8, 6), 5.0),
    (5, (9, 5, 7), 6.0),
    (10, (64, 8, 8), 6.0),
    (6, (256, 8, 8), 8.0),
]


def _grids(nx, nv, v_max, x0=0.0, x1=1.0):
    return (P.PhaseGrid(P.build_spatial_grid(x0, x1, nx), P.build_velocity_grid(v_max, nv)),
            O.Mesh(x0, x1, nx, v_max, nv))


def _rand_f(mesh, rng, jitter=0.2):
    U = random_moments(mesh.nx, rng)
    f = O.lift(*U, mesh)
    return f * rng.uniform(1 - jitter, 1 + jitter, size=f.shape)


@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: "x".join(map(str, (s[0],) + s[1])))
@pytest.mark.parametrize("normalize", [False, True])
def test_lift_matches_oracle(shape, normalize):
    nx, nv, vm = shape
    grid, mesh = _grids(nx, nv, vm)
    U = random_moments(nx, np.random.default_rng(1))
    got = P.lift(P.MomentField(*U), grid, normalize_mass=normalize).values
    want = O.lift(*U, mesh, normalize=normalize)
    assert rel_inf(got, want) <= 1e-13


@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: "x".join(map(str, (s[0],) + s[1])))
def test_project_matches_oracle(shape):
    nx, nv, vm = shape
    grid, mesh = _grids(nx, nv, vm)
    f = _rand_f(mesh, np.random.default_rng(2))
    got = mf(P.project(P.Distribution(f), grid))
    assert moment_gap(got, O.project(f, mesh)) <= 1e-13


@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: "x".join(map(str, (s[0],) + s[1])))
def test_project_even_data_exact_zero(shape):
    # mirror-symmetric in every velocity axis -> folded first moments are exactly 0
    nx, nv, vm = shape
    grid, mesh = _grids(nx, nv, vm)
    rng = np.random.default_rng(3)
    f = rng.uniform(0.1, 1.0, size=(nx,) + nv)
    f = f + f[:, ::-1]
    f = f + f[:, :, ::-1]
    f = f + f[:, :, :, ::-1]
    U = P.project(P.Distribution(f), grid)
    assert np.all(U.u == 0.0)


@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: "x".join(map(str, (s[0],) + s[1])))
@pytest.mark.parametrize("periodic", [True, False])
@pytest.mark.parametrize("field", [False, True])
def test_transport_bitwise(shape, periodic, field):
    nx, nv, vm = shape
    grid, mesh = _grids(nx, nv, vm)
    rng = np.random.default_rng(4)
    f = _rand_f(mesh, rng)
    E = 0.5 * np.sin(2 * np.pi * mesh.xc) if field else None
    dt = 0.4 * O.fine_cap(mesh, 0.5, E)
    bc = P.BoundaryKind.PERIODIC if periodic else P.BoundaryKind.ABSORBING
    got = P.transport_update(P.Distribution(f), dt, grid, P.KineticParams(1.0, force=E), bc).values
    want = O.transport(f, dt, mesh, periodic, E)
    if field:  # the v_x flux is reassociated (cp lo + cm hi): within an ulp per face
        assert rel_inf(got, want) <= 1e-14
    else:      # x transport: the reference's operation order, bit for bit
        assert np.array_equal(got, want), rel_inf(got, want)


@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: "x".join(map(str, (s[0],) + s[1])))
def test_relax_matches_oracle(shape):
    nx, nv, vm = shape
    grid, mesh = _grids(nx, nv, vm)
    f = _rand_f(mesh, np.random.default_rng(5))
    got = P.bgk_relax(P.Distribution(f), 2e-3, grid, P.KineticParams(1e-2)).values
    assert rel_inf(got, O.relax(f, 2e-3, mesh, 1e-2)) <= 1e-13


@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: "x".join(map(str, (s[0],) + s[1])))
@pytest.mark.parametrize("periodic", [True, False])
@pytest.mark.parametrize("field", [False, True])
def test_propagate_matches_oracle(shape, periodic, field):
    nx, nv, vm = shape
    grid, mesh = _grids(nx, nv, vm)
    f = _rand_f(mesh, np.random.default_rng(6))
    E = 0.5 * np.sin(2 * np.pi * mesh.xc) if field else None
    cap = O.fine_cap(mesh, 0.5, E)
    t1 = 5.5 * cap  # 6 steps, the last one partial
    bc = P.BoundaryKind.PERIODIC if periodic else P.BoundaryKind.ABSORBING
    got = P.propagate_kinetic(P.Distribution(f), 0.0, t1, grid, P.KineticParams(1e-2, force=E), bc)
    want = O.fine_propagate(f, 0.0, t1, mesh, 1e-2, periodic, E)
    assert rel_inf(got.values, want) <= 1e-12


@pytest.mark.parametrize("periodic", [True, False])
@pytest.mark.parametrize("field", [False, True])
def test_fluid_bitwise(periodic, field):
    nx = 40
    grid, mesh = _grids(nx, (4, 4, 4), 8.0)
    rng = np.random.default_rng(7)
    U = random_moments(nx, rng)
    E = 0.3 * np.sin(2 * np.pi * mesh.xc) if field else None
    bc = P.BoundaryKind.PERIODIC if periodic else P.BoundaryKind.ABSORBING
    got = mf(P.propagate_fluid(P.MomentField(*U), 0.0, 0.05, grid, P.FluidParams(force=E), bc,
                               dt_max=0.01))
    want = O.coarse_propagate(*U, 0.0, 0.05, mesh, periodic, E, 0.01)
    for a, b in zip(got, want):
        assert np.array_equal(a, b), rel_inf(a, b)


@pytest.mark.parametrize("frozen", [True, False])
def test_parareal_small_matches_oracle(frozen):
    mesh = O.Mesh(0.0, 1.0, 16, 8.0, (8, 8, 8))
    prob = O.Problem(mesh, 0.05, 4, 16, 1e-2, False)
    U0 = O.two_state(mesh, 0.5, (1.0, 0.0, 1.0), (0.125, 0.0, 0.8))
    want_s, want_e = O.parareal(prob, U0, 3, 1e-300, frozen)
    disc = P.Discretization(P.PhaseGrid(P.build_spatial_grid(0.0, 1.0, 16),
                                        P.build_velocity_grid(8.0, 8)),
                            P.build_time_grids(0.05, 4, 16), P.BoundaryKind.ABSORBING)
    traj, rec = P.run_parareal(P.MomentField(*U0), P.PararealConfig(3, 1e-300, frozen), disc,
                               P.KineticParams(1e-2), P.FluidParams())
    assert len(rec) == len(want_e)
    for a, b in zip(traj.snapshots, want_s):
        assert moment_gap(mf(a), b) <= 1e-10
    for e1, e2 in zip([r.error for r in rec], want_e):
        assert abs(e1 - e2) <= 1e-10 * max(1.0, abs(e2))
