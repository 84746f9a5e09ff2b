"""Trapezoidal velocity quadrature on the GPU (BASELINE
config 0's "trapezoidal quadrature") against the builder's ORACLE EXTENSION
``oracle.bgk.Mesh(quadrature="trapezoid")`` (self-pinned).  Nodes include the
cube ends, dv = 2 v_max/(n-1), end nodes weigh 1/2 in every velocity sum."""

import numpy as np
import pytest

from oracle import bgk as O
from helpers import mf, moment_gap, random_moments, rel_inf

pytestmark = pytest.mark.gpu
P = pytest.importorskip("paper_2502_02704_b200")

SHAPES = [(12, (8, 8, 8), 8.0), (9, (32, 32, 32), 8.0), (7, (48, 48, 48), 10.0),
          (5, (64, 64, 64), 8.0), (8, (16, 8, 6), 5.0), (5, (9, 5, 7), 6.0)]


def _grids(nx, nv, vm):
    return (P.PhaseGrid(P.build_spatial_grid(0.0, 1.0, nx),
                        P.build_velocity_grid(vm, nv, quadrature="trapezoid")),
            O.Mesh(0.0, 1.0, nx, vm, nv, "trapezoid"))


@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: "x".join(map(str, (s[0],) + s[1])))
def test_trapezoid_lift_project_relax(shape):
    nx, nv, vm = shape
    grid, mesh = _grids(nx, nv, vm)
    assert all(np.array_equal(a, b) for a, b in zip(grid.velocity.centers, mesh.vc))
    rng = np.random.default_rng(nx)
    U = random_moments(nx, rng)
    for norm in (False, True):
        got = P.lift(P.MomentField(*U), grid, normalize_mass=norm).values
        assert rel_inf(got, O.lift(*U, mesh, normalize=norm)) <= 1e-13
    f = O.lift(*U, mesh) * rng.uniform(0.8, 1.2, (nx,) + nv)
    assert moment_gap(mf(P.project(P.Distribution(f), grid)), O.project(f, mesh)) <= 1e-13
    dt = 0.3 * O.fine_cap(mesh, 0.5)
    got = P.bgk_relax(P.Distribution(f), dt, grid, P.KineticParams(2e-2)).values
    assert rel_inf(got, O.relax(f, dt, mesh, 2e-2)) <= 1e-13


@pytest.mark.parametrize("shape", SHAPES[:4], ids=lambda s: "x".join(map(str, (s[0],) + s[1])))
@pytest.mark.parametrize("bc", ["periodic", "absorbing", "outflow"])
@pytest.mark.parametrize("scheme", ["upwind", "muscl"])
def test_trapezoid_propagate(shape, bc, scheme):
    nx, nv, vm = shape
    grid, mesh = _grids(nx, nv, vm)
    rng = np.random.default_rng(3)
    f = O.lift(*random_moments(nx, rng), mesh) * rng.uniform(0.8, 1.2, (nx,) + nv)
    t1 = 5.5 * O.fine_cap(mesh, 0.5)
    got = P.propagate_kinetic(P.Distribution(f), 0.0, t1, grid,
                              P.KineticParams(1e-2, scheme=scheme), P.BoundaryKind(bc))
    want = O.fine_propagate(f, 0.0, t1, mesh, 1e-2, bc, scheme=scheme)
    assert rel_inf(got.values, want) <= 1e-12


def test_trapezoid_even_data_zero_velocity():
    grid, mesh = _grids(6, (16, 16, 16), 8.0)
    rng = np.random.default_rng(1)
    half = rng.uniform(0.1, 1.0, (6, 8, 16, 16))
    f = np.concatenate([half, half[:, ::-1]], axis=1)
    f = np.concatenate([f[:, :, :8], f[:, :, :8][:, :, ::-1]], axis=2)
    f = np.concatenate([f[..., :8], f[..., :8][..., ::-1]], axis=3)
    U = P.project(P.Distribution(f), grid)
    assert np.all(U.u == 0.0)


def test_config0_trapezoid_parareal():
    # BASELINE config 0 as worded: Sod, 64 x 16^3 on [-8, 8]^3 with trapezoidal
    # quadrature, outflow, eps 1e-2, 8 slices, K = 2
    from paper_2502_02704_b200.configs import config
    w = config("0t")
    mesh = O.Mesh(w.x_min, w.x_max, w.nx, w.v_max, w.nv, "trapezoid")
    prob = O.Problem(mesh, w.t_final, w.n_g, w.n_f, w.eps, w.bc)
    raw = w.raw_moments()
    U0o = O.project(O.lift(*raw, mesh), mesh)
    want_s, want_e = O.parareal(prob, U0o, w.k_max, w.tol)
    g = P.PhaseGrid(P.build_spatial_grid(0.0, 1.0, w.nx),
                    P.build_velocity_grid(w.v_max, w.nv, quadrature="trapezoid"))
    d = P.Discretization(g, P.build_time_grids(w.t_final, w.n_g, w.n_f), P.BoundaryKind(w.bc))
    U0p = P.project(P.lift(P.MomentField(*raw), g, bc=d.bc), g, bc=d.bc)
    traj, rec = P.run_parareal(U0p, P.PararealConfig(w.k_max, w.tol), d, P.KineticParams(w.eps),
                               P.FluidParams())
    assert len(rec) == len(want_e) == 2
    for a, b in zip(traj.snapshots, want_s):
        assert moment_gap(mf(a), b) <= 1e-10


def test_trapezoid_rejects_field():
    grid, _ = _grids(4, (8, 8, 8), 8.0)
    f = np.ones((4, 8, 8, 8))
    with pytest.raises(P.ConfigurationError):
        P.propagate_kinetic(P.Distribution(f), 0.0, 1e-3, grid,
                            P.KineticParams(1e-2, force=np.ones(4)), P.BoundaryKind.PERIODIC)
