"""Diffusive-scaling extension on the GPU (BASELINE config 3b).

alpha = 1 fine propagator and the drift-diffusion coarse propagator, checked
against the builder's ORACLE EXTENSIONS (``oracle/bgk.py`` ``fine_propagate(
alpha=1)``, ``dd_propagate``): parity is self-pinned, the reference has no
diffusive path.  Same bars as the reference-pinned paths: G bitwise,
F <= 1e-12, parareal <= 1e-10 with identical iteration counts.
"""

import numpy as np
import pytest

from oracle import bgk as O
from helpers import mf, moment_gap, random_moments, rel_inf

pytestmark = pytest.mark.gpu
P = pytest.importorskip("paper_2502_02704_b200")


def _grids(nx, nv, v_max):
    return (P.PhaseGrid(P.build_spatial_grid(0.0, 1.0, nx), P.build_velocity_grid(v_max, nv)),
            O.Mesh(0.0, 1.0, nx, v_max, nv))


@pytest.mark.parametrize("bc", ["periodic", "outflow", "absorbing"])
@pytest.mark.parametrize("field", [False, True])
@pytest.mark.parametrize("nx", [37, 1024, 3000])
def test_drift_diffusion_G_bitwise(bc, field, nx):
    grid, mesh = _grids(nx, (16, 4, 4), 8.0)
    rng = np.random.default_rng(nx)
    U = random_moments(nx, rng)
    E = 0.5 * np.sin(2 * np.pi * mesh.xc) if field else None
    D = O.dd_m2(mesh)
    fp = P.FluidParams(force=E, model="drift_diffusion")
    assert P.drift_diffusion_m2(8.0, 16) == D
    span = 40.5 * O.dd_cap(mesh.dx, D, O.field_bound(E), 0.9)
    got = mf(P.propagate_fluid(P.MomentField(*U), 0.0, span, grid, fp, P.BoundaryKind(bc)))
    want = O.dd_propagate(U[0], 0.0, span, mesh, bc, E, None, 0.9, D)
    for a, b in zip(got, want):
        assert np.array_equal(a, b), rel_inf(a, b)
    # dt_max cap and an explicit diffusivity
    fp2 = P.FluidParams(force=E, model="drift_diffusion", diffusivity=0.7)
    got = mf(P.propagate_fluid(P.MomentField(*U), 0.0, span, grid, fp2, P.BoundaryKind(bc),
                               dt_max=span / 7.0))
    want = O.dd_propagate(U[0], 0.0, span, mesh, bc, E, span / 7.0, 0.9, 0.7)
    assert np.array_equal(got[0], want[0])


def test_drift_diffusion_G_blowup_step():
    grid, mesh = _grids(8, (8, 4, 4), 8.0)
    rho = np.full(8, 1e-3)
    rho[3] = 1.0
    U = P.MomentField(rho, np.zeros((8, 3)), np.ones(8))
    fp = P.FluidParams(cfl=3.0, model="drift_diffusion", diffusivity=1.0)
    with pytest.raises(P.BlowUpError) as ei:
        P.propagate_fluid(U, 0.0, 1.0, grid, fp, P.BoundaryKind.PERIODIC)
    assert ei.value.step == 1
    with pytest.raises(P.ConfigurationError):
        P.FluidParams(model="navier_stokes")


@pytest.mark.parametrize("shape", [(12, (8, 8, 8), 8.0), (9, (32, 32, 32), 8.0),
                                   (5, (64, 64, 64), 8.0)],
                         ids=lambda s: "x".join(map(str, (s[0],) + s[1])))
@pytest.mark.parametrize("field", [False, True])
def test_alpha1_fine_propagator(shape, field):
    nx, nv, vm = shape
    grid, mesh = _grids(nx, nv, vm)
    rng = np.random.default_rng(11)
    U = random_moments(nx, rng)
    f = O.lift(*U, mesh) * rng.uniform(0.8, 1.2, (nx,) + nv)
    E = 0.5 * np.sin(2 * np.pi * mesh.xc) if field else None
    eps = 1e-2
    kp = P.KineticParams(eps, force=E, alpha=1)
    cap = O.scaled_cap(mesh, 0.5, E, eps, 1)
    assert P.stable_dt_kinetic(grid, kp) == cap
    t1 = 6.5 * cap
    got = P.propagate_kinetic(P.Distribution(f), 0.0, t1, grid, kp, P.BoundaryKind.PERIODIC)
    want = O.fine_propagate(f, 0.0, t1, mesh, eps, True, E, alpha=1)
    assert rel_inf(got.values, want) <= 1e-12
    # the single-step API scales the same way
    d = 0.5 * cap
    tr = P.transport_update(P.Distribution(f), d, grid, kp, P.BoundaryKind.PERIODIC)
    assert rel_inf(tr.values, O.transport(f, d / eps, mesh, True, E)) <= (1e-14 if field else 0.0)
    rx = P.bgk_relax(P.Distribution(f), d, grid, kp)
    assert rel_inf(rx.values, O.relax(f, d / eps, mesh, eps)) <= 1e-13


@pytest.mark.parametrize("frozen", [True, False])
def test_config3b_reduced_parareal(frozen):
    # BASELINE config 3 as stated (alpha = 1, drift-diffusion G, E = 0.5 sin 2 pi x,
    # rho = 1 + 0.3 cos 2 pi x, periodic) on a reduced phase grid and time span
    from dataclasses import replace
    from paper_2502_02704_b200.configs import config, reduced
    w = replace(reduced(config("3b"), 48, (16, 16, 16), n_g=4), t_final=2e-3, k_max=3)
    mesh = O.Mesh(w.x_min, w.x_max, w.nx, w.v_max, w.nv)
    prob = O.Problem(mesh, w.t_final, w.n_g, w.n_f, w.eps, True, w.force(), alpha=1,
                     g_model="drift_diffusion")
    raw = w.raw_moments()
    U0o = O.project(O.lift(*raw, mesh), mesh)
    want_s, want_e = O.parareal(prob, U0o, w.k_max, w.tol, frozen)
    g = P.PhaseGrid(P.build_spatial_grid(0.0, 1.0, w.nx), P.build_velocity_grid(w.v_max, w.nv))
    d = P.Discretization(g, P.build_time_grids(w.t_final, w.n_g, w.n_f), P.BoundaryKind.PERIODIC)
    U0p = P.project(P.lift(P.MomentField(*raw), g), g)
    traj, rec = P.run_parareal(U0p, P.PararealConfig(w.k_max, w.tol, frozen), d,
                               P.KineticParams(w.eps, force=w.force(), alpha=1),
                               P.FluidParams(force=w.force(), model="drift_diffusion"))
    assert len(rec) == len(want_e)
    for a, b in zip(traj.snapshots, want_s):
        assert moment_gap(mf(a), b) <= 1e-10
    for e1, e2 in zip([r.error for r in rec], want_e):
        assert abs(e1 - e2) <= 1e-10 * max(1.0, abs(e2))
    # G really is the diffusive one: iteration 0 snapshots have u = 0, theta = 1
    assert want_e[0] > 0.0
