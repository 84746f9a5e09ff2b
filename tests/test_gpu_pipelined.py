"""Pipelined parareal on the GPU: the side-stream G
jumps and correction trailing the fine windows must reproduce the phased
iteration BIT FOR BIT (same kernels on the same inputs), for the Euler and
the drift-diffusion coarse propagators, and raise the phased run's errors."""

import numpy as np
import pytest

from helpers import mf

pytestmark = pytest.mark.gpu
P = pytest.importorskip("paper_2502_02704_b200")


def _sod(nx, nv, t, n_g, n_f, bc):
    g = P.PhaseGrid(P.build_spatial_grid(0.0, 1.0, nx), P.build_velocity_grid(8.0, nv))
    d = P.Discretization(g, P.build_time_grids(t, n_g, n_f), bc)
    x = g.space.centers
    U0 = P.MomentField(np.where(x < 0.5, 1.0, 0.125), np.zeros((nx, 3)), np.where(x < 0.5, 1.0, 0.8))
    return d, U0


def _same(a, b):
    for s, t in zip(a.snapshots, b.snapshots):
        for x, y in zip(mf(s), mf(t)):
            assert np.array_equal(x, y)


@pytest.mark.parametrize("frozen", [True, False])
@pytest.mark.parametrize("nv", [8, 32])
def test_pipelined_bitwise_equals_phased_euler(frozen, nv):
    d, U0 = _sod(64, nv, 0.05, 6, 24, P.BoundaryKind.OUTFLOW)
    kp, fp = P.KineticParams(1e-2), P.FluidParams()
    t1, r1 = P.run_parareal(U0, P.PararealConfig(4, 1e-300, frozen), d, kp, fp)
    t2, r2 = P.run_parareal(U0, P.PararealConfig(4, 1e-300, frozen, pipelined=True), d, kp, fp)
    assert [r.error for r in r1] == [r.error for r in r2]
    _same(t1, t2)
    _same(P.ParTrajectory(t1.jumps, [], []), P.ParTrajectory(t2.jumps, [], []))


def test_pipelined_bitwise_equals_phased_drift_diffusion():
    nx = 128
    g = P.PhaseGrid(P.build_spatial_grid(0.0, 1.0, nx), P.build_velocity_grid(8.0, 16))
    d = P.Discretization(g, P.build_time_grids(2e-3, 4, 4), P.BoundaryKind.PERIODIC)
    x = g.space.centers
    E = 0.5 * np.sin(2 * np.pi * x)
    U0 = P.MomentField(1.0 + 0.3 * np.cos(2 * np.pi * x), np.zeros((nx, 3)), np.ones(nx))
    kp = P.KineticParams(1e-2, force=E, alpha=1)
    fp = P.FluidParams(force=E, model="drift_diffusion")
    t1, r1 = P.run_parareal(U0, P.PararealConfig(3, 1e-300), d, kp, fp)
    t2, r2 = P.run_parareal(U0, P.PararealConfig(3, 1e-300, pipelined=True), d, kp, fp)
    assert [r.error for r in r1] == [r.error for r in r2]
    _same(t1, t2)


def test_pipelined_stops_at_tolerance_like_phased():
    d, U0 = _sod(32, 8, 0.05, 4, 16, P.BoundaryKind.ABSORBING)
    kp, fp = P.KineticParams(1e-2), P.FluidParams()
    _, r1 = P.run_parareal(U0, P.PararealConfig(4, 1e-300), d, kp, fp)
    tol = 0.5 * (r1[1].error + r1[2].error)  # stops after iteration 3
    _, ra = P.run_parareal(U0, P.PararealConfig(4, tol), d, kp, fp)
    _, rb = P.run_parareal(U0, P.PararealConfig(4, tol, pipelined=True), d, kp, fp)
    assert [r.k for r in ra] == [r.k for r in rb] == [1, 2, 3]


def test_pipelined_overshoot_raises_like_phased():
    # the reference's absorbing BC on config 2 overshoots in iteration 1
    # (DESIGN.md 7); both schedules must raise the same slice index
    from dataclasses import replace
    from paper_2502_02704_b200.configs import config, reduced
    w = replace(reduced(config(2), 64, (16, 16, 16), n_g=8), outflow=False)
    g = P.PhaseGrid(P.build_spatial_grid(0.0, 1.0, w.nx), P.build_velocity_grid(w.v_max, w.nv))
    d = P.Discretization(g, P.build_time_grids(w.t_final, w.n_g, w.n_f), P.BoundaryKind.ABSORBING)
    U0 = P.project(P.lift(P.MomentField(*w.raw_moments()), g), g)
    kp, fp = P.KineticParams(w.eps), P.FluidParams()
    out = []
    for pipe in (False, True):
        try:
            P.run_parareal(U0, P.PararealConfig(3, 1e-300, pipelined=pipe), d, kp, fp)
            out.append(None)
        except P.CorrectionOvershootError as e:
            out.append(e.slice_index)
    assert out[0] == out[1]


def test_fine_stage_failure_same_error_both_schedules():
    # an unstable kinetic CFL: the batched fine stage (phased) and the
    # per-window calls (pipelined) must raise the same error -- the
    # reference's precedence makes it DegenerateStateError (rho or theta <= 0)
    # or BlowUpError (non-finite), with the same step
    # long windows (~85 steps at CFL 6): the upwind amplification runs away
    d, U0 = _sod(32, 8, 4.0, 2, 2, P.BoundaryKind.PERIODIC)
    kp, fp = P.KineticParams(1e-2, cfl=6.0), P.FluidParams()
    seen = []
    for pipe in (False, True):
        with pytest.raises(P.SolverError) as ei:
            P.run_parareal(U0, P.PararealConfig(2, 1e-300, pipelined=pipe), d, kp, fp)
        seen.append((type(ei.value).__name__, getattr(ei.value, "step", None), str(ei.value)))
    assert seen[0] == seen[1]
