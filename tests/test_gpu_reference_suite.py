"""The reference test suite's claims, re-checked against the GPU package.

Each test restates one behaviour the reference's own suite pins
(pkg/tests/test_kinetic.py, test_moments.py, test_lifting.py, test_fluid.py,
test_parareal.py, test_acceptance.py) with the same
tolerance, against ``paper_2502_02704_b200`` instead of ``parabgk``.  Bitwise
claims of the reference are kept bitwise where the GPU arithmetic is in the
reference's operation order (transport, G) or is a deterministic replay of
itself (dt-cap replay, worker/rank determinism).
"""

import math

import numpy as np
import pytest

import riemann

pytestmark = pytest.mark.gpu
P = pytest.importorskip("paper_2502_02704_b200")


def grid(n_x=8, v_max=8.0, n_v=8, x_max=2.0):
    return P.PhaseGrid(P.build_spatial_grid(0.0, x_max, n_x), P.build_velocity_grid(v_max, n_v))


def uniform(n_x, rho, u, theta):
    return P.MomentField(np.full(n_x, float(rho)), np.tile(np.asarray(u, float), (n_x, 1)),
                         np.full(n_x, float(theta)))


def sod(space, edge=1.0):
    x = space.centers
    return P.MomentField(np.where(x < edge, 1.0, 0.125), np.zeros((x.size, 3)),
                         np.where(x < edge, 1.0, 0.8))


PER, ABS = P.BoundaryKind.PERIODIC, P.BoundaryKind.ABSORBING


# --------------------------------------------------------------------- kinetic

def test_transport_keeps_a_constant_state_exactly():
    g = grid()
    f = P.lift(uniform(8, 1.0, (0.3, 0, 0), 1.0), g)
    out = P.transport_update(f, 1e-3, g, P.KineticParams(1.0), PER)
    assert np.array_equal(out.values, f.values)


def test_upwind_moves_a_parcel_one_cell_at_unit_courant():
    g = grid()
    cx = g.velocity.centers[0]
    j = int(np.argmax(cx))
    f = np.zeros((8, 8, 8, 8))
    f[3, j, 4, 4] = 1.0
    out = P.transport_update(P.Distribution(f), g.space.dx / cx[j], g, P.KineticParams(1.0),
                             PER).values
    assert out[4, j, 4, 4] == pytest.approx(1.0, rel=1e-14)
    assert out[3, j, 4, 4] == 0.0
    assert out.sum() == pytest.approx(1.0, rel=1e-14)


def test_absorbing_boundary_lets_mass_leave():
    g = grid()
    j = int(np.argmax(g.velocity.centers[0]))
    f = np.zeros((8, 8, 8, 8))
    f[7, j, 4, 4] = 1.0
    out = P.transport_update(P.Distribution(f), g.space.dx / g.velocity.centers[0][j], g,
                             P.KineticParams(1.0), ABS).values
    assert out.sum() == 0.0


def test_field_term_momentum_source_and_mass():
    g = grid(n_x=4, n_v=32)
    params = P.KineticParams(1.0, force=np.full(4, 0.7))
    f = P.lift(uniform(4, 1.3, (0.2, 0, 0), 0.9), g)
    b = P.project(f, g)
    a = P.project(P.transport_update(f, 1e-3, g, params, PER), g)
    np.testing.assert_allclose(a.rho * a.u[:, 0] - b.rho * b.u[:, 0], 1e-3 * 0.7 * b.rho, rtol=1e-12)
    g16 = grid(n_x=4, n_v=16)
    f = P.lift(uniform(4, 1.0, (0, 0, 0), 1.0), g16)
    out = P.transport_update(f, 2e-3, g16, P.KineticParams(1.0, force=np.full(4, 0.9)), PER)
    assert out.values.sum() == pytest.approx(f.values.sum(), rel=1e-14)


def test_relax_fixed_point_half_blend_and_stiff_limit():
    g = grid(n_x=2, n_v=32)
    f = P.lift(uniform(2, 1.0, (0, 0, 0), 1.0), g, normalize_mass=True)
    out = P.bgk_relax(f, 1e-2, g, P.KineticParams(1e-2))
    assert np.max(np.abs(out.values - f.values)) <= 1e-14
    g16 = grid(n_x=2, n_v=16)
    base = P.lift(uniform(2, 1.0, (0, 0, 0), 1.0), g16).values
    fv = base * np.random.default_rng(5).uniform(0.5, 1.5, base.shape)
    out = P.bgk_relax(P.Distribution(fv.copy()), 0.25, g16, P.KineticParams(0.25)).values
    M = P.lift(P.project(P.Distribution(fv), g16), g16, normalize_mass=True).values
    np.testing.assert_allclose(out, 0.5 * (fv + M), rtol=1e-14)
    probe = fv.copy()
    probe[0, 3, 4, 5] = 0.0
    M2 = P.lift(P.project(P.Distribution(probe), g16), g16, normalize_mass=True).values
    out2 = P.bgk_relax(P.Distribution(probe), 0.25, g16, P.KineticParams(0.25)).values
    assert out2[0, 3, 4, 5] == pytest.approx(0.5 * M2[0, 3, 4, 5], rel=1e-14)
    fs = base * 1.3
    out = P.bgk_relax(P.Distribution(fs), 1e-2, g16, P.KineticParams(1e-6)).values
    Ms = P.lift(P.project(P.Distribution(fs), g16), g16, normalize_mass=True).values
    assert np.max(np.abs(out - Ms)) <= np.max(np.abs(fs - Ms)) / (1e-2 / 1e-6) * 1.001


def test_relax_conserves_discrete_mass():
    g = grid(n_x=3, n_v=16)
    base = P.lift(uniform(3, 1.0, (0.1, -0.2, 0.3), 0.8), g).values
    f = base * np.random.default_rng(9).uniform(0.8, 1.2, base.shape)
    out = P.bgk_relax(P.Distribution(f), 5e-3, g, P.KineticParams(1e-2)).values
    np.testing.assert_allclose(out.sum(axis=(1, 2, 3)), f.sum(axis=(1, 2, 3)), rtol=1e-14)


def _two_beams(g, n_x):
    u1 = np.zeros((n_x, 3)); u1[:, 0] = 0.5
    u2 = np.zeros((n_x, 3)); u2[:, 0] = -0.75
    return (P.lift(P.MomentField(np.full(n_x, 0.6), u1, np.full(n_x, 0.6)), g).values +
            P.lift(P.MomentField(np.full(n_x, 0.4), u2, np.full(n_x, 0.5)), g).values)


@pytest.mark.parametrize("steps,dt,eps", [(12, 2e-3, 1e-1), (50, 2e-3, 0.1)])
def test_homogeneous_relaxation_closed_form(steps, dt, eps):
    n_x = 2 if steps == 12 else 4
    g = grid(n_x=n_x, n_v=32)
    f0 = _two_beams(g, n_x)
    got = P.propagate_kinetic(P.Distribution(f0), 0.0, dt * steps, g, P.KineticParams(eps), PER,
                              dt_max=dt).values
    a = (1.0 / (1.0 + dt / eps)) ** steps
    M0 = P.lift(P.project(P.Distribution(f0), g), g, normalize_mass=True).values
    assert np.max(np.abs(got - (a * f0 + (1 - a) * M0))) <= 1e-13 * np.max(np.abs(f0))


def test_empty_and_reversed_intervals():
    g = grid(n_x=2)
    f = P.lift(uniform(2, 1.0, (0, 0, 0), 1.0), g)
    assert P.propagate_kinetic(f, 0.3, 0.3, g, P.KineticParams(1.0), PER) is f
    with pytest.raises(P.ConfigurationError):
        P.propagate_kinetic(f, 1.0, 0.0, g, P.KineticParams(1.0), PER)


def test_dt_cap_replay_is_bitwise():
    g = grid()
    params = P.KineticParams(1e-1)
    f0 = P.lift(P.MomentField(np.linspace(1.0, 2.0, 8), np.zeros((8, 3)), np.full(8, 0.8)), g)
    cap = P.stable_dt_kinetic(g, params)
    span = 3.5 * cap
    from paper_2502_02704_b200 import runtime as rt
    with rt.ctx_for(g, PER).fusion_levels(0):  # the one-step path: the same ops, bit for bit
        out = P.propagate_kinetic(f0, 0.0, span, g, params, PER)
    fused = P.propagate_kinetic(f0, 0.0, span, g, params, PER)  # multi-step default
    f = f0
    done = 0.0
    while span - done > 1e-12 * span:
        dt = min(cap, span - done)
        f = P.bgk_relax(P.transport_update(f, dt, g, params, PER), dt, g, params)
        done += dt
    assert np.array_equal(out.values, f.values)
    # the multi-step path takes its relax moments from the recursion and
    # associates the transport differently: the same schedule to rounding
    assert np.max(np.abs(fused.values - f.values)) <= 1e-13 * np.max(np.abs(f.values))


def test_absorbing_outflow_bookkeeping():
    g = grid(n_x=10)
    params = P.KineticParams(1e-2)
    f = P.lift(sod(g.space), g)
    dvol, dx = g.velocity.cell_volume, g.space.dx
    vp, vm = np.maximum(g.velocity.centers[0], 0), np.minimum(g.velocity.centers[0], 0)
    cap = P.stable_dt_kinetic(g, params)
    span = 10.5 * cap
    mass0 = math.fsum(f.values.ravel()) * dvol * dx
    lost = []
    done = 0.0
    while span - done > 1e-12 * span:
        dt = min(cap, span - done)
        v = f.values
        lost.append(dt * (np.einsum("j,jkl->", vp, v[-1]) + np.einsum("j,jkl->", -vm, v[0])) * dvol)
        f = P.bgk_relax(P.transport_update(f, dt, g, params, ABS), dt, g, params)
        done += dt
    mass1 = math.fsum(f.values.ravel()) * dvol * dx
    assert mass0 - mass1 > 0
    assert abs((mass0 - mass1) - math.fsum(lost)) <= 1e-12 * mass0


def test_non_finite_state_reports_step_one():
    g = grid(n_x=4)
    f = P.lift(uniform(4, 1.0, (0, 0, 0), 1.0), g)
    f.values[0, 0, 0, 0] = np.nan
    with pytest.raises(P.BlowUpError) as info:
        P.propagate_kinetic(f, 0.0, 0.1, g, P.KineticParams(1e-2), PER)
    assert info.value.step == 1


def test_general_tau_callable_matches_constant():
    g = grid(n_x=6, n_v=8)
    f = P.lift(sod(g.space), g)
    span = 3.5 * P.stable_dt_kinetic(g, P.KineticParams(1e-2))
    a = P.propagate_kinetic(f, 0.0, span, g, P.KineticParams(1e-2, tau=P.ConstantTau(2.0)), ABS)
    b = P.propagate_kinetic(f, 0.0, span, g, P.KineticParams(1e-2, tau=lambda r, t: 2.0 + 0 * r), ABS)
    assert np.max(np.abs(a.values - b.values)) <= 1e-13 * np.max(a.values)


# --------------------------------------------------------------------- moments / lift

def test_projection_quadrature_and_exact_cases():
    g = grid(n_x=4, n_v=32)
    U = P.project(P.lift(uniform(4, 1.0, (0, 0, 0), 1.0), g), g)
    np.testing.assert_allclose(U.rho, 1.0, atol=1e-6)
    np.testing.assert_allclose(U.theta, 1.0, atol=1e-6)
    g2 = grid(n_x=2, n_v=16)
    half = np.random.default_rng(7).uniform(0.1, 1.0, size=(2, 8, 16, 16))
    assert np.all(P.project(P.Distribution(np.concatenate([half, half[:, ::-1]], axis=1)), g2).u[:, 0] == 0.0)
    g8 = grid(n_x=2, n_v=8)
    v = np.zeros((2, 8, 8, 8))
    v[:, 5, 2, 7] = 1.0 / g8.velocity.cell_volume
    U = P.project(P.Distribution(v), g8)
    c = g8.velocity.centers
    assert np.all(U.rho == 1.0) and np.all(U.theta == 0.0)
    assert list(U.u[0]) == [c[0][5], c[1][2], c[2][7]]
    with pytest.raises(P.DegenerateStateError):
        P.project(P.Distribution(np.zeros((2, 8, 8, 8))), g8)


def test_lift_nodewise_mass_and_fidelity():
    g = grid(n_x=2, n_v=8)
    rho, u, th = 0.7, (0.5, -0.3, 1.1), 0.9
    f = P.lift(uniform(2, rho, u, th), g).values
    c = g.velocity.centers
    for jx in (0, 3, 7):
        for jy in (1, 6):
            for jz in (0, 5):
                want = P.maxwellian(rho, u, th, (c[0][jx], c[1][jy], c[2][jz]))
                np.testing.assert_allclose(f[0, jx, jy, jz], want, rtol=1e-12)
    g32 = grid(n_x=2, n_v=32)
    U = uniform(2, 1.0, (0, 0, 0), 0.25)
    raw = P.lift(U, g32).values.sum(axis=(1, 2, 3)) * g32.velocity.cell_volume
    assert np.all(np.abs(raw - 1.0) < 1e-3)
    norm = P.lift(U, g32, normalize_mass=True).values.sum(axis=(1, 2, 3)) * g32.velocity.cell_volume
    np.testing.assert_allclose(norm, 1.0, rtol=1e-14)
    errs = [uniform(2, 1.0, (0.5, 0, -0.5), 0.8).sup_distance(
        P.project(P.lift(uniform(2, 1.0, (0.5, 0, -0.5), 0.8), grid(n_x=2, n_v=n)), grid(n_x=2, n_v=n)))
        for n in (16, 32)]
    assert errs[1] < errs[0]
    with pytest.raises(P.DegenerateStateError):
        P.lift(uniform(2, 0.0, (0, 0, 0), 1.0), g)
    with pytest.raises(P.DegenerateStateError):
        P.lift(uniform(2, 1.0, (0, 0, 0), -1.0), g)


def test_lift_project_round_trip_per_cell():
    g = grid(n_x=3, n_v=32)
    U = P.MomentField(np.array([0.5, 1.0, 2.0]), np.array([[0.0, 0, 0], [0.5, 0, 0], [-0.5, 0, 0]]),
                      np.array([0.5, 1.0, 2.0]))
    assert U.sup_distance(P.project(P.lift(U, g), g)) <= 1e-5


# --------------------------------------------------------------------- fluid

def test_fluid_constant_symmetry_conservation():
    g = grid(n_x=16, n_v=4)
    U = P.MomentField(np.full(16, 0.7), np.tile([0.3, 0, 0], (16, 1)), np.full(16, 1.2))
    assert U.sup_distance(P.propagate_fluid(U, 0.0, 0.3, g, P.FluidParams(), PER)) <= 1e-13
    g40 = grid(n_x=40, n_v=4)
    x = g40.space.centers
    rho = 1.0 + 0.5 * np.exp(-8.0 * (x - 1.0) ** 2)
    rho = 0.5 * (rho + rho[::-1])
    ux = np.sin(np.pi * x)
    ux = 0.5 * (ux - ux[::-1])
    out = P.propagate_fluid(P.MomentField(rho, np.stack([ux, 0 * x, 0 * x], 1), np.ones(40)), 0.0,
                            0.2, g40, P.FluidParams(), PER)
    assert np.array_equal(out.rho, out.rho[::-1])
    assert np.array_equal(out.u[:, 0], -out.u[::-1, 0])
    g50 = grid(n_x=50, n_v=4)
    U = sod(g50.space)
    V0 = P.primitive_to_conserved(U)
    V1 = P.primitive_to_conserved(P.propagate_fluid(U, 0.0, 1.0, g50, P.FluidParams(), PER, dt_max=2e-3))
    assert abs(math.fsum(V1.rho) - math.fsum(V0.rho)) <= 1e-13 * math.fsum(V0.rho)
    assert abs(math.fsum(V1.energy) - math.fsum(V0.energy)) <= 1e-13 * math.fsum(V0.energy)


def test_fluid_force_accounting_and_guards():
    g = grid(n_x=20, n_v=4)
    x = g.space.centers
    E = -5.0 * x ** 4 * (x - 2.0) ** 4 * (x - 1.0)
    U = P.MomentField(np.full(20, 2.0), np.stack([0.1 * np.sin(np.pi * x), 0 * x, 0 * x], 1),
                      np.ones(20))
    V0 = P.primitive_to_conserved(U)
    V1 = P.primitive_to_conserved(P.propagate_fluid(U, 0.0, 1e-3, g, P.FluidParams(force=E), PER))
    assert math.fsum(V1.mom[:, 0]) - math.fsum(V0.mom[:, 0]) == pytest.approx(
        1e-3 * math.fsum(2.0 * E), rel=1e-12)
    g4 = grid(n_x=4, n_v=4)
    U4 = P.MomentField(np.ones(4), np.zeros((4, 3)), np.ones(4))
    assert P.propagate_fluid(U4, 0.5, 0.5, g4, P.FluidParams(), PER) is U4
    with pytest.raises(P.ConfigurationError):
        P.propagate_fluid(U4, 1.0, 0.5, g4, P.FluidParams(), PER)
    g50 = grid(n_x=50, n_v=4)
    u = np.zeros((50, 3)); u[:, 0] = 1.0
    with pytest.raises(P.BlowUpError) as info:
        P.propagate_fluid(P.MomentField(np.ones(50), u, np.full(50, 1e-3)), 0.0, 1.0, g50,
                          P.FluidParams(force=np.full(50, -1000.0)), PER)
    assert info.value.step >= 1


@pytest.mark.parametrize("n_x,t", [(200, 0.05), (200, 0.1)])
def test_sod_density_matches_exact_riemann(n_x, t):
    g = grid(n_x=n_x, n_v=4)
    out = P.propagate_fluid(sod(g.space), 0.0, t, g, P.FluidParams(), ABS)
    exact = riemann.density((1.0, 0.0, 1.0), (0.125, 0.0, 0.1), (g.space.centers - 1.0) / t)
    assert float(np.sum(np.abs(out.rho - exact)) * g.space.dx) <= 0.05


# --------------------------------------------------------------------- parareal

def disc(n_g=4, n_f=16, n_x=12, n_v=8, bc=ABS, t_final=0.1, v_max=8.0):
    return P.Discretization(grid(n_x=n_x, n_v=n_v, v_max=v_max), P.build_time_grids(t_final, n_g, n_f), bc)


def test_coarse_sweep_is_the_composition_of_G():
    d = disc()
    U0 = sod(d.phase.space)
    traj = P.initial_coarse_sweep(U0, d, P.FluidParams())
    assert len(traj.snapshots) == 5 and traj.snapshots[0].sup_distance(U0) == 0.0
    U = U0
    for n in range(1, 5):
        U = P.propagate_fluid(U, float(d.time.coarse_times[n - 1]), float(d.time.coarse_times[n]),
                              d.phase, P.FluidParams(), d.bc, dt_max=d.time.dt_g)
        assert traj.snapshots[n].sup_distance(U) == 0.0


def test_jumps_vanish_on_equilibrium_and_last_window_only():
    d = disc(bc=PER, n_v=32)
    U = P.MomentField(np.ones(12), np.zeros((12, 3)), np.ones(12))
    traj = P.initial_coarse_sweep(U, d, P.FluidParams())
    P.compute_jumps(traj, 1, d, P.KineticParams(1e-2), P.FluidParams())
    for j in traj.jumps:
        assert max(abs(j.rho).max(), abs(j.u).max(), abs(j.theta).max()) <= 1e-12
    d2 = disc()
    traj = P.initial_coarse_sweep(sod(d2.phase.space), d2, P.FluidParams())
    P.compute_jumps(traj, 4, d2, P.KineticParams(1e-2), P.FluidParams())
    assert [bool(np.any(j.rho != 0.0)) for j in traj.jumps] == [False, False, False, True]


def test_frozen_prefix_fine_chain_and_equivalence():
    d = disc()
    kin, flu = P.KineticParams(1e-2), P.FluidParams()
    U0 = sod(d.phase.space)
    chain = P.fine_moment_chain(U0, d, kin)
    traj, _ = P.run_parareal(U0, P.PararealConfig(3, 1e-300), d, kin, flu)
    assert traj.frozen_upto == 3
    for n in range(4):
        assert traj.snapshots[n].sup_distance(chain[n]) <= 1e-13
    for k in (1, 2, 4):
        a, _ = P.run_parareal(U0, P.PararealConfig(k, 1e-300, True), d, kin, flu)
        b, _ = P.run_parareal(U0, P.PararealConfig(k, 1e-300, False), d, kin, flu)
        for x, y in zip(a.snapshots, b.snapshots):
            assert x.sup_distance(y) <= 1e-12


def test_stopping_sink_and_determinism():
    d = disc()
    kin, flu = P.KineticParams(1e-2), P.FluidParams()
    U0 = sod(d.phase.space)
    traj, rec = P.run_parareal(U0, P.PararealConfig(5, math.inf), d, kin, flu)
    assert len(rec) == 1 and traj.iteration == 1
    seen = []
    _, rec = P.run_parareal(U0, P.PararealConfig(3, 1e-300), d, kin, flu, sink=seen.append)
    assert [r.k for r in seen] == [1, 2, 3] and seen == rec
    a, ra = P.run_parareal(U0, P.PararealConfig(3, 1e-300, workers=1), d, kin, flu)
    b, rb = P.run_parareal(U0, P.PararealConfig(3, 1e-300, workers=2), d, kin, flu)
    assert [r.error for r in ra] == [r.error for r in rb]
    for x, y in zip(a.snapshots, b.snapshots):
        assert np.array_equal(x.rho, y.rho) and np.array_equal(x.u, y.u)


def test_overshoot_reports_slice_and_zero_jumps_zero_error():
    d = disc()
    traj = P.initial_coarse_sweep(sod(d.phase.space), d, P.FluidParams())
    assert P.sequential_correction(traj, 1, d, P.FluidParams()) == 0.0
    traj = P.initial_coarse_sweep(sod(d.phase.space), d, P.FluidParams())
    traj.jumps[2].rho[:] = -10.0
    with pytest.raises(P.CorrectionOvershootError) as info:
        P.sequential_correction(traj, 1, d, P.FluidParams())
    assert info.value.slice_index == 3


# --------------------------------------------------------------------- acceptance

def test_acceptance_parareal_reproduces_fine_chain_and_first_window():
    d = disc(n_g=8, n_f=32, n_x=20, v_max=5.0)
    kin, flu = P.KineticParams(1e-2), P.FluidParams()
    U0 = sod(d.phase.space)
    chain = P.fine_moment_chain(U0, d, kin)
    traj, _ = P.run_parareal(U0, P.PararealConfig(8, 1e-300), d, kin, flu)
    assert max(a.sup_distance(b) for a, b in zip(traj.snapshots, chain)) <= 1e-10
    t1, _ = P.run_parareal(U0, P.PararealConfig(1, 1e-300), d, kin, flu)
    f = P.propagate_kinetic(P.lift(U0, d.phase), 0.0, float(d.time.coarse_times[1]), d.phase, kin,
                            d.bc, dt_max=d.time.dt_f)
    assert t1.snapshots[1].sup_distance(P.project(f, d.phase)) <= 1e-12


def test_acceptance_exponential_convergence():
    d = disc(n_g=50, n_f=200, n_x=50, n_v=16, t_final=0.25)
    _, rec = P.run_parareal(sod(d.phase.space), P.PararealConfig(10, 1e-300), d, P.KineticParams(1e-2),
                            P.FluidParams())
    e = [r.error for r in rec]
    assert len(e) == 10 and all(e[i + 1] < e[i] for i in range(7))
    k = np.arange(1, 11)
    y = np.log10(e)
    s, c = np.polyfit(k, y, 1)
    res = y - (s * k + c)
    assert s < 0 and 1 - (res @ res) / ((y - y.mean()) @ (y - y.mean())) > 0.9


def test_acceptance_kinetic_mass_conservation_500_steps():
    g = P.PhaseGrid(P.build_spatial_grid(0.0, 2.0, 30), P.build_velocity_grid(8.0, (16, 8, 8)))
    f = P.lift(sod(g.space), g)
    cell = g.velocity.cell_volume * g.space.dx
    m0 = float(f.values.sum()) * cell
    f = P.propagate_kinetic(f, 0.0, 0.1, g, P.KineticParams(1e-2), PER, dt_max=0.1 / 500)
    assert abs(float(f.values.sum()) * cell - m0) / m0 <= 1e-12


def test_acceptance_ap_trend_in_epsilon():
    g = grid(n_x=100, n_v=16)
    x = g.space.centers
    u = np.zeros((100, 3)); u[:, 0] = 0.2 * np.sin(np.pi * x)
    U0 = P.MomentField(np.ones(100), u, 2.0 * np.ones(100))
    ref = P.propagate_fluid(U0, 0.0, 0.05, g, P.FluidParams(), PER)
    gaps = []
    for eps in (1e-1, 1e-2, 1e-3):
        f = P.propagate_kinetic(P.lift(U0, g), 0.0, 0.05, g, P.KineticParams(eps), PER)
        gaps.append(float(np.abs(P.project(f, g).rho - ref.rho).sum() * g.space.dx))
    assert gaps[0] > gaps[1] > gaps[2]


def test_acceptance_confined_beams_with_force():
    g = P.PhaseGrid(P.build_spatial_grid(0.0, 2.0, 50), P.build_velocity_grid(6.0, (64, 8, 8)))
    d = P.Discretization(g, P.build_time_grids(0.5, 8, 240), PER)
    x = g.space.centers
    E = -5.0 * x ** 4 * (x - 2.0) ** 4 * (x - 1.0)
    ones = np.ones(50)
    uf = np.zeros((50, 3)); uf[:, 0] = 1.0
    beams = P.lift(P.MomentField(ones, uf, ones), g).values + P.lift(P.MomentField(ones, -uf, ones), g).values
    U0 = P.project(P.Distribution(beams), g)
    kin, flu = P.KineticParams(1e-3, force=E), P.FluidParams(force=E)
    chain = P.fine_moment_chain(U0, d, kin)
    traj, _ = P.run_parareal(U0, P.PararealConfig(6, 1e-300), d, kin, flu)
    assert max(a.sup_distance(b) for a, b in zip(traj.snapshots, chain)) <= 1e-4
    fin = traj.snapshots[-1]
    assert abs(x[int(np.argmax(fin.rho))] - 1.0) <= 0.1
    assert fin.rho.max() > 1.05 * U0.rho.max()
