"""Host-side logic of the drop-in package (no device needed)."""

import numpy as np
import pytest

from oracle import bgk as O

import paper_2502_02704_b200 as P
from paper_2502_02704_b200 import runtime as rt
from paper_2502_02704_b200.configs import config, reduced
from paper_2502_02704_b200.kinetic import fine_schedule, tau_constant


def test_grids_match_reference_arithmetic():
    for nx, nv, vm in [(64, 16, 8.0), (7, (9, 5, 4), 6.0)]:
        g = P.PhaseGrid(P.build_spatial_grid(0.0, 1.0, nx), P.build_velocity_grid(vm, nv))
        m = O.Mesh(0.0, 1.0, nx, vm, (nv,) * 3 if np.isscalar(nv) else nv)
        assert g.space.dx == m.dx and np.array_equal(g.space.centers, m.xc)
        for a in range(3):
            assert g.velocity.dv[a] == m.dv[a]
            assert np.array_equal(g.velocity.centers[a], m.vc[a])
            assert np.array_equal(g.velocity.centers[a], -g.velocity.centers[a][::-1])
        assert g.velocity.cell_volume == m.dvol
    t = P.build_time_grids(0.1, 8, 8)
    assert t.coarse_times[-1] == 0.1 and t.dt_g == 0.1 / 8


def test_grid_validation():
    with pytest.raises(P.ConfigurationError):
        P.build_spatial_grid(1.0, 0.0, 4)
    with pytest.raises(P.ConfigurationError):
        P.build_spatial_grid(0.0, 1.0, 1)
    with pytest.raises(P.ConfigurationError):
        P.build_velocity_grid(-1.0, 8)
    with pytest.raises(P.ConfigurationError):
        P.build_time_grids(0.1, 4, 2)


def test_stable_dt_and_schedule():
    g = P.PhaseGrid(P.build_spatial_grid(0.0, 2.0, 200), P.build_velocity_grid(8.0, 8))
    assert P.stable_dt_kinetic(g, P.KineticParams(1.0, cfl=0.9)) == 0.9 * 0.01 / 8.0
    g2 = P.PhaseGrid(P.build_spatial_grid(0.0, 2.0, 100), P.build_velocity_grid(8.0, (256, 8, 8)))
    assert P.stable_dt_kinetic(g2, P.KineticParams(1.0, force=np.full(100, 0.8))) == \
        0.5 / (8.0 / 0.02 + 0.8 / 0.0625)
    for span, cap in [(0.2, 2.44140625e-4), (3.5e-3, 1e-3), (1.0 / 1024, 3.0517578125e-5)]:
        assert fine_schedule(span, cap) == O.fine_schedule(0.0, span, cap)
    # config 1: 820 steps, last one partial
    d = fine_schedule(0.2, 0.5 / (8.0 * 256))
    assert len(d) == 820 and d[-1] == pytest.approx(4.88281250000111e-05, rel=1e-12)


def test_config_window_steps():
    expect = {0: 13, 1: 820, 2: 32, 3: 26, 4: 32}
    for idx, n in expect.items():
        w = config(idx)
        assert w.window_steps() == n, (idx, w.window_steps())
        m = O.Mesh(w.x_min, w.x_max, w.nx, w.v_max, w.nv)
        cap = O.fine_cap(m, 0.5, w.force())
        if w.mode == "parareal":
            cap = min(cap, w.t_final / w.n_f)
            span = w.t_final / w.n_g
        else:
            span = w.t_final
        assert len(O.fine_schedule(0.0, span, cap)) == n
    assert config(4).bc == "outflow" and config(1).bc == "periodic"
    r = reduced(config(2), 64, 12)
    assert r.nv == (12, 12, 12) and r.init == "sod_noise"


def test_work_distribution_and_cost_model():
    assert [P.work_distribution(10, 3, r)[:2] for r in range(3)] == [(1, 4), (5, 7), (8, 10)]
    e = P.work_distribution(5, 8, 5)
    assert (e.start, e.end, e.size) == (6, 5, 0)
    for work in range(0, 40):
        for n_p in range(1, 9):
            own = []
            for r in range(n_p):
                w = P.work_distribution(work, n_p, r)
                own += list(range(w.start, w.end + 1))
                assert w == P.WorkRange(*O.work_range(work, n_p, r))
            assert own == list(range(1, work + 1))
    with pytest.raises(P.ConfigurationError):
        P.work_distribution(3, 0, 0)
    assert P.estimate_k_opt(10.0, 0.1, 0.05, 0.05, 100, 32) == 24
    assert P.estimate_k_opt(10.0, 0.0, 0.0, 0.0, 100, 1) == 1


def test_parareal_config_validation():
    for bad in [dict(k_max=0, tol=1e-8), dict(k_max=1, tol=0.0), dict(k_max=1, tol=1e-8, workers=0)]:
        with pytest.raises(P.ConfigurationError):
            P.PararealConfig(**bad)


def test_moment_algebra_and_conversions():
    a = P.MomentField(np.ones(3), np.tile([0.5, 0, 0], (3, 1)), np.ones(3))
    b = P.MomentField(np.full(3, 0.25), np.tile([0.1, 0, 0], (3, 1)), np.full(3, 0.5))
    assert np.all((a + b).rho == 1.25) and np.all((a - b).theta == 0.5)
    assert a.sup_distance(b) == 0.75 and a.sup_distance(a.copy()) == 0.0
    V = P.primitive_to_conserved(P.MomentField(np.ones(1), np.array([[1.0, 0, 0]]), np.array([2.0])))
    assert V.energy[0] == 3.5
    with pytest.raises(P.DegenerateStateError):
        P.conserved_to_primitive(P.ConservedField(np.ones(1), np.zeros((1, 3)), np.zeros(1)))
    rng = np.random.default_rng(3)
    U = P.MomentField(rng.uniform(0.1, 3, 20), rng.uniform(-2, 2, (20, 3)), rng.uniform(0.05, 4, 20))
    assert U.sup_distance(P.conserved_to_primitive(P.primitive_to_conserved(U))) <= 4e-13
    packed = rt.pack_moments_np(U.rho, U.u, U.theta)
    W = P.MomentField.from_packed(packed)
    assert np.array_equal(W.rho, U.rho) and np.array_equal(W.u, U.u)


def test_fluid_flux_helpers():
    def packed(r, ux, t):
        return P.primitive_to_conserved(P.MomentField(np.array([r]), np.array([[ux, 0, 0]]),
                                                      np.array([t]))).to_array()[0]
    assert list(P.euler_flux(packed(1.0, 0.0, 1.0))) == [0.0, 1.0, 0.0, 0.0, 0.0]
    np.testing.assert_allclose(P.rusanov_flux(packed(1.0, 0.0, 1.0), packed(0.125, 0.0, 0.8)),
                               [0.4375, 0.55, 0.0, 0.0, 0.675], rtol=1e-15)
    v = packed(0.9, 0.4, 1.3)
    np.testing.assert_allclose(P.rusanov_flux(v, v), P.euler_flux(v), rtol=1e-15)
    assert P.rusanov_flux(packed(0.7, 0.9, 1.1), packed(0.7, -0.9, 1.1))[0] == 0.0


def test_status_keys_map_to_reference_exceptions():
    key = lambda unit, step, kind: (unit << 40) | (step << 8) | kind  # noqa: E731
    rt.raise_kinetic(-1)
    with pytest.raises(P.DegenerateStateError):
        rt.raise_kinetic(key(0, 3, 0))
    with pytest.raises(P.DegenerateStateError):
        rt.raise_kinetic(key(0, 0, 1))
    with pytest.raises(P.BlowUpError) as e:
        rt.raise_kinetic(key(0, 7, 2))
    assert e.value.step == 7
    with pytest.raises(P.CorrectionOvershootError) as e:
        rt.raise_fluid(key(3, 0, 4))
    assert e.value.slice_index == 3
    with pytest.raises(P.BlowUpError) as e:
        rt.raise_fluid(key(2, 5, 3))
    assert e.value.step == 5


def test_tau_detection():
    assert tau_constant(P.constant_tau) == 1.0
    assert tau_constant(P.ConstantTau(2.5)) == 2.5
    assert tau_constant(lambda r, t: 1.0) is None


def test_distribution_host_authority():
    f = np.ones((2, 2, 2, 2))
    d = P.Distribution(f)
    assert d.values is f and not d.is_device
    d.values[0, 0, 0, 0] = 5.0
    assert d.copy().values[0, 0, 0, 0] == 5.0


def test_no_cpu_fallback_without_device(monkeypatch):
    import torch
    monkeypatch.setattr(torch.cuda, "is_available", lambda: False)
    g = P.PhaseGrid(P.build_spatial_grid(0.0, 1.0, 4), P.build_velocity_grid(8.0, 8))
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        P.project(P.Distribution(np.ones((4, 8, 8, 8))), g)


from hypothesis import given, settings, strategies as st  # noqa: E402


@settings(max_examples=200, deadline=None)
@given(st.integers(0, 5000), st.integers(1, 64))
def test_partition_property(work, n_p):
    # ref tests/test_parareal.py:199-230: exhaustive, contiguous, balanced
    sizes, prev_end = [], 0
    for r in range(n_p):
        w = P.work_distribution(work, n_p, r)
        assert w.start == prev_end + 1
        prev_end = w.end if w.size else prev_end
        sizes.append(w.size)
        assert w == P.WorkRange(*O.work_range(work, n_p, r))
    assert sum(sizes) == work and max(sizes) - min(sizes) <= 1


@settings(max_examples=100, deadline=None)
@given(st.integers(1, 80), st.integers(1, 80), st.integers(1, 9))
def test_pipelined_rounds_cover_each_window_once(n_g, k, world):
    # PipelinedRun deals windows k..n_g cyclically, one per rank per round
    start = min(k, n_g)
    windows = list(range(start, n_g + 1))
    rounds = [windows[i:i + world] for i in range(0, len(windows), world)]
    mine = [[wr[r] for wr in rounds if r < len(wr)] for r in range(world)]
    assert sorted(sum(mine, [])) == windows
    assert all(r == sorted(r) for r in mine)


def test_velocity_centres_odd_symmetric_bitwise():
    # ref tests/test_grid.py:47-52
    for n in (1, 2, 7, 8, 16, 33, 48, 64):
        c = P.build_velocity_grid(8.0, n).centers[0]
        assert np.array_equal(c, -c[::-1])
