"""Round-2 pass kernel of the multi-step path (msweep.cu, include/pbgk.h
pbgk_set_msweep): 4 or 8 fine steps per pass over f, the window's final
relax + projection folded into its last pass.

Parity as for the round-1 kernel (tests/test_gpu_fused.py): the oracle's F
(ref/kinetic.py:137-161) from L(U) or a given f0 to 1e-12 on f_S and on the
moments, the one-step path to 1e-13 (transport and relax re-associated, a few
ulps per step), every boundary, pass counts that are not multiples of L, a
single pass that both synthesises L(U) and projects, batched windows, the
concurrent recursion, failure keys equal to the one-step path's."""

import numpy as np
import pytest
import torch

from oracle import bgk as O
from helpers import moment_gap, random_moments, rel_inf

pytestmark = pytest.mark.gpu
P = pytest.importorskip("paper_2502_02704_b200")
from paper_2502_02704_b200 import runtime as rt  # noqa: E402
from paper_2502_02704_b200.kinetic import _run_schedule, fine_schedule, stable_dt_kinetic  # noqa: E402

SHAPES = [
    (10, (16, 16, 16), 8.0),
    (9, (32, 32, 32), 8.0),
    (7, (48, 48, 48), 10.0),
    (5, (64, 64, 64), 8.0),
    (6, (32, 16, 48), 7.0),
]
BCS = ["periodic", "absorbing", "outflow"]
LEVELS = [4, 8]


def _grids(nx, nv, vm):
    g = P.PhaseGrid(P.build_spatial_grid(0.0, 1.0, nx), P.build_velocity_grid(vm, nv))
    return g, O.Mesh(0.0, 1.0, nx, vm, nv)


def _unpack(m):
    return m[0], m[1:4].T, m[4]


def _window(g, bc, U, t1, levels, kp=None, want_f=True):
    """f_S and P(f_S) of one window from moments U; levels 0 = one-step path."""
    kp = kp or P.KineticParams(1e-2)
    ctx = rt.ctx_for(g, P.BoundaryKind(bc))
    m0 = rt.to_device_moments(P.MomentField(*U), ctx.device)
    dts = fine_schedule(t1, stable_dt_kinetic(g, kp))
    out, mo = ctx.empty_f(), ctx.empty_moments()
    if levels == 0:
        with ctx.fusion_levels(0):
            code = _run_schedule(ctx, None, m0, dts, kp, out, want_f=want_f, mom_out=mo)
    else:
        with ctx.msweep_mode(True, levels):
            assert ctx.msweep_levels() == levels
            code = _run_schedule(ctx, None, m0, dts, kp, out, want_f=want_f, mom_out=mo)
    torch.cuda.synchronize()
    return out.cpu().numpy(), mo.cpu().numpy(), code, len(dts)


def _from_f0(g, bc, f0, t1, levels):
    kp = P.KineticParams(1e-2)
    ctx = rt.ctx_for(g, P.BoundaryKind(bc))
    fd = torch.from_numpy(np.ascontiguousarray(f0)).to(ctx.device)
    dts = fine_schedule(t1, stable_dt_kinetic(g, kp))
    out = ctx.empty_f()
    if levels == 0:
        with ctx.fusion_levels(0):
            code = _run_schedule(ctx, fd, None, dts, kp, out)
    else:
        with ctx.msweep_mode(True, levels):
            code = _run_schedule(ctx, fd, None, dts, kp, out)
    torch.cuda.synchronize()
    return out.cpu().numpy(), code


@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: "x".join(map(str, (s[0],) + s[1])))
@pytest.mark.parametrize("bc", BCS)
@pytest.mark.parametrize("levels", LEVELS)
@pytest.mark.parametrize("steps", [7, 19])
def test_window_matches_oracle(shape, bc, levels, steps):
    nx, nv, vm = shape
    g, mesh = _grids(nx, nv, vm)
    U = random_moments(nx, np.random.default_rng(nx + len(bc) + steps))
    t1 = (steps - 0.5) * O.fine_cap(mesh, 0.5, None)  # the last step partial
    f, m, code, S = _window(g, bc, U, t1, levels)
    assert code == -1 and S == steps
    want_f = O.fine_propagate(O.lift(*U, mesh), 0.0, t1, mesh, 1e-2, bc)
    assert rel_inf(f, want_f) <= 1e-12
    assert moment_gap(_unpack(m), O.project(want_f, mesh)) <= 1e-12
    f1, m1, c1, _ = _window(g, bc, U, t1, 0)
    assert c1 == -1
    assert rel_inf(f, f1) <= 1e-13
    assert moment_gap(_unpack(m), _unpack(m1)) <= 1e-13


@pytest.mark.parametrize("levels", LEVELS)
def test_projection_only_window(levels):
    # the parareal fine stage: no f_S stored, P(f_S) from the last pass's partials
    g, mesh = _grids(8, (32, 32, 32), 8.0)
    U = random_moments(8, np.random.default_rng(4))
    t1 = 12.5 * O.fine_cap(mesh, 0.5, None)
    _, m, code, _ = _window(g, "outflow", U, t1, levels, want_f=False)
    assert code == -1
    want = O.project(O.fine_propagate(O.lift(*U, mesh), 0.0, t1, mesh, 1e-2, "outflow"), mesh)
    assert moment_gap(_unpack(m), want) <= 1e-12


@pytest.mark.parametrize("shape", SHAPES[:4], ids=lambda s: "x".join(map(str, (s[0],) + s[1])))
@pytest.mark.parametrize("bc", BCS)
@pytest.mark.parametrize("levels", LEVELS)
def test_given_f0_matches_oracle(shape, bc, levels):
    nx, nv, vm = shape
    g, mesh = _grids(nx, nv, vm)
    rng = np.random.default_rng(11 * nx)
    f0 = O.lift(*random_moments(nx, rng), mesh) * rng.uniform(0.8, 1.2, (nx,) + nv)
    t1 = 10.5 * O.fine_cap(mesh, 0.5, None)
    want = O.fine_propagate(f0, 0.0, t1, mesh, 1e-2, bc)
    got, c = _from_f0(g, bc, f0, t1, levels)
    one, c0 = _from_f0(g, bc, f0, t1, 0)
    assert c == c0 == -1
    assert rel_inf(got, want) <= 1e-12
    assert rel_inf(got, one) <= 1e-13


@pytest.mark.parametrize("levels", LEVELS)
def test_even_data_keeps_exact_zero_velocity(levels):
    # x-homogeneous, velocity-even data: every marginal stays mirror-symmetric
    # through the passes and the folded projection (ref/moments.py:80-88)
    nx = 6
    g, _ = _grids(nx, (32, 32, 32), 8.0)
    U = (np.full(nx, 1.3), np.zeros((nx, 3)), np.full(nx, 0.9))
    t1 = 11.0 * stable_dt_kinetic(g, P.KineticParams(1e-2))
    _, m, code, _ = _window(g, "periodic", U, t1, levels, want_f=False)
    assert code == -1
    assert np.all(m[1:4] == 0.0)


@pytest.mark.parametrize("levels", LEVELS)
@pytest.mark.parametrize("bad", [np.nan, -0.5])
def test_failure_keys_equal_one_step_path(levels, bad):
    g, _ = _grids(8, (16, 16, 16), 8.0)
    t1 = 10.5 * stable_dt_kinetic(g, P.KineticParams(1e-2))
    rho, u, th = random_moments(8, np.random.default_rng(5))
    rho[3] = bad
    _, _, c0, _ = _window(g, "outflow", (rho, u, th), t1, 0)
    _, _, c, _ = _window(g, "outflow", (rho, u, th), t1, levels)
    assert c0 != -1
    assert c == c0


@pytest.mark.parametrize("levels", LEVELS)
def test_given_f0_non_finite_reports_step_one(levels):
    g, mesh = _grids(8, (16, 16, 16), 8.0)
    f0 = O.lift(*random_moments(8, np.random.default_rng(2)), mesh)
    f0[2, 3, 4, 5] = np.nan
    t1 = 9.5 * O.fine_cap(mesh, 0.5, None)
    _, c0 = _from_f0(g, "periodic", f0, t1, 0)
    _, c = _from_f0(g, "periodic", f0, t1, levels)
    assert c0 != -1 and c == c0
    with pytest.raises(P.BlowUpError) as info:
        rt.raise_kinetic(c)
    assert info.value.step == 1


@pytest.mark.parametrize("levels", LEVELS)
@pytest.mark.parametrize("bc", ["outflow", "periodic", "absorbing"])
def test_batched_windows_equal_one_step_path(levels, bc):
    # pbgk_propagate_windows: the batched recursion, then each window's msweep
    # passes; windows of different lengths, an empty one, a failing one
    from paper_2502_02704_b200.kinetic import propagate_windows
    g, mesh = _grids(10, (16, 16, 16), 8.0)
    kp = P.KineticParams(1e-2)
    ctx = rt.ctx_for(g, P.BoundaryKind(bc))
    cap = stable_dt_kinetic(g, kp)
    spans = [17.5 * cap, 4.0 * cap, 0.0, 9.2 * cap, 8.0 * cap]
    rng = np.random.default_rng(9)
    Us = [random_moments(10, rng) for _ in spans]
    Us[3][0][4] = np.nan  # window 3 fails (BlowUpError at some step)
    mom_in = torch.stack([rt.to_device_moments(P.MomentField(*U), ctx.device) for U in Us])
    res = {}
    for L in (0, levels):
        out = ctx.empty_moments(len(spans))
        if L == 0:
            with ctx.fusion_levels(0):
                codes = propagate_windows(ctx, mom_in, spans, g, kp, None, out)
        else:
            with ctx.msweep_mode(True, L):
                codes = propagate_windows(ctx, mom_in, spans, g, kp, None, out)
        res[L] = (out.cpu().numpy(), codes)
    (m0, c0), (m1, c1) = res[0], res[levels]
    assert c1 == c0 and c0[3] != -1 and c0[2] == -1
    for w in (0, 1, 2, 4):
        assert moment_gap(_unpack(m1[w]), _unpack(m0[w])) <= 1e-13
    want = O.project(O.fine_propagate(O.lift(*Us[0], mesh), 0.0, spans[0], mesh, 1e-2, bc), mesh)
    assert moment_gap(_unpack(m1[0]), want) <= 1e-12


@pytest.mark.parametrize("bc", BCS)
@pytest.mark.parametrize("levels", LEVELS)
def test_long_propagation_concurrent_recursion(bc, levels):
    # >= 8 L steps on a small grid: the recursion on a side stream on reserved
    # SMs, the producer warp of each pass waiting on its progress word
    g, mesh = _grids(24, (32, 32, 32), 8.0)
    rng = np.random.default_rng(17)
    f0 = O.lift(*random_moments(24, rng), mesh) * rng.uniform(0.9, 1.1, (24, 32, 32, 32))
    t1 = 70.5 * O.fine_cap(mesh, 0.5, None)  # 71 steps
    one, c0 = _from_f0(g, bc, f0, t1, 0)
    got, c = _from_f0(g, bc, f0, t1, levels)
    assert c == c0 == -1
    assert rel_inf(got, one) <= 1e-12


def test_parareal_equals_one_step_path():
    from dataclasses import replace
    from paper_2502_02704_b200.configs import config
    w = replace(config(0), outflow=True)
    g = P.PhaseGrid(P.build_spatial_grid(w.x_min, w.x_max, w.nx), P.build_velocity_grid(w.v_max, w.nv))
    bc = P.BoundaryKind(w.bc)
    d = P.Discretization(g, P.build_time_grids(w.t_final, w.n_g, w.n_f), bc)
    U0 = P.project(P.lift(P.MomentField(*w.raw_moments()), g, bc=bc), g, bc=bc)
    cfg = P.PararealConfig(w.k_max, w.tol)
    ctx = rt.ctx_for(g, bc)
    with ctx.fusion_levels(0):
        t0, r0 = P.run_parareal(U0, cfg, d, P.KineticParams(w.eps), P.FluidParams())
    for L in LEVELS:
        with ctx.msweep_mode(True, L):
            t, r = P.run_parareal(U0, cfg, d, P.KineticParams(w.eps), P.FluidParams())
        assert len(r) == len(r0)
        for a, b in zip(t.snapshots, t0.snapshots):
            assert moment_gap((a.rho, a.u, a.theta), (b.rho, b.u, b.theta)) <= 1e-12


@pytest.mark.parametrize("levels", LEVELS)
def test_batched_windows_in_groups(levels):
    # a table budget of about two windows (pbgk_set_batch_bytes): the batched
    # recursion runs in groups of two, the empty and the failing window in the
    # second group; results as on one group and as on the one-step path
    from paper_2502_02704_b200.kinetic import propagate_windows
    g, mesh = _grids(10, (16, 16, 16), 8.0)
    kp = P.KineticParams(1e-2)
    ctx = rt.ctx_for(g, P.BoundaryKind.OUTFLOW)
    cap = stable_dt_kinetic(g, kp)
    spans = [17.5 * cap, 4.0 * cap, 0.0, 9.2 * cap, 8.0 * cap]
    rng = np.random.default_rng(13)
    Us = [random_moments(10, rng) for _ in spans]
    Us[3][0][4] = np.nan
    mom_in = torch.stack([rt.to_device_moments(P.MomentField(*U), ctx.device) for U in Us])
    smax = 18
    per_window = 8.0 * ((smax + 1) * 10 * P_table_len(ctx) + 2 * 10 * 5 * 16 + 12 * 10)
    res = []
    for budget in (0.0, 2.2 * per_window):
        ctx.set_batch_bytes(budget)
        out = ctx.empty_moments(len(spans))
        with ctx.msweep_mode(True, levels):
            codes = propagate_windows(ctx, mom_in, spans, g, kp, None, out)
        res.append((out.cpu().numpy(), codes))
    ctx.set_batch_bytes(0.0)
    with ctx.fusion_levels(0):
        out = ctx.empty_moments(len(spans))
        c0 = propagate_windows(ctx, mom_in, spans, g, kp, None, out)
        m0 = out.cpu().numpy()
    (ma, ca), (mb, cb) = res
    assert ca == cb == c0 and c0[3] != -1 and c0[2] == -1
    for w in (0, 1, 2, 4):
        assert np.array_equal(ma[w], mb[w])  # grouping does not change a window's arithmetic
        assert moment_gap(_unpack(mb[w]), _unpack(m0[w])) <= 1e-13


@pytest.mark.parametrize("levels", LEVELS)
@pytest.mark.parametrize("bc", BCS)
@pytest.mark.parametrize("nsteps", [3.5, 8.0, 21.3])
def test_equal_windows_run_as_one_batch(levels, bc, nsteps, monkeypatch):
    # windows of equal step counts on a small grid: every pass is ONE launch
    # over all windows (grid.y = window, capi.cu ms_windows_batched).  Same
    # arithmetic per window as the window-by-window passes (bitwise), the
    # oracle's P(F(L(U))) (ref/parareal.py:123-142) to 1e-12, a failing window
    # keeps its one-step key and does not disturb its neighbours
    from paper_2502_02704_b200.kinetic import propagate_windows
    g, mesh = _grids(10, (16, 16, 16), 8.0)
    kp = P.KineticParams(1e-2)
    ctx = rt.ctx_for(g, P.BoundaryKind(bc))
    cap = stable_dt_kinetic(g, kp)
    spans = [nsteps * cap] * 5
    rng = np.random.default_rng(31)
    Us = [random_moments(10, rng) for _ in spans]
    Us[2][0][7] = np.nan
    mom_in = torch.stack([rt.to_device_moments(P.MomentField(*U), ctx.device) for U in Us])
    res = []
    for nobatch in (False, True):
        if nobatch:
            monkeypatch.setenv("PBGK_NO_WBATCH", "1")
        out = ctx.empty_moments(len(spans))
        with ctx.msweep_mode(True, levels):
            codes = propagate_windows(ctx, mom_in, spans, g, kp, None, out)
        res.append((out.cpu().numpy(), codes))
    monkeypatch.delenv("PBGK_NO_WBATCH")
    with ctx.fusion_levels(0):
        out = ctx.empty_moments(len(spans))
        c0 = propagate_windows(ctx, mom_in, spans, g, kp, None, out)
    (ma, ca), (mb, cb) = res
    assert ca == cb == c0 and c0[2] != -1 and all(c0[w] == -1 for w in (0, 1, 3, 4))
    for w in (0, 1, 3, 4):
        assert np.array_equal(ma[w], mb[w])
        want = O.project(O.fine_propagate(O.lift(*Us[w], mesh), 0.0, spans[w], mesh, 1e-2, bc), mesh)
        assert moment_gap(_unpack(ma[w]), want) <= 1e-12


def P_table_len(ctx):
    return int(ctx.lib.pbgk_table_len(ctx.h))


@pytest.mark.parametrize("levels", LEVELS)
def test_high_transverse_mach_matches_oracle(levels):
    # the recursion's one-pass transverse variance Q2 - 2 u Q1 + u^2 Q0 loses
    # about log10(u^2 / theta) digits: a drifting cold state (|u_y| / sqrt
    # theta = 10, |u_z| / sqrt theta = 8) must still match the oracle's
    # two-pass projection (ref/moments.py:108-112)
    nx = 8
    g, mesh = _grids(nx, (32, 32, 32), 8.0)
    rng = np.random.default_rng(23)
    rho = rng.uniform(0.8, 1.2, nx)
    th = rng.uniform(0.36, 0.44, nx)
    u = np.zeros((nx, 3))
    u[:, 0] = rng.uniform(-0.3, 0.3, nx)
    u[:, 1] = 10.0 * np.sqrt(th) * rng.choice([-1.0, 1.0], nx)
    u[:, 2] = 8.0 * np.sqrt(th)
    t1 = 19.5 * O.fine_cap(mesh, 0.5, None)
    for bc in ("periodic", "outflow"):
        f, m, code, _ = _window(g, bc, (rho, u, th), t1, levels)
        assert code == -1
        want_f = O.fine_propagate(O.lift(rho, u, th, mesh), 0.0, t1, mesh, 1e-2, bc)
        assert rel_inf(f, want_f) <= 1e-12
        assert moment_gap(_unpack(m), O.project(want_f, mesh)) <= 1e-12


def test_release_contexts_frees_and_recreates():
    g, mesh = _grids(6, (16, 16, 16), 8.0)
    U = random_moments(6, np.random.default_rng(3))
    t1 = 9.5 * O.fine_cap(mesh, 0.5, None)
    _, m1, c1, _ = _window(g, "periodic", U, t1, 8)
    assert P.release_contexts() >= 1
    _, m2, c2, _ = _window(g, "periodic", U, t1, 8)  # a fresh context
    assert c1 == c2 == -1 and np.array_equal(m1, m2)


@pytest.mark.parametrize("levels", LEVELS)
@pytest.mark.parametrize("bc", BCS)
def test_precomputed_row_factors_are_bitwise_the_in_kernel_ones(levels, bc, monkeypatch):
    # the per-row factors (ls gxa, keep r, a r) of every step come from a small
    # kernel once per window (msweep.cu ms_prep_kernel) or, with PBGK_MS_NOPRE
    # and under a concurrent recursion, are formed in the pass kernel: the same
    # rounded operations, so f_S and P(f_S) agree bit for bit (19 steps: a
    # ragged last pass; from moments and from a given f0)
    g, mesh = _grids(9, (32, 16, 48), 7.0)
    U = random_moments(9, np.random.default_rng(77))
    t1 = 18.5 * O.fine_cap(mesh, 0.5, None)
    f_a, m_a, c_a, _ = _window(g, bc, U, t1, levels)
    g0, _ = _from_f0(g, bc, f_a * 1.0, 6.5 * O.fine_cap(mesh, 0.5, None), levels)
    monkeypatch.setenv("PBGK_MS_NOPRE", "1")
    f_b, m_b, c_b, _ = _window(g, bc, U, t1, levels)
    g1, _ = _from_f0(g, bc, f_a * 1.0, 6.5 * O.fine_cap(mesh, 0.5, None), levels)
    monkeypatch.delenv("PBGK_MS_NOPRE")
    assert c_a == c_b == -1
    assert np.array_equal(f_a, f_b) and np.array_equal(m_a, m_b) and np.array_equal(g0, g1)
