"""Multi-step path (fsweep.cu + marginal.cu, include/pbgk.h pbgk_set_fusion):
windows from moments advanced L fine steps per pass over f, with the relax
tables of every step from the 2-D marginal recursion.

Parity: the oracle's F (ref/kinetic.py:137-161) from L(U) to 1e-12 on f_S and
on the moments, the one-step path to 1e-13 (the marginal summation order and
the transport's association differ), every boundary, both quadratures, 1-4 levels and ragged pass counts;
the status keys (step and kind of a failure) equal to the one-step path's."""

import numpy as np
import pytest
import torch

from oracle import bgk as O
from helpers import moment_gap, random_moments, rel_inf

pytestmark = pytest.mark.gpu
P = pytest.importorskip("paper_2502_02704_b200")
from paper_2502_02704_b200 import runtime as rt  # noqa: E402
from paper_2502_02704_b200.kinetic import _run_schedule, fine_schedule, stable_dt_kinetic  # noqa: E402

# one per multi-step tile shape (nvz % 64, 48, 32, 16, 8) plus a generic shape
# that falls back to the one-step path
SHAPES = [
    (12, (8, 8, 8), 8.0),
    (10, (16, 16, 16), 8.0),
    (9, (32, 32, 32), 8.0),
    (7, (48, 48, 48), 10.0),
    (5, (64, 64, 64), 8.0),
    (10, (64, 8, 8), 6.0),
    (8, (16, 8, 6), 5.0),
]
BCS = ["periodic", "absorbing", "outflow"]


def _grids(nx, nv, vm, quad="midpoint"):
    g = P.PhaseGrid(P.build_spatial_grid(0.0, 1.0, nx), P.build_velocity_grid(vm, nv, quadrature=quad))
    return g, O.Mesh(0.0, 1.0, nx, vm, nv, quadrature=quad)


def _window(g, bc, U, t1, levels, kp=None):
    """f_S and P(f_S) of one window from moments U on `levels` steps per pass."""
    kp = kp or P.KineticParams(1e-2)
    ctx = rt.ctx_for(g, P.BoundaryKind(bc))
    m0 = rt.to_device_moments(P.MomentField(*U), ctx.device)
    dts = fine_schedule(t1, stable_dt_kinetic(g, kp))
    out, mo = ctx.empty_f(), ctx.empty_moments()
    with ctx.fusion_levels(levels):
        code = _run_schedule(ctx, None, m0, dts, kp, out, want_f=True, mom_out=mo)
    torch.cuda.synchronize()
    return out.cpu().numpy(), mo.cpu().numpy(), code, len(dts)


def _unpack(m):
    return m[0], m[1:4].T, m[4]


@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: "x".join(map(str, (s[0],) + s[1])))
@pytest.mark.parametrize("bc", BCS)
@pytest.mark.parametrize("levels", [2, 3, 4])
def test_window_matches_oracle(shape, bc, levels):
    nx, nv, vm = shape
    g, mesh = _grids(nx, nv, vm)
    U = random_moments(nx, np.random.default_rng(nx + len(bc)))
    t1 = 6.5 * O.fine_cap(mesh, 0.5, None)  # 7 steps, the last one partial
    f, m, code, S = _window(g, bc, U, t1, levels)
    assert code == -1 and S == 7
    want_f = O.fine_propagate(O.lift(*U, mesh), 0.0, t1, mesh, 1e-2, bc)
    assert rel_inf(f, want_f) <= 1e-12
    assert moment_gap(_unpack(m), O.project(want_f, mesh)) <= 1e-12


@pytest.mark.parametrize("shape", SHAPES[:6], ids=lambda s: "x".join(map(str, (s[0],) + s[1])))
@pytest.mark.parametrize("bc", BCS)
def test_levels_agree_with_one_step_path(shape, bc):
    nx, nv, vm = shape
    g, mesh = _grids(nx, nv, vm)
    U = random_moments(nx, np.random.default_rng(7 * nx))
    t1 = 9.3 * O.fine_cap(mesh, 0.5, None)  # 10 steps: ragged passes for L = 3
    f0, m0, c0, _ = _window(g, bc, U, t1, 0)
    for L in (1, 2, 3, 4):
        f, m, c, _ = _window(g, bc, U, t1, L)
        assert c == c0 == -1
        assert rel_inf(f, f0) <= 1e-13
        assert moment_gap(_unpack(m), _unpack(m0)) <= 1e-13


@pytest.mark.parametrize("bc", BCS)
@pytest.mark.parametrize("levels", [1, 2, 3, 4])
def test_trapezoid_matches_oracle(bc, levels):
    g, mesh = _grids(9, (16, 16, 16), 8.0, quad="trapezoid")
    U = random_moments(9, np.random.default_rng(3))
    t1 = 4.5 * O.fine_cap(mesh, 0.5, None)
    f, m, code, _ = _window(g, bc, U, t1, levels)
    assert code == -1
    want_f = O.fine_propagate(O.lift(*U, mesh), 0.0, t1, mesh, 1e-2, bc)
    assert rel_inf(f, want_f) <= 1e-12
    assert moment_gap(_unpack(m), O.project(want_f, mesh)) <= 1e-12


@pytest.mark.parametrize("levels", [2, 3])
def test_even_data_keeps_exact_zero_velocity(levels):
    # x-homogeneous, velocity-even data: transport cancels exactly and every
    # marginal stays mirror-symmetric, so u is exactly 0 (ref/moments.py:80-88)
    nx = 6
    g, _ = _grids(nx, (32, 32, 32), 8.0)
    U = (np.full(nx, 1.3), np.zeros((nx, 3)), np.full(nx, 0.9))
    t1 = 5.0 * stable_dt_kinetic(g, P.KineticParams(1e-2))
    _, m, code, _ = _window(g, "periodic", U, t1, levels)
    assert code == -1
    assert np.all(m[1:4] == 0.0)


@pytest.mark.parametrize("levels", [1, 2, 3, 4])
def test_failure_keys_equal_one_step_path(levels):
    # a NaN density passes the reference's rho <= 0 test and surfaces as
    # BlowUpError; a negative one as DegenerateStateError -- same step and
    # kind on both paths
    g, _ = _grids(8, (16, 16, 16), 8.0)
    t1 = 4.5 * stable_dt_kinetic(g, P.KineticParams(1e-2))
    for bad in (np.nan, -0.5):
        rho, u, th = random_moments(8, np.random.default_rng(5))
        rho[3] = bad
        _, _, c0, _ = _window(g, "outflow", (rho, u, th), t1, 0)
        _, _, c, _ = _window(g, "outflow", (rho, u, th), t1, levels)
        assert c0 != -1
        assert c == c0


def test_parareal_equals_one_step_path():
    # BASELINE config 0 parareal (outflow) on both paths: same iteration
    # count, snapshots within 1e-12 (the oracle parity of this run is in
    # test_gpu_configs.py, on the default multi-step path)
    from dataclasses import replace
    from paper_2502_02704_b200.configs import config
    w = replace(config(0), outflow=True)
    g = P.PhaseGrid(P.build_spatial_grid(w.x_min, w.x_max, w.nx), P.build_velocity_grid(w.v_max, w.nv))
    bc = P.BoundaryKind(w.bc)
    d = P.Discretization(g, P.build_time_grids(w.t_final, w.n_g, w.n_f), bc)
    U0 = P.project(P.lift(P.MomentField(*w.raw_moments()), g, bc=bc), g, bc=bc)
    cfg = P.PararealConfig(w.k_max, w.tol)
    runs = []
    for L in (0, 2, 3, 4):
        with rt.ctx_for(g, bc).fusion_levels(L):
            runs.append(P.run_parareal(U0, cfg, d, P.KineticParams(w.eps), P.FluidParams()))
    (t0, r0), *rest = runs
    for t, r in rest:
        assert len(r) == len(r0)
        for a, b in zip(t.snapshots, t0.snapshots):
            assert moment_gap((a.rho, a.u, a.theta), (b.rho, b.u, b.theta)) <= 1e-12


def _from_f0(g, bc, f0, t1, levels):
    """F over [0, t1] of a given f0 (propagate_kinetic's path) on `levels` steps per pass."""
    kp = P.KineticParams(1e-2)
    ctx = rt.ctx_for(g, P.BoundaryKind(bc))
    fd = torch.from_numpy(np.ascontiguousarray(f0)).to(ctx.device)
    dts = fine_schedule(t1, stable_dt_kinetic(g, kp))
    out = ctx.empty_f()
    with ctx.fusion_levels(levels):
        code = _run_schedule(ctx, fd, None, dts, kp, out)
    torch.cuda.synchronize()
    return out.cpu().numpy(), code


@pytest.mark.parametrize("shape", SHAPES[:6], ids=lambda s: "x".join(map(str, (s[0],) + s[1])))
@pytest.mark.parametrize("bc", BCS)
def test_given_f0_matches_oracle_and_one_step(shape, bc):
    # propagate_kinetic from a non-Maxwellian f0: the recursion starts from the
    # weighted sums of f0 itself (identity tables for step 0)
    nx, nv, vm = shape
    g, mesh = _grids(nx, nv, vm)
    rng = np.random.default_rng(11 * nx)
    f0 = O.lift(*random_moments(nx, rng), mesh) * rng.uniform(0.8, 1.2, (nx,) + nv)
    t1 = 6.5 * O.fine_cap(mesh, 0.5, None)
    want = O.fine_propagate(f0, 0.0, t1, mesh, 1e-2, bc)
    one, c0 = _from_f0(g, bc, f0, t1, 0)
    for L in (2, 3):
        got, c = _from_f0(g, bc, f0, t1, L)
        assert c == c0 == -1
        assert rel_inf(got, want) <= 1e-12
        assert rel_inf(got, one) <= 1e-13


@pytest.mark.parametrize("levels", [2, 3])
def test_given_f0_non_finite_reports_step_one(levels):
    g, mesh = _grids(8, (16, 16, 16), 8.0)
    f0 = O.lift(*random_moments(8, np.random.default_rng(2)), mesh)
    f0[2, 3, 4, 5] = np.nan
    t1 = 3.5 * O.fine_cap(mesh, 0.5, None)
    _, c0 = _from_f0(g, "periodic", f0, t1, 0)
    _, c = _from_f0(g, "periodic", f0, t1, levels)
    assert c0 != -1 and c == c0
    with pytest.raises(P.BlowUpError) as info:
        rt.raise_kinetic(c)
    assert info.value.step == 1


@pytest.mark.parametrize("levels", [2, 3])
@pytest.mark.parametrize("bc", ["outflow", "periodic"])
def test_batched_windows_equal_one_step_path(levels, bc):
    # pbgk_propagate_windows runs the recursion of all windows batched (one
    # launch per step, windows of different lengths, an empty one, a failing
    # one) -- per-window moments and keys as on the one-step path (window
    # groups smaller than the batch: test_gpu_msweep.py)
    from paper_2502_02704_b200.kinetic import propagate_windows
    g, mesh = _grids(10, (16, 16, 16), 8.0)
    kp = P.KineticParams(1e-2)
    ctx = rt.ctx_for(g, P.BoundaryKind(bc))
    cap = stable_dt_kinetic(g, kp)
    spans = [7.5 * cap, 4.0 * cap, 0.0, 9.2 * cap, 2.5 * cap]
    rng = np.random.default_rng(9)
    Us = [random_moments(10, rng) for _ in spans]
    Us[3][0][4] = np.nan  # window 3 fails (BlowUpError at some step)
    mom_in = torch.stack([rt.to_device_moments(P.MomentField(*U), ctx.device) for U in Us])
    res = {}
    for L in (0, levels):
        out = ctx.empty_moments(len(spans))
        with ctx.fusion_levels(L):
            codes = propagate_windows(ctx, mom_in, spans, g, kp, None, out)
        res[L] = (out.cpu().numpy(), codes)
    (m0, c0), (m1, c1) = res[0], res[levels]
    assert c1 == c0 and c0[3] != -1 and c0[2] == -1
    for w in (0, 1, 2, 4):
        assert moment_gap(_unpack(m1[w]), _unpack(m0[w])) <= 1e-13


@pytest.mark.parametrize("bc", BCS)
@pytest.mark.parametrize("levels", [2, 4])
def test_long_propagation_concurrent_recursion(bc, levels):
    # >= 8 L steps on a small grid: the recursion runs on a side stream on
    # reserved SMs while the passes wait on its device progress word
    g, mesh = _grids(24, (32, 32, 32), 8.0)
    rng = np.random.default_rng(17)
    f0 = O.lift(*random_moments(24, rng), mesh) * rng.uniform(0.9, 1.1, (24, 32, 32, 32))
    t1 = 59.5 * O.fine_cap(mesh, 0.5, None)  # 60 steps
    one, c0 = _from_f0(g, bc, f0, t1, 0)
    got, c = _from_f0(g, bc, f0, t1, levels)
    assert c == c0 == -1
    assert rel_inf(got, one) <= 1e-12
    U = random_moments(24, rng)
    _, m0, k0, _ = _window(g, bc, U, t1, 0)
    _, m1, k1, S = _window(g, bc, U, t1, levels)
    assert S == 60 and k0 == k1 == -1
    assert moment_gap(_unpack(m1), _unpack(m0)) <= 1e-12


def _window_field(g, bc, U, t1, levels, E):
    kp = P.KineticParams(1e-2, force=E)
    return _window(g, bc, U, t1, levels, kp=kp)


@pytest.mark.parametrize("shape", [(9, (32, 32, 32), 8.0), (7, (48, 48, 48), 10.0), (5, (64, 64, 64), 8.0),
                                   (10, (16, 8, 8), 6.0)],
                         ids=lambda s: "x".join(map(str, (s[0],) + s[1])))
@pytest.mark.parametrize("bc", BCS)
def test_field_window_matches_oracle_and_one_step(shape, bc):
    # the v_x field term: the recursion carries it, the passes are one-step
    # sweeps on its tables without the marginal partials
    nx, nv, vm = shape
    g, mesh = _grids(nx, nv, vm)
    E = 0.5 * np.sin(2 * np.pi * mesh.xc)
    U = random_moments(nx, np.random.default_rng(nx + 5))
    t1 = 6.5 * O.fine_cap(mesh, 0.5, E)
    f, m, code, S = _window_field(g, bc, U, t1, -1, E)
    f0, m0, c0, _ = _window_field(g, bc, U, t1, 0, E)
    assert code == c0 == -1 and S == 7
    want_f = O.fine_propagate(O.lift(*U, mesh), 0.0, t1, mesh, 1e-2, bc, E)
    assert rel_inf(f, want_f) <= 1e-12
    assert moment_gap(_unpack(m), O.project(want_f, mesh)) <= 1e-12
    assert rel_inf(f, f0) <= 1e-13
    assert moment_gap(_unpack(m), _unpack(m0)) <= 1e-13


def test_field_batched_windows_and_nan_key():
    from paper_2502_02704_b200.kinetic import propagate_windows
    g, mesh = _grids(12, (32, 32, 32), 8.0)
    E = 0.5 * np.sin(2 * np.pi * mesh.xc)
    kp = P.KineticParams(1e-2, force=E)
    ctx = rt.ctx_for(g, P.BoundaryKind.PERIODIC)
    cap = stable_dt_kinetic(g, kp)
    spans = [5.5 * cap, 3.0 * cap, 7.2 * cap]
    rng = np.random.default_rng(21)
    Us = [random_moments(12, rng) for _ in spans]
    Us[1][0][7] = np.nan
    mom_in = torch.stack([rt.to_device_moments(P.MomentField(*U), ctx.device) for U in Us])
    res = {}
    for L in (0, -1):
        out = ctx.empty_moments(len(spans))
        with ctx.fusion_levels(L):
            codes = propagate_windows(ctx, mom_in, spans, g, kp, None, out)
        res[L] = (out.cpu().numpy(), codes)
    (m0, c0), (m1, c1) = res[0], res[-1]
    assert c1 == c0 and c0[1] != -1
    for w in (0, 2):
        assert moment_gap(_unpack(m1[w]), _unpack(m0[w])) <= 1e-13
