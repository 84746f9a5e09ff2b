"""Multi-step passes WITH the v_x field term (csrc/esweep.cu, include/pbgk.h
pbgk_set_esweep): a warp per (whole v_x column, x segment), up to 4 fine
steps per pass.

Parity: the oracle's F with a force (ref/kinetic.py:114-123,137-161) to 1e-12
on f_S and on the moments, and the one-step path to 1e-12, for every
boundary, 1..4 levels (ragged last passes), windows from moments (the first
pass synthesises the lift) and from a given f0, segment lengths down to one
plane (many warps per column: every halo / ghost branch), and the status keys
of a non-finite start equal to the one-step path's."""

import numpy as np
import pytest
import torch

from oracle import bgk as O
from helpers import moment_gap, random_moments, rel_inf

pytestmark = pytest.mark.gpu
P = pytest.importorskip("paper_2502_02704_b200")
from paper_2502_02704_b200 import runtime as rt  # noqa: E402
from paper_2502_02704_b200.kinetic import _run_schedule, fine_schedule, stable_dt_kinetic  # noqa: E402

BCS = ["periodic", "absorbing", "outflow"]
# nvx = 16 / 32 / 48 (V = 2 / 4 / 6 rows per lane); nx from one segment per
# column to many
SHAPES = [
    (9, (32, 32, 32), 8.0),
    (10, (16, 8, 8), 6.0),
    (7, (48, 48, 16), 10.0),
    (40, (16, 16, 16), 8.0),
    (3, (32, 8, 8), 8.0),
]


def _grids(nx, nv, vm):
    g = P.PhaseGrid(P.build_spatial_grid(0.0, 1.0, nx), P.build_velocity_grid(vm, nv))
    return g, O.Mesh(0.0, 1.0, nx, vm, nv)


def _field(mesh):
    return 0.5 * np.sin(2 * np.pi * mesh.xc) + 0.2


def _run(g, bc, E, t1, levels, U=None, f0=None, es=True):
    kp = P.KineticParams(1e-2, force=E)
    ctx = rt.ctx_for(g, P.BoundaryKind(bc))
    m0 = rt.to_device_moments(P.MomentField(*U), ctx.device) if U is not None else None
    fd = torch.from_numpy(np.ascontiguousarray(f0)).to(ctx.device) if f0 is not None else None
    dts = fine_schedule(t1, stable_dt_kinetic(g, kp))
    out, mo = ctx.empty_f(), ctx.empty_moments()
    with ctx.fusion_levels(levels), ctx.esweep_mode(es):
        code = _run_schedule(ctx, fd, m0, dts, kp, out, want_f=True, mom_out=mo)
    torch.cuda.synchronize()
    return out.cpu().numpy(), mo.cpu().numpy(), code, len(dts)


def _unpack(m):
    return m[0], m[1:4].T, m[4]


def test_levels_reported():
    g, _ = _grids(9, (32, 32, 32), 8.0)
    ctx = rt.ctx_for(g, P.BoundaryKind.PERIODIC)
    with ctx.fusion_levels(-1):
        assert ctx.esweep_levels() == 3
        with ctx.esweep_mode(False):
            assert ctx.esweep_levels() == 0
    with ctx.fusion_levels(2):
        assert ctx.esweep_levels() == 2
    g64, _ = _grids(5, (64, 8, 8), 8.0)
    assert rt.ctx_for(g64, P.BoundaryKind.PERIODIC).esweep_levels() == 0


@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: "x".join(map(str, (s[0],) + s[1])))
@pytest.mark.parametrize("bc", BCS)
@pytest.mark.parametrize("levels", [1, 2, 3, 4])
def test_window_from_moments_matches_oracle(shape, bc, levels):
    nx, nv, vm = shape
    g, mesh = _grids(nx, nv, vm)
    E = _field(mesh)
    U = random_moments(nx, np.random.default_rng(7 * nx + levels))
    t1 = 7.5 * O.fine_cap(mesh, 0.5, E)
    f, m, code, S = _run(g, bc, E, t1, levels, U=U)
    f0, m0, c0, _ = _run(g, bc, E, t1, 0, U=U)
    assert code == c0 == -1 and S == 8
    want_f = O.fine_propagate(O.lift(*U, mesh), 0.0, t1, mesh, 1e-2, bc, E)
    assert rel_inf(f, want_f) <= 1e-12
    assert moment_gap(_unpack(m), O.project(want_f, mesh)) <= 1e-12
    assert rel_inf(f, f0) <= 1e-12
    assert moment_gap(_unpack(m), _unpack(m0)) <= 1e-12


@pytest.mark.parametrize("shape", SHAPES[:3], ids=lambda s: "x".join(map(str, (s[0],) + s[1])))
@pytest.mark.parametrize("bc", BCS)
def test_given_f0_matches_oracle(shape, bc):
    nx, nv, vm = shape
    g, mesh = _grids(nx, nv, vm)
    E = _field(mesh)
    rng = np.random.default_rng(3 * nx)
    f0 = O.lift(*random_moments(nx, rng), mesh) * rng.uniform(0.8, 1.2, (nx,) + nv)
    t1 = 6.5 * O.fine_cap(mesh, 0.5, E)
    want = O.fine_propagate(f0, 0.0, t1, mesh, 1e-2, bc, E)
    for L in (-1, 2):
        got, _, c, _ = _run(g, bc, E, t1, L, f0=f0)
        assert c == -1
        assert rel_inf(got, want) <= 1e-12


def test_esweep_equals_one_step_field_passes():
    # the same multi-step tables, the field passes one step each vs several
    g, mesh = _grids(24, (32, 16, 16), 8.0)
    E = _field(mesh)
    U = random_moments(24, np.random.default_rng(5))
    t1 = 13.3 * O.fine_cap(mesh, 0.5, E)
    for bc in BCS:
        a = _run(g, bc, E, t1, -1, U=U, es=True)
        b = _run(g, bc, E, t1, -1, U=U, es=False)
        assert a[2] == b[2] == -1 and a[3] == 14
        assert rel_inf(a[0], b[0]) <= 1e-12
        assert moment_gap(_unpack(a[1]), _unpack(b[1])) <= 1e-12


def test_high_field_and_long_x():
    # |E| near the CFL split's limit, many segments per column on a long x grid
    g, mesh = _grids(300, (16, 8, 8), 6.0)
    E = 3.0 * np.cos(2 * np.pi * mesh.xc)
    U = random_moments(300, np.random.default_rng(9))
    t1 = 9.0 * O.fine_cap(mesh, 0.5, E)
    for bc in ("periodic", "outflow"):
        f, m, code, S = _run(g, bc, E, t1, -1, U=U)
        want = O.fine_propagate(O.lift(*U, mesh), 0.0, t1, mesh, 1e-2, bc, E)
        assert code == -1 and S >= 9
        assert rel_inf(f, want) <= 1e-12


@pytest.mark.parametrize("levels", [-1, 2])
def test_non_finite_start_key_equals_one_step_path(levels):
    g, mesh = _grids(10, (32, 8, 8), 8.0)
    E = _field(mesh)
    f0 = O.lift(*random_moments(10, np.random.default_rng(4)), mesh)
    f0[6, 20, 3, 5] = np.inf
    t1 = 5.5 * O.fine_cap(mesh, 0.5, E)
    _, _, c0, _ = _run(g, "periodic", E, t1, 0, f0=f0)
    _, _, c, _ = _run(g, "periodic", E, t1, levels, f0=f0)
    assert c0 != -1 and c == c0
    with pytest.raises(P.BlowUpError) as info:
        rt.raise_kinetic(c)
    assert info.value.step == 1


def _window_moments(g, bc, E, t1, levels, U):
    """P(f_S) of one window from moments, no f_S wanted: the last field pass
    projects (FINAL) unless PBGK_ES_NOFINAL is set."""
    kp = P.KineticParams(1e-2, force=E)
    ctx = rt.ctx_for(g, P.BoundaryKind(bc))
    m0 = rt.to_device_moments(P.MomentField(*U), ctx.device)
    dts = fine_schedule(t1, stable_dt_kinetic(g, kp))
    out, mo = ctx.empty_f(), ctx.empty_moments()
    with ctx.fusion_levels(levels), ctx.esweep_mode(True):
        code = _run_schedule(ctx, None, m0, dts, kp, out, want_f=False, mom_out=mo)
    torch.cuda.synchronize()
    return mo.cpu().numpy(), code, len(dts)


@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: "x".join(map(str, (s[0],) + s[1])))
@pytest.mark.parametrize("bc", BCS)
@pytest.mark.parametrize("levels", [1, 2, 3, 4])
def test_final_pass_projects_like_the_oracle(shape, bc, levels, monkeypatch):
    # the window's last field pass applies R_S and writes the partial records
    # of P(f_S) (ref/kinetic.py:130-134, ref/moments.py:60-112) instead of f_S;
    # 5.5 / 8 steps: ragged and full last passes, a single SYNTH + FINAL pass
    nx, nv, vm = shape
    g, mesh = _grids(nx, nv, vm)
    E = _field(mesh)
    U = random_moments(nx, np.random.default_rng(11 * nx + levels))
    for steps in (2.5, 7.5):
        t1 = steps * O.fine_cap(mesh, 0.5, E)
        m, code, S = _window_moments(g, bc, E, t1, levels, U)
        monkeypatch.setenv("PBGK_ES_NOFINAL", "1")
        m1, c1, _ = _window_moments(g, bc, E, t1, levels, U)
        monkeypatch.delenv("PBGK_ES_NOFINAL")
        assert code == c1 == -1
        want = O.project(O.fine_propagate(O.lift(*U, mesh), 0.0, t1, mesh, 1e-2, bc, E), mesh)
        assert moment_gap(_unpack(m), want) <= 1e-12
        assert moment_gap(_unpack(m), _unpack(m1)) <= 1e-13


def test_final_pass_even_data_keeps_zero_transverse_velocity():
    # u_y = u_z = 0 data stays even in v_y, v_z under F with a v_x force: the
    # folded first moments (ref/moments.py:80-88) of the FINAL pass's records
    # are exactly zero (the same tree for an entry and its mirror)
    g, mesh = _grids(12, (32, 16, 16), 8.0)
    E = _field(mesh)
    rho, u, th = random_moments(12, np.random.default_rng(2))
    u[:, 1:] = 0.0
    for bc in BCS:
        m, code, _ = _window_moments(g, bc, E, 9.5 * O.fine_cap(mesh, 0.5, E), -1, (rho, u, th))
        assert code == -1
        assert np.all(m[2] == 0.0) and np.all(m[3] == 0.0)


def test_final_pass_windows_keys_and_groups(monkeypatch):
    # pbgk_propagate_windows with a force: windows of different lengths, an
    # empty and a failing one; FINAL passes vs the separate final sweep
    from paper_2502_02704_b200.kinetic import propagate_windows
    g, mesh = _grids(10, (32, 8, 8), 8.0)
    E = _field(mesh)
    kp = P.KineticParams(1e-2, force=E)
    ctx = rt.ctx_for(g, P.BoundaryKind.PERIODIC)
    cap = stable_dt_kinetic(g, kp)
    spans = [9.5 * cap, 3.0 * cap, 0.0, 6.2 * cap, 6.0 * cap]
    rng = np.random.default_rng(19)
    Us = [random_moments(10, rng) for _ in spans]
    Us[3][0][4] = np.nan
    mom_in = torch.stack([rt.to_device_moments(P.MomentField(*U), ctx.device) for U in Us])
    res = []
    for nofinal in (False, True):
        if nofinal:
            monkeypatch.setenv("PBGK_ES_NOFINAL", "1")
        out = ctx.empty_moments(len(spans))
        codes = propagate_windows(ctx, mom_in, spans, g, kp, None, out)
        res.append((out.cpu().numpy(), codes))
    monkeypatch.delenv("PBGK_ES_NOFINAL")
    (ma, ca), (mb, cb) = res
    assert ca == cb and ca[3] != -1 and ca[2] == -1
    for w in (0, 1, 2, 4):
        assert moment_gap(_unpack(ma[w]), _unpack(mb[w])) <= 1e-13
    want = O.project(O.fine_propagate(O.lift(*Us[0], mesh), 0.0, spans[0], mesh, 1e-2, "periodic", E), mesh)
    assert moment_gap(_unpack(ma[0]), want) <= 1e-12
