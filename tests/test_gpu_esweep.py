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
