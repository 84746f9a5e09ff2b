"""x-sharded fine propagator: slabs of x cells on
ranks with per-step halo exchange must give BITWISE the single-GPU F of the
one-step path (the slabs' path; the multi-step path agrees with it to 1e-13,
tests/test_gpu_fused.py).

Multi-rank cases run 2-3 processes on cuda:0 over gloo: the halo exchange is
host-staged and synchronous between steps, so no kernel waits on another
process's kernel (B200_PROFILING.md); what is exercised is the product path
of an NCCL launch (slab contexts, padded buffers, exchange order, global
boundary halos, error agreement)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu
P = pytest.importorskip("paper_2502_02704_b200")


def _setup(nx=13, nv=(16, 8, 8), field=False, bc="periodic"):
    g = P.PhaseGrid(P.build_spatial_grid(0.0, 1.0, nx), P.build_velocity_grid(6.0, nv))
    x = g.space.centers
    E = 0.4 * np.sin(2 * np.pi * x) if field else None
    kp = P.KineticParams(1e-2, force=E)
    rng = np.random.default_rng(nx)
    U = P.MomentField(rng.uniform(0.5, 1.5, nx), rng.uniform(-0.3, 0.3, (nx, 3)),
                      rng.uniform(0.6, 1.4, nx))
    f0 = P.lift(U, g).values * rng.uniform(0.8, 1.2, (nx,) + nv)
    return g, kp, U, f0, P.BoundaryKind(bc)


def _reference(g, kp, U, f0, bc, t1):
    from paper_2502_02704_b200 import runtime as rt
    from paper_2502_02704_b200.kinetic import propagate_window
    ctx = rt.ctx_for(g, bc)
    mo = ctx.empty_moments()
    with ctx.fusion_levels(0):  # slabs run the one-step path; compare like with like
        f = P.propagate_kinetic(P.Distribution(f0), 0.0, t1, g, kp, bc).values
        code = propagate_window(ctx, rt.to_device_moments(U, ctx.device), 0.0, t1, g, kp, None, mo)
    assert code == -1
    return np.asarray(f), mo.cpu().numpy()


def _slab_run(g, kp, U, f0, bc, t1):
    from paper_2502_02704_b200 import runtime as rt
    from paper_2502_02704_b200.sharded import SlabFine
    sl = SlabFine(g, bc, kp, torch.device("cuda", 0))
    a, b = sl.x0, sl.x0 + sl.n
    fl, _ = sl.propagate(0.0, t1, f0=torch.from_numpy(np.ascontiguousarray(f0[a:b])).cuda())
    _, ml = sl.propagate(0.0, t1, mom0=rt.to_device_moments(U, torch.device("cuda", 0))[:, a:b],
                         want_f=False, want_moments=True)
    return sl.gather(fl, 0).cpu().numpy(), sl.gather(ml, 1).cpu().numpy()


@pytest.mark.parametrize("bc", ["periodic", "absorbing", "outflow"])
@pytest.mark.parametrize("field", [False, True])
def test_single_slab_equals_unsharded(bc, field):
    g, kp, U, f0, bck = _setup(field=field, bc=bc)
    t1 = 4.5 * P.stable_dt_kinetic(g, kp)
    want_f, want_m = _reference(g, kp, U, f0, bck, t1)
    got_f, got_m = _slab_run(g, kp, U, f0, bck, t1)
    assert np.array_equal(got_f, want_f)
    assert np.array_equal(got_m, want_m)


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, bc, field, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g, kp, U, f0, bck = _setup(field=field, bc=bc)
        t1 = 4.5 * P.stable_dt_kinetic(g, kp)
        q.put((rank, _slab_run(g, kp, U, f0, bck, t1)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("bc,field", [("periodic", True), ("absorbing", False), ("outflow", True)])
def test_multi_rank_slabs_bitwise(world, bc, field):
    g, kp, U, f0, bck = _setup(field=field, bc=bc)
    t1 = 4.5 * P.stable_dt_kinetic(g, kp)
    want_f, want_m = _reference(g, kp, U, f0, bck, t1)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, bc, field, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(world):
        got_f, got_m = res[r]
        assert np.array_equal(got_f, want_f)
        assert np.array_equal(got_m, want_m)


CFG = """case = sod
x_min = 0.0
x_max = 1.0
n_x = 23
v_max = 8.0
n_vx = 16
n_vy = 8
n_vz = 8
epsilon = 1e-2
bc = outflow
t_final = 0.02
n_g = 3
n_f = 6
k_max = 1
tol = 1e-8
mode = fine
"""


def _fine_worker(rank, world, port, path, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2502_02704_b200.runner import prepare, run_fine_mode
        cfg = P.parse_config(path)
        disc, kin, _, _ = prepare(cfg)
        snaps = run_fine_mode(cfg, disc, kin)
        q.put((rank, [np.stack([s.rho, s.theta]) for s in snaps]))
    finally:
        dist.destroy_process_group()


def test_run_fine_mode_x_sharded_bitwise(tmp_path):
    from paper_2502_02704_b200.runner import prepare, run_fine_mode
    path = tmp_path / "f.cfg"
    path.write_text(CFG)
    cfg = P.parse_config(path)
    disc, kin, _, _ = prepare(cfg)
    from paper_2502_02704_b200 import runtime as rt
    with rt.ctx_for(disc.phase, disc.bc).fusion_levels(0):  # the slab path is one-step
        want = [np.stack([s.rho, s.theta]) for s in run_fine_mode(cfg, disc, kin)]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_fine_worker, args=(r, 2, port, str(path), q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(2):
        assert len(res[r]) == len(want)
        for a, b in zip(res[r], want):
            assert np.array_equal(a, b)
