"""Multi-rank parareal (windows sharded with work_distribution, one jump
all-gather per iteration) on CPU ranks over gloo.

The numerical backend is the oracle (tests/oracle_backend.py); what is under
test is the product's ShardedRun: partition, exchange, assembly, error
agreement, and bitwise independence of the rank count.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import bgk as O


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _problem():
    mesh = O.Mesh(0.0, 1.0, 10, 6.0, (6, 6, 6))
    return O.Problem(mesh, 0.04, 5, 10, 1e-2, False)


def _disc(P):
    g = P.PhaseGrid(P.build_spatial_grid(0.0, 1.0, 10), P.build_velocity_grid(6.0, 6))
    return P.Discretization(g, P.build_time_grids(0.04, 5, 10), P.BoundaryKind.ABSORBING)


def _worker(rank, world, port, frozen, fail_window, q, pipelined=False):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2502_02704_b200 as P
        from oracle_backend import OracleBackend
        prob = _problem()
        U0 = O.two_state(prob.mesh, 0.5, (1.0, 0.0, 1.0), (0.125, 0.0, 0.8))
        be = OracleBackend(prob, fail_window)
        try:
            traj, rec = P.run_parareal(P.MomentField(*U0),
                                       P.PararealConfig(3, 1e-300, frozen, pipelined=pipelined),
                                       _disc(P), P.KineticParams(1e-2), P.FluidParams(),
                                       backend=be)
            out = ("ok", [np.stack([s.rho, s.theta]) for s in traj.snapshots],
                   [np.stack([s.u]) for s in traj.snapshots], [r.error for r in rec],
                   sorted(be.windows_done))
        except P.SolverError as e:
            out = ("err", type(e).__name__, getattr(e, "step", None),
                   getattr(e, "slice_index", None), None)
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def _run(world, frozen=True, fail_window=None, pipelined=False):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, frozen, fail_window, q, pipelined))
             for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=180) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


def _serial(frozen=True):
    prob = _problem()
    U0 = O.two_state(prob.mesh, 0.5, (1.0, 0.0, 1.0), (0.125, 0.0, 0.8))
    return O.parareal(prob, U0, 3, 1e-300, frozen)


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("frozen", [True, False])
@pytest.mark.parametrize("pipelined", [False, True])
def test_sharded_parareal_bitwise_equals_serial(world, frozen, pipelined):
    snaps, errs = _serial(frozen)
    res = _run(world, frozen, pipelined=pipelined)
    first = None
    all_windows = []
    for rank in range(world):
        status, rt_, u, e, done = res[rank]
        assert status == "ok"
        assert e == errs  # identical iteration count and errors
        for n, s in enumerate(snaps):
            assert np.array_equal(rt_[n][0], s[0]) and np.array_equal(rt_[n][1], s[2])
            assert np.array_equal(u[n][0], s[1])
        if first is None:
            first = rt_
        all_windows += done
    # each window of each iteration computed exactly once across ranks
    n_g = 5
    expect = sorted(sum((list(range(k if frozen else 1, n_g + 1)) for k in (1, 2, 3)), []))
    assert sorted(all_windows) == expect


@pytest.mark.parametrize("pipelined", [False, True])
def test_sharded_failure_raises_same_error_on_every_rank(pipelined):
    res = _run(2, fail_window=4, pipelined=pipelined)
    for rank in range(2):
        status, name, step, sl, _ = res[rank]
        assert status == "err" and name == "BlowUpError" and step == 2


@pytest.mark.parametrize("frozen", [True, False])
def test_pipelined_single_process_bitwise_equals_serial(frozen):
    import paper_2502_02704_b200 as P
    from oracle_backend import OracleBackend
    snaps, errs = _serial(frozen)
    prob = _problem()
    U0 = O.two_state(prob.mesh, 0.5, (1.0, 0.0, 1.0), (0.125, 0.0, 0.8))
    be = OracleBackend(prob)
    traj, rec = P.run_parareal(P.MomentField(*U0), P.PararealConfig(3, 1e-300, frozen, pipelined=True),
                               _disc(P), P.KineticParams(1e-2), P.FluidParams(), backend=be)
    assert [r.error for r in rec] == errs
    for a, s in zip(traj.snapshots, snaps):
        assert np.array_equal(a.rho, s[0]) and np.array_equal(a.u, s[1]) and np.array_equal(a.theta, s[2])
