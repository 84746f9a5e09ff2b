"""Multi-rank parareal with the REAL GPU backend, two ranks sharing cuda:0.

The collectives go through gloo (host side), so no kernel waits on another
process's kernel (B200_PROFILING.md); what is exercised is the product path
of a torchrun launch -- ShardedRun over GpuBackend, the jump all-gather and
the replicated correction -- and the claim that the trajectory is bitwise
independent of the rank count.
"""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _problem(P):
    g = P.PhaseGrid(P.build_spatial_grid(0.0, 1.0, 32), P.build_velocity_grid(8.0, 16))
    d = P.Discretization(g, P.build_time_grids(0.05, 6, 24), P.BoundaryKind.OUTFLOW)
    x = g.space.centers
    U0 = P.MomentField(np.where(x < 0.5, 1.0, 0.125), np.zeros((32, 3)), np.where(x < 0.5, 1.0, 0.8))
    return d, U0


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2502_02704_b200 as P
        d, U0 = _problem(P)
        traj, rec = P.run_parareal(U0, P.PararealConfig(4, 1e-300), d, P.KineticParams(1e-2),
                                   P.FluidParams())
        q.put((rank, [np.stack([s.rho, s.theta]) for s in traj.snapshots],
               [r.error for r in rec]))
    finally:
        dist.destroy_process_group()


def test_two_ranks_on_one_gpu_bitwise_equal_single_process():
    import paper_2502_02704_b200 as P
    d, U0 = _problem(P)
    traj, rec = P.run_parareal(U0, P.PararealConfig(4, 1e-300), d, P.KineticParams(1e-2),
                               P.FluidParams())
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict((r, (s, e)) for r, s, e in (q.get(timeout=300) for _ in range(2)))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(2):
        snaps, errs = res[r]
        assert errs == [x.error for x in rec]
        for a, b in zip(snaps, traj.snapshots):
            assert np.array_equal(a[0], b.rho) and np.array_equal(a[1], b.theta)
