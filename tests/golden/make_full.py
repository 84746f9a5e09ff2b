"""Full-size BASELINE.json workloads on the CPU: fixtures for the GPU parity
tests at the sizes the bench reports (tests/test_gpu_full_size.py).

Run in the build container (hours of CPU; each job writes one file):

    PYTHONPATH=/root/reference/pkg/src:. python tests/golden/make_full.py JOB [workers]

Jobs and what computes them:

* ``cfg1``      -- the UNMODIFIED reference: ``propagate_kinetic`` over the whole
                   T = 0.2 horizon (820 steps, 256 x 32^3 periodic), 1 core.
* ``cfg3a``     -- the UNMODIFIED reference: ``run_parareal`` (K = 5, tol 1e-8,
                   ``workers`` fork pool, ref/parareal.py:161-170) on 1024 x 32^3
                   with the field; then window n_g's f after the run
                   (``propagate_kinetic(lift(snapshots[n_g - 1]))``).
* ``cfg2_e1``, ``cfg2_e0.1`` -- the oracle (outflow is an oracle extension;
                   the reference has only the absorbing ghost): the parareal loop
                   of ref/parareal.py:251-278 with each iteration's windows in a
                   process pool; per-iteration errors, and whether / in which
                   iteration and window ``CorrectionOvershootError`` fires.
* ``cfg4w1``    -- the oracle (outflow): one full 2048 x 64^3 window P F L and
                   G from U0 (32 fine steps), plus f slices of the result.
* ``abs_cfg2``  -- the UNMODIFIED reference, absorbing ghost, config 2 (eps 1)
                   full size, one iteration: the overshoot that made configs
                   2 / 4 move to the outflow extension.
* ``abs_cfg4x8`` -- the same on config 4's x grid with an 8^3 velocity grid.

Problem data come from ``paper_2502_02704_b200.configs`` (pure numpy).
"""

from __future__ import annotations

import multiprocessing as mp
import sys
import time
from dataclasses import replace
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, "/root/reference/pkg/src")

from oracle import bgk as O  # noqa: E402
from paper_2502_02704_b200.configs import config  # noqa: E402

OUT = Path(__file__).resolve().parent


def _ref():
    import parabgk as R
    return R


def ref_setup(w):
    R = _ref()
    g = R.PhaseGrid(R.build_spatial_grid(w.x_min, w.x_max, w.nx), R.build_velocity_grid(w.v_max, w.nv))
    bc = R.BoundaryKind.PERIODIC if w.periodic else R.BoundaryKind.ABSORBING
    assert w.bc in ("periodic", "absorbing")
    d = R.Discretization(g, R.build_time_grids(w.t_final, w.n_g, w.n_f), bc)
    E = w.force()
    return R, g, bc, d, R.KineticParams(w.eps, force=E), R.FluidParams(force=E)


def oracle_setup(w):
    m = O.Mesh(w.x_min, w.x_max, w.nx, w.v_max, w.nv)
    return m, O.Problem(m, w.t_final, w.n_g, w.n_f, w.eps, w.bc, w.force())


def marg(f):
    return [np.add.reduce(f, axis=(2, 3)), np.add.reduce(f, axis=(1, 3)), np.add.reduce(f, axis=(1, 2))]


def save(name, **d):
    np.savez_compressed(OUT / ("full_%s.npz" % name), **d)
    print("wrote full_%s.npz" % name, sum(np.asarray(v).nbytes for v in d.values()), "bytes", flush=True)


# ---------------------------------------------------------------------------

def job_cfg1(workers):
    w = config(1)
    R, g, bc, d, kin, flu = ref_setup(w)
    f0 = R.lift(R.MomentField(*w.raw_moments()), g)
    tic = time.time()
    f = R.propagate_kinetic(f0, 0.0, w.t_final, g, kin, bc).values
    sec = time.time() - tic
    U = R.project(R.Distribution(f), g)
    mx, my, mz = marg(f)
    save("cfg1", rho=U.rho, u=U.u, theta=U.theta, mx=mx, my=my, mz=mz,
         planes_i=np.array([64, 191]), planes=f[[64, 191]], seconds=sec)


def job_cfg3a(workers, perturb=0.0):
    w = config(3)
    R, g, bc, d, kin, flu = ref_setup(w)
    U0 = R.project(R.lift(R.MomentField(*w.raw_moments()), g), g)
    if perturb:
        # the reference's sensitivity to rounding-level differences in its
        # fine solves: every window jump gets a seeded absolute perturbation
        # of size `perturb` (what another correct fp64 implementation of F
        # differs by), the rest of the run unmodified
        import parabgk.parareal as RP
        orig = RP._window_jump

        def jump(n, U, *args, **kw):
            n_, delta, st = orig(n, U, *args, **kw)
            seed = int(np.frombuffer(np.float64(U.rho[0] + 7 * U.theta[-1]).tobytes(), np.uint64)[0] % 2**32)
            rng = np.random.default_rng([n, seed])
            delta = R.MomentField(delta.rho + perturb * rng.uniform(-1, 1, delta.rho.shape),
                                  delta.u + perturb * rng.uniform(-1, 1, delta.u.shape),
                                  delta.theta + perturb * rng.uniform(-1, 1, delta.theta.shape))
            return n_, delta, st
        RP._window_jump = jump
    tic = time.time()
    traj, rec = R.run_parareal(U0, R.PararealConfig(w.k_max, w.tol, workers=workers), d, kin, flu)
    sec = time.time() - tic
    S = traj.snapshots
    if perturb:
        save("cfg3a_pert", perturb=perturb, snap_rho=np.stack([s.rho for s in S]),
             snap_u=np.stack([s.u for s in S]), snap_theta=np.stack([s.theta for s in S]),
             errors=np.array([r.error for r in rec]), k=np.array([r.k for r in rec]), seconds=sec)
        return
    t = d.time.coarse_times
    f = R.lift(S[w.n_g - 1], g)
    f = R.propagate_kinetic(f, float(t[w.n_g - 1]), float(t[w.n_g]), g, kin, bc,
                            dt_max=d.time.dt_f).values
    Uf = R.project(R.Distribution(f), g)
    mx, my, mz = marg(f)
    save("cfg3a", rho0=U0.rho, u0=U0.u, theta0=U0.theta,
         snap_rho=np.stack([s.rho for s in S]), snap_u=np.stack([s.u for s in S]),
         snap_theta=np.stack([s.theta for s in S]),
         errors=np.array([r.error for r in rec]), k=np.array([r.k for r in rec]),
         f_rho=Uf.rho, f_u=Uf.u, f_theta=Uf.theta, f_mx=mx, f_my=my, f_mz=mz,
         planes_i=np.array([256, 700]), planes=f[[256, 700]], seconds=sec, workers=workers)


_PROB = None


def _init(prob):
    global _PROB
    _PROB = prob


def _jump(args):
    n, U = args
    return n, O.window_jump(_PROB, U, n)


def job_cfg2(eps, workers):
    w = config(2, eps)
    m, prob = oracle_setup(w)
    U0 = O.project(O.lift(*w.raw_moments(), m), m)
    snaps = [tuple(np.array(x, copy=True) for x in U0)]
    for n in range(1, w.n_g + 1):
        snaps.append(O.G(prob, snaps[-1], n))
    errors, overshoot = [], (0, 0)
    done_snaps = snaps
    tic = time.time()
    with mp.get_context("fork").Pool(workers, initializer=_init, initargs=(prob,)) as pool:
        for k in range(1, w.k_max + 1):
            jumps = dict(pool.imap_unordered(_jump, [(n, snaps[n - 1]) for n in range(k, w.n_g + 1)]))
            new = list(snaps)
            err = 0.0
            for n in range(k, w.n_g + 1):  # ref/parareal.py:217-248
                cor = O._add(O.G(prob, new[n - 1], n), jumps[n])
                ok = all(np.all(np.isfinite(x)) for x in cor)
                if not ok or np.any(cor[0] <= 0.0) or np.any(cor[2] <= 0.0):
                    overshoot = (k, n)
                    break
                err = max(err, O.sup_gap(cor, snaps[n]))
                new[n] = cor
            if overshoot[0]:
                break
            snaps = new
            done_snaps = snaps
            errors.append(err)
            print("cfg2 eps %g iteration %d error %.17g (%.0f s)" % (eps, k, err, time.time() - tic),
                  flush=True)
            if err < w.tol:
                break
    save("cfg2_e%g" % eps, rho0=U0[0], u0=U0[1], theta0=U0[2], errors=np.array(errors),
         overshoot_k=overshoot[0], overshoot_slice=overshoot[1],
         snap_rho=np.stack([s[0] for s in done_snaps]), snap_u=np.stack([s[1] for s in done_snaps]),
         snap_theta=np.stack([s[2] for s in done_snaps]), seconds=time.time() - tic, workers=workers)


def job_cfg4w1(workers):
    w = config(4)
    m, prob = oracle_setup(w)
    U0 = O.project(O.lift(*w.raw_moments(), m), m)
    t = prob.times
    tic = time.time()
    f = O.lift(*U0, m, normalize=False)
    f = O.fine_propagate(f, float(t[0]), float(t[1]), m, w.eps, w.bc, None, prob.dt_f)
    sec = time.time() - tic
    P = O.project(f, m)
    G = O.G(prob, U0, 1)
    cells = np.arange(1016, 1032)
    mx, my, mz = (np.add.reduce(f[cells], axis=(2, 3)), np.add.reduce(f[cells], axis=(1, 3)),
                  np.add.reduce(f[cells], axis=(1, 2)))
    save("cfg4w1", rho0=U0[0], u0=U0[1], theta0=U0[2], rho=P[0], u=P[1], theta=P[2],
         g_rho=G[0], g_u=G[1], g_theta=G[2], cells=cells, mx=mx, my=my, mz=mz,
         slice_i=np.array([0, 1024, 2047]), slices=f[[0, 1024, 2047], :, :, 32], seconds=sec)


def _abs_overshoot(w, workers, name):
    R, g, bc, d, kin, flu = ref_setup(w)
    U0 = R.project(R.lift(R.MomentField(*w.raw_moments()), g), g)
    tic = time.time()
    slice_index, err = 0, np.nan
    try:
        _, rec = R.run_parareal(U0, R.PararealConfig(1, 1e-300, workers=workers), d, kin, flu)
        err = rec[0].error
    except R.CorrectionOvershootError as e:
        slice_index = e.slice_index
    print(name, "overshoot slice", slice_index, flush=True)
    save(name, overshoot_slice=slice_index, error=err, seconds=time.time() - tic)


def job_abs_cfg2(workers):
    _abs_overshoot(replace(config(2, 1.0), outflow=False), workers, "abs_cfg2")


def job_abs_cfg4x8(workers):
    _abs_overshoot(replace(config(4), outflow=False, nv=(8, 8, 8)), workers, "abs_cfg4x8")


if __name__ == "__main__":
    job = sys.argv[1]
    nw = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    if job == "cfg3a_pert":
        job_cfg3a(nw, perturb=1e-13)
    elif job.startswith("cfg2_e"):
        job_cfg2(float(job[6:]), nw)
    else:
        globals()["job_" + job](nw)
