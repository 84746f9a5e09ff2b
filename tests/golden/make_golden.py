"""Generate tests/golden/*.npz from the UNMODIFIED reference package.

Run in the build container, where /root/reference exists:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Each fixture stores its inputs and the reference outputs (small shapes, so
the files stay a few hundred KB).  The GPU box has no /root/reference; the
oracle and the CUDA path are pinned against these files there.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
sys.path.insert(0, str(REF))
import parabgk as R  # noqa: E402

OUT = Path(__file__).resolve().parent


def phase(nx, nv, vmax, x0=0.0, x1=1.0):
    return R.PhaseGrid(R.build_spatial_grid(x0, x1, nx), R.build_velocity_grid(vmax, nv))


def moments(rng, nx):
    return (rng.uniform(0.5, 1.5, nx), rng.uniform(-0.4, 0.4, (nx, 3)), rng.uniform(0.5, 1.5, nx))


def main():
    rng = np.random.default_rng(20250207)
    cases = {}

    # -- kinetic building blocks on a small anisotropic grid -----------------
    nx, nv, vm = 6, (8, 6, 5), 6.0
    g = phase(nx, nv, vm)
    rho, u, th = moments(rng, nx)
    U = R.MomentField(rho, u, th)
    f_raw = R.lift(U, g).values
    f = f_raw * rng.uniform(0.8, 1.2, f_raw.shape)
    E = 0.5 * np.sin(2 * np.pi * g.space.centers)
    kp = R.KineticParams(epsilon=2e-2)
    kpE = R.KineticParams(epsilon=2e-2, force=E)
    dt = 0.4 * R.stable_dt_kinetic(g, kpE)
    P = R.project(R.Distribution(f), g)
    out = dict(nx=nx, nv=np.array(nv), vmax=vm, rho=rho, u=u, theta=th, f=f, E=E, dt=dt,
               lift_raw=f_raw, lift_norm=R.lift(U, g, normalize_mass=True).values,
               proj_rho=P.rho, proj_u=P.u, proj_theta=P.theta,
               tr_per=R.transport_update(R.Distribution(f), dt, g, kp, R.BoundaryKind.PERIODIC).values,
               tr_abs=R.transport_update(R.Distribution(f), dt, g, kp, R.BoundaryKind.ABSORBING).values,
               tr_fieldper=R.transport_update(R.Distribution(f), dt, g, kpE,
                                              R.BoundaryKind.PERIODIC).values,
               relax=R.bgk_relax(R.Distribution(f), dt, g, kp).values,
               cap=R.stable_dt_kinetic(g, kp), capE=R.stable_dt_kinetic(g, kpE))
    t1 = 4.5 * out["cap"]
    out["t1"] = t1
    out["prop_abs"] = R.propagate_kinetic(R.Distribution(f), 0.0, t1, g, kp,
                                          R.BoundaryKind.ABSORBING).values
    out["prop_fieldper"] = R.propagate_kinetic(R.Distribution(f), 0.0, 4.5 * out["capE"], g, kpE,
                                               R.BoundaryKind.PERIODIC).values
    cases["kinetic"] = out

    # -- coarse propagator -----------------------------------------------------
    nx = 24
    g = phase(nx, 4, 8.0)
    rho, u, th = moments(rng, nx)
    E = 0.3 * np.cos(2 * np.pi * g.space.centers)
    res = {}
    for name, bc, force in (("abs", R.BoundaryKind.ABSORBING, None),
                            ("perE", R.BoundaryKind.PERIODIC, E)):
        V = R.propagate_fluid(R.MomentField(rho, u, th), 0.0, 0.04, g, R.FluidParams(force=force),
                              bc, dt_max=0.01)
        res.update({name + "_rho": V.rho, name + "_u": V.u, name + "_theta": V.theta})
    cases["fluid"] = dict(nx=nx, rho=rho, u=u, theta=th, E=E, **res)

    # -- parareal on a small Sod tube -----------------------------------------
    nx = 16
    g = phase(nx, 8, 8.0)
    disc = R.Discretization(g, R.build_time_grids(0.05, 4, 16), R.BoundaryKind.ABSORBING)
    x = g.space.centers
    U0 = R.MomentField(np.where(x < 0.5, 1.0, 0.125), np.zeros((nx, 3)),
                       np.where(x < 0.5, 1.0, 0.8))
    traj, rec = R.run_parareal(U0, R.PararealConfig(k_max=3, tol=1e-300), disc,
                               R.KineticParams(epsilon=1e-2), R.FluidParams())
    chain = R.fine_moment_chain(U0, disc, R.KineticParams(epsilon=1e-2))
    cases["parareal"] = dict(
        nx=nx, rho0=U0.rho, u0=U0.u, theta0=U0.theta,
        snap_rho=np.stack([s.rho for s in traj.snapshots]),
        snap_u=np.stack([s.u for s in traj.snapshots]),
        snap_theta=np.stack([s.theta for s in traj.snapshots]),
        errors=np.array([r.error for r in rec]),
        chain_rho=np.stack([s.rho for s in chain]),
        chain_theta=np.stack([s.theta for s in chain]))

    # -- known-answer scalars ---------------------------------------------------
    cases["scalars"] = dict(
        wd_10_3=np.array([R.work_distribution(10, 3, r)[:2] for r in range(3)]),
        kopt=R.estimate_k_opt(10.0, 0.1, 0.05, 0.05, 100, 32),
        stable_dt_200=R.stable_dt_kinetic(phase(200, 8, 8.0, 0.0, 2.0), R.KineticParams(1.0, cfl=0.9)),
        rusanov_sod=R.rusanov_flux(
            R.primitive_to_conserved(R.MomentField(np.array([1.0]), np.zeros((1, 3)),
                                                   np.array([1.0]))).to_array()[0],
            R.primitive_to_conserved(R.MomentField(np.array([0.125]), np.zeros((1, 3)),
                                                   np.array([0.8]))).to_array()[0]))

    # -- run_mode artifacts of the reference's criterion-11 configuration --------
    import tempfile
    with tempfile.TemporaryDirectory() as tmp:
        cfg = R.RunConfig(case="sod", x_min=0.0, x_max=2.0, n_x=20, v_max=5.0, n_vx=8, n_vy=8,
                          n_vz=8, epsilon=1e-2, bc="absorbing", t_final=0.1, n_g=8, n_f=32,
                          k_max=8, tol=1e-8, workers=1)
        outp = R.run_mode(cfg, tmp + "/par")
        snaps = [R.read_snapshot(p) for p in sorted(Path(outp).glob("snap_*.csv"))]
        recs = R.read_convergence(Path(outp) / "convergence.csv")
        from dataclasses import replace as _rep
        outf = R.run_mode(_rep(cfg, mode="fine"), tmp + "/fine")
        fine = [R.read_snapshot(p) for p in sorted(Path(outf).glob("snap_*.csv"))]
    cases["artifacts"] = dict(
        par=np.stack([np.stack([s[k] for k in ("x", "rho", "ux", "uy", "uz", "theta")]) for s in snaps]),
        k=np.array([r.k for r in recs]), err=np.array([r.error for r in recs]),
        fine=np.stack([np.stack([s[k] for k in ("x", "rho", "ux", "uy", "uz", "theta")]) for s in fine]))

    for name, d in cases.items():
        np.savez_compressed(OUT / ("%s.npz" % name), **d)
        print("wrote", name, sum(np.asarray(v).nbytes for v in d.values()), "bytes")


if __name__ == "__main__":
    main()
