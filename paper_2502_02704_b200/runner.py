"""Mode drivers, run configuration, test-case data and CSV/JSON artifacts.

The command-line layer of the reference (ref/runner.py, ref/config.py,
ref/cases.py, ref/io.py, ref/cli.py), kept thin around the GPU solver:

* ``run_fine_mode`` marches ONE distribution through all windows on the
  device (no re-lift, ref/runner.py:40-49) -- the serial fine reference and
  the speed-up denominator of ``run_comparison``;
* ``run_fluid_mode`` / ``run_parareal_mode`` are the G sweep and the parareal
  loop of this package;
* artifacts are byte-compatible with the reference: ``snap_NNNNN.csv``
  (x, rho, ux, uy, uz, theta; repr floats), ``convergence.csv`` (k, error,
  seconds), ``timing.json``;
* configuration files are the reference's key=value format (presets sod /
  blast / beams, ``#`` comments, per-line error messages).
"""

from __future__ import annotations

import csv
import json
import time
from dataclasses import asdict, dataclass, field
from pathlib import Path
from typing import Optional

import numpy as np
import torch

from .errors import ConfigurationError
from .fluid import FluidParams
from .grid import (BoundaryKind, Discretization, PhaseGrid, build_spatial_grid, build_time_grids,
                   build_velocity_grid)
from .kinetic import ConstantTau, KineticParams, constant_tau, propagate_kinetic
from .lifting import Distribution, lift
from .moments import MomentField, project
from .parareal import (ConvergenceRecord, PararealConfig, estimate_k_opt, initial_coarse_sweep,
                       run_parareal)

__all__ = ["CasePreset", "PRESETS", "sod_moments", "blast_moments", "external_force",
           "initial_distribution", "initial_moments", "force_field", "RunConfig", "parse_config",
           "build_discretization", "build_params", "TimingReport", "write_snapshots",
           "read_snapshot", "write_convergence", "read_convergence", "write_timing", "prepare",
           "run_fluid_mode", "run_fine_mode", "run_parareal_mode", "run_mode", "run_comparison"]


# ---------------------------------------------------------------------------
# test problems (ref/cases.py:29-137)
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class CasePreset:
    name: str
    x_min: float
    x_max: float
    n_x: int
    v_max: float
    n_v: tuple
    epsilon: float
    bc: BoundaryKind
    t_final: float
    n_g: int
    n_f: int
    k_max: int
    tol: float
    has_force: bool


# the paper's three test problems at publication scale (ref/cases.py:49-56)
PRESETS = {
    "sod": CasePreset("sod", 0.0, 2.0, 200, 8.0, (32, 32, 32), 1e-2, BoundaryKind.ABSORBING, 0.5,
                      200, 800, 80, 1e-8, False),
    "blast": CasePreset("blast", 0.0, 2.0, 200, 8.0, (32, 32, 32), 1e-2, BoundaryKind.ABSORBING,
                        0.5, 200, 800, 10, 1e-8, False),
    "beams": CasePreset("beams", 0.0, 2.0, 100, 8.0, (256, 16, 16), 1e-5, BoundaryKind.PERIODIC,
                        0.5, 200, 800, 80, 1e-8, True),
}


def _piecewise(space, edges, states) -> MomentField:
    """states[q] on [edges[q-1], edges[q]) classified by cell centre."""
    x = space.centers
    rho, th = np.empty_like(x), np.empty_like(x)
    u = np.zeros((x.size, 3))
    bounds = [-np.inf] + list(edges) + [np.inf]
    for q, (r, ux, t) in enumerate(states):
        m = (x >= bounds[q]) & (x < bounds[q + 1])
        rho[m], u[m, 0], th[m] = r, ux, t
    return MomentField(rho, u, th)


def sod_moments(space) -> MomentField:
    """(1, 0, 1) left of x = 1, (0.125, 0, 0.8) right (ref/cases.py:73-77)."""
    return _piecewise(space, [1.0], [(1.0, 0.0, 1.0), (0.125, 0.0, 0.8)])


def blast_moments(space) -> MomentField:
    """Opposed streams around a hot band on [0.4, 1.6] (ref/cases.py:80-84)."""
    return _piecewise(space, [0.4, 1.6], [(1.0, 1.0, 2.0), (1.0, 0.0, 0.25), (1.0, -1.0, 2.0)])


def external_force(x) -> np.ndarray:
    """-5 x^4 (x-2)^4 (x-1): confines mass toward x = 1 (ref/cases.py:111-114)."""
    x = np.asarray(x, dtype=float)
    return -5.0 * x ** 4 * (x - 2.0) ** 4 * (x - 1.0)


def initial_distribution(case: str, grid, bc=None) -> Distribution:
    """Kinetic initial state of a case, on the device."""
    if case == "sod":
        return lift(sod_moments(grid.space), grid, bc=bc)
    if case == "blast":
        return lift(blast_moments(grid.space), grid, bc=bc)
    if case == "beams":  # two unit Maxwellian beams at u_x = +-1 (ref/cases.py:89-108)
        n = grid.space.n_x
        uf = np.zeros((n, 3))
        uf[:, 0] = 1.0
        a = lift(MomentField(np.ones(n), uf, np.ones(n)), grid, bc=bc).device_tensor()
        b = lift(MomentField(np.ones(n), -uf, np.ones(n)), grid, bc=bc).device_tensor()
        return Distribution(a.add_(b))
    raise ConfigurationError("unknown case '%s'" % case)


def initial_moments(case: str, grid) -> MomentField:
    return project(initial_distribution(case, grid), grid)


def force_field(case: str, space):
    if case not in PRESETS:
        raise ConfigurationError("unknown case '%s'" % case)
    return external_force(space.centers) if case == "beams" else None


# ---------------------------------------------------------------------------
# key=value run configuration (ref/config.py:25-164)
# ---------------------------------------------------------------------------

MODES = ("parareal", "fine", "fluid")


@dataclass
class RunConfig:
    case: str
    x_min: float
    x_max: float
    n_x: int
    v_max: float
    n_vx: int
    n_vy: int
    n_vz: int
    epsilon: float
    bc: str
    t_final: float
    n_g: int
    n_f: int
    k_max: int
    tol: float
    tau: float = 1.0
    cfl_kinetic: float = 0.5
    cfl_fluid: float = 0.9
    workers: int = 1
    mode: str = "parareal"
    out_dir: str = "out"
    use_frozen_prefix: bool = True
    preset: Optional[str] = None
    # extensions beyond the reference
    alpha: int = 0                 # 1: diffusive scaling
    coarse: str = "euler"          # "drift_diffusion": the diffusive G
    x_scheme: str = "upwind"       # "muscl": minmod-limited x transport
    schedule: str = "phased"       # "pipelined": coarse work trails the fine windows


def _boolean(text: str) -> bool:
    t = text.lower()
    if t in ("true", "yes", "on", "1"):
        return True
    if t in ("false", "no", "off", "0"):
        return False
    raise ValueError("not a boolean: %r" % (text,))


_TYPES = dict(preset=str, case=str, bc=str, mode=str, out_dir=str, x_min=float, x_max=float,
              v_max=float, epsilon=float, t_final=float, tol=float, tau=float, cfl_kinetic=float,
              cfl_fluid=float, n_x=int, n_vx=int, n_vy=int, n_vz=int, n_g=int, n_f=int, k_max=int,
              workers=int, use_frozen_prefix=_boolean, alpha=int, coarse=str, x_scheme=str,
              schedule=str)
_NEEDED = ("case", "x_min", "x_max", "n_x", "v_max", "n_vx", "n_vy", "n_vz", "epsilon", "bc",
           "t_final", "n_g", "n_f", "k_max", "tol")


def parse_config(path) -> RunConfig:
    """Read and validate a key=value run configuration."""
    path = Path(path)
    kv = {}
    for ln, raw in enumerate(path.read_text().splitlines(), start=1):
        body = raw.split("#", 1)[0].strip()
        if not body:
            continue
        if "=" not in body:
            raise ConfigurationError("%s:%d: expected key=value, got %r" % (path, ln, raw))
        key, _, val = body.partition("=")
        key, val = key.strip(), val.strip()
        if key not in _TYPES:
            raise ConfigurationError("%s:%d: unknown key '%s'" % (path, ln, key))
        try:
            kv[key] = _TYPES[key](val)
        except ValueError as exc:
            raise ConfigurationError("%s:%d: bad value for '%s': %s" % (path, ln, key, exc))
    name = kv.pop("preset", None)
    if name is not None:
        if name not in PRESETS:
            raise ConfigurationError("unknown preset '%s', expected one of %s"
                                     % (name, sorted(PRESETS)))
        p = PRESETS[name]
        vals = dict(case=p.name, x_min=p.x_min, x_max=p.x_max, n_x=p.n_x, v_max=p.v_max,
                    n_vx=p.n_v[0], n_vy=p.n_v[1], n_vz=p.n_v[2], epsilon=p.epsilon, bc=p.bc.value,
                    t_final=p.t_final, n_g=p.n_g, n_f=p.n_f, k_max=p.k_max, tol=p.tol)
        vals.update(kv)
        vals["preset"] = name
    else:
        missing = [k for k in _NEEDED if k not in kv]
        if missing:
            raise ConfigurationError("%s: no preset given and required keys missing: %s"
                                     % (path, missing))
        vals = kv
    cfg = RunConfig(**vals)
    if cfg.case not in PRESETS:
        raise ConfigurationError("unknown case '%s'" % cfg.case)
    if cfg.bc not in [k.value for k in BoundaryKind]:
        raise ConfigurationError("unknown bc '%s'" % cfg.bc)
    if cfg.mode not in MODES:
        raise ConfigurationError("unknown mode '%s', expected one of %s" % (cfg.mode, MODES))
    for label in ("epsilon", "tau", "tol"):
        if not getattr(cfg, label) > 0:
            raise ConfigurationError("need %s > 0, got %r" % (label, getattr(cfg, label)))
    for label in ("cfl_kinetic", "cfl_fluid"):
        if not 0.0 < getattr(cfg, label) <= 1.0:
            raise ConfigurationError("need 0 < %s <= 1, got %r" % (label, getattr(cfg, label)))
    if cfg.k_max < 1 or cfg.workers < 1:
        raise ConfigurationError("need k_max >= 1 and workers >= 1")
    if cfg.alpha not in (0, 1):
        raise ConfigurationError("need alpha in {0, 1}, got %r" % (cfg.alpha,))
    if cfg.coarse not in ("euler", "drift_diffusion"):
        raise ConfigurationError("unknown coarse model '%s'" % cfg.coarse)
    if cfg.x_scheme not in ("upwind", "muscl"):
        raise ConfigurationError("unknown x_scheme '%s'" % cfg.x_scheme)
    if cfg.schedule not in ("phased", "pipelined"):
        raise ConfigurationError("unknown schedule '%s'" % cfg.schedule)
    return cfg


def build_discretization(cfg: RunConfig) -> Discretization:
    g = PhaseGrid(build_spatial_grid(cfg.x_min, cfg.x_max, cfg.n_x),
                  build_velocity_grid(cfg.v_max, (cfg.n_vx, cfg.n_vy, cfg.n_vz)))
    return Discretization(g, build_time_grids(cfg.t_final, cfg.n_g, cfg.n_f), BoundaryKind(cfg.bc))


def build_params(cfg: RunConfig, disc: Discretization):
    E = force_field(cfg.case, disc.phase.space)
    tau = constant_tau if cfg.tau == 1.0 else ConstantTau(cfg.tau)
    return (KineticParams(cfg.epsilon, tau=tau, force=E, cfl=cfg.cfl_kinetic, alpha=cfg.alpha,
                          scheme=cfg.x_scheme),
            FluidParams(force=E, cfl=cfg.cfl_fluid, model=cfg.coarse))


# ---------------------------------------------------------------------------
# artifacts (ref/io.py:34-108): repr floats -> byte-identical, exact round trip
# ---------------------------------------------------------------------------

@dataclass
class TimingReport:
    iterations: list = field(default_factory=list)
    t_lift: float = 0.0
    t_kin: float = 0.0
    t_proj: float = 0.0
    t_fluid: float = 0.0
    fine_seconds: Optional[float] = None
    fluid_seconds: Optional[float] = None
    parareal_seconds: Optional[float] = None
    speedup: Optional[float] = None
    k_opt: Optional[int] = None


def write_snapshots(snapshots, space, out_dir) -> list:
    out = Path(out_dir)
    out.mkdir(parents=True, exist_ok=True)
    paths = []
    for n, U in enumerate(snapshots):
        p = out / ("snap_%05d.csv" % n)
        with p.open("w", newline="") as fh:
            w = csv.writer(fh)
            w.writerow(["x", "rho", "ux", "uy", "uz", "theta"])
            for i in range(U.n_x):
                w.writerow([repr(float(v)) for v in (space.centers[i], U.rho[i], U.u[i, 0],
                                                      U.u[i, 1], U.u[i, 2], U.theta[i])])
        paths.append(p)
    return paths


def read_snapshot(path) -> dict:
    with Path(path).open(newline="") as fh:
        rows = list(csv.reader(fh))
    data = np.asarray([[float(c) for c in r] for r in rows[1:]])
    return {name: data[:, j] for j, name in enumerate(rows[0])}


def write_convergence(records, out_dir) -> Path:
    out = Path(out_dir)
    out.mkdir(parents=True, exist_ok=True)
    p = out / "convergence.csv"
    with p.open("w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(["k", "error", "seconds"])
        for r in records:
            w.writerow([r.k, repr(r.error), repr(r.seconds)])
    return p


def read_convergence(path) -> list:
    with Path(path).open(newline="") as fh:
        rows = list(csv.reader(fh))[1:]
    return [ConvergenceRecord(int(k), float(e), float(s)) for k, e, s in rows]


def write_timing(report: TimingReport, out_dir) -> Path:
    out = Path(out_dir)
    out.mkdir(parents=True, exist_ok=True)
    p = out / "timing.json"
    p.write_text(json.dumps(asdict(report), indent=2) + "\n")
    return p


# ---------------------------------------------------------------------------
# mode drivers (ref/runner.py:27-117)
# ---------------------------------------------------------------------------

def prepare(cfg: RunConfig):
    disc = build_discretization(cfg)
    kinetic, fluid = build_params(cfg, disc)
    U0 = project(initial_distribution(cfg.case, disc.phase, disc.bc), disc.phase, disc.bc)
    return disc, kinetic, fluid, U0


def run_fluid_mode(cfg, disc, fluid, U0):
    return initial_coarse_sweep(U0, disc, fluid).snapshots


def run_fine_mode(cfg, disc, kinetic, group=None):
    """One distribution marched across all windows, f resident on the device.

    Under torch.distributed (world > 1) the x cells are sharded over the
    ranks (``sharded.SlabFine``, halo exchange per step) -- bitwise the
    single-GPU run, the snapshots gathered on every rank."""
    dist = torch.distributed
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        return _run_fine_sharded(cfg, disc, kinetic, group)
    f = initial_distribution(cfg.case, disc.phase, disc.bc)
    t = disc.time.coarse_times
    snaps = [project(f, disc.phase, disc.bc)]
    for n in range(1, disc.time.n_g + 1):
        f = propagate_kinetic(f, float(t[n - 1]), float(t[n]), disc.phase, kinetic, disc.bc,
                              dt_max=disc.time.dt_f)
        snaps.append(project(f, disc.phase, disc.bc))
    return snaps


def _run_fine_sharded(cfg, disc, kinetic, group):
    from .sharded import SlabFine
    sl = SlabFine(disc.phase, disc.bc, kinetic, group=group)
    f = initial_distribution(cfg.case, disc.phase, disc.bc).device_tensor(sl.device)
    f = f[sl.x0:sl.x0 + sl.n].contiguous()
    t = disc.time.coarse_times
    f, m = sl.propagate(0.0, 0.0, f0=f, want_moments=True)  # the projection of f0
    snaps = [MomentField.from_packed(sl.gather(m, 1))]
    for n in range(1, disc.time.n_g + 1):
        f, m = sl.propagate(float(t[n - 1]), float(t[n]), f0=f, dt_max=disc.time.dt_f,
                            want_moments=True)
        snaps.append(MomentField.from_packed(sl.gather(m, 1)))
    return snaps


def run_parareal_mode(cfg, disc, kinetic, fluid, U0, timing=None):
    pc = PararealConfig(cfg.k_max, cfg.tol, use_frozen_prefix=cfg.use_frozen_prefix,
                        workers=cfg.workers, pipelined=cfg.schedule == "pipelined")
    return run_parareal(U0, pc, disc, kinetic, fluid, timing=timing)


def run_mode(cfg: RunConfig, out_dir=None) -> Path:
    out = Path(out_dir if out_dir is not None else cfg.out_dir)
    disc, kinetic, fluid, U0 = prepare(cfg)
    if cfg.mode == "fluid":
        snaps = run_fluid_mode(cfg, disc, fluid, U0)
    elif cfg.mode == "fine":
        snaps = run_fine_mode(cfg, disc, kinetic)
    else:
        traj, recs = run_parareal_mode(cfg, disc, kinetic, fluid, U0)
        snaps = traj.snapshots
        write_convergence(recs, out)
    write_snapshots(snaps, disc.phase.space, out)
    return out


def _timed(fn):
    torch.cuda.synchronize()
    tic = time.perf_counter()
    res = fn()
    torch.cuda.synchronize()
    return res, time.perf_counter() - tic


def run_comparison(cfg: RunConfig, out_dir=None) -> TimingReport:
    out = Path(out_dir if out_dir is not None else cfg.out_dir)
    disc, kinetic, fluid, U0 = prepare(cfg)
    sp = disc.phase.space
    fl, t_fl = _timed(lambda: run_fluid_mode(cfg, disc, fluid, U0))
    write_snapshots(fl, sp, out / "fluid")
    fi, t_fi = _timed(lambda: run_fine_mode(cfg, disc, kinetic))
    write_snapshots(fi, sp, out / "fine")
    stages: dict = {}
    (traj, recs), t_pa = _timed(lambda: run_parareal_mode(cfg, disc, kinetic, fluid, U0, stages))
    write_snapshots(traj.snapshots, sp, out / "parareal")
    write_convergence(recs, out / "parareal")
    rep = TimingReport(iterations=[r.seconds for r in recs],
                       t_lift=stages.get("t_lift", 0.0), t_kin=stages.get("t_kin", 0.0),
                       t_proj=stages.get("t_proj", 0.0), t_fluid=stages.get("t_fluid", 0.0),
                       fine_seconds=t_fi, fluid_seconds=t_fl, parareal_seconds=t_pa,
                       speedup=t_fi / t_pa,
                       k_opt=estimate_k_opt(stages.get("t_kin", 0.0), stages.get("t_fluid", 0.0),
                                            stages.get("t_lift", 0.0), stages.get("t_proj", 0.0),
                                            disc.time.n_g, cfg.workers))
    write_timing(rep, out)
    return rep
