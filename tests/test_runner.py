"""Runner layer: config files, artifacts, CLI, mode drivers."""

from pathlib import Path

import numpy as np
import pytest

from helpers import rel_inf

P = pytest.importorskip("paper_2502_02704_b200")
from paper_2502_02704_b200 import runner  # noqa: E402
from paper_2502_02704_b200.__main__ import main as cli_main  # noqa: E402

GOLD = Path(__file__).resolve().parent / "golden"
CRIT11 = """# the reference's criterion-11 shock tube
case = sod
x_min = 0.0
x_max = 2.0
n_x = 20
v_max = 5.0
n_vx = 8
n_vy = 8
n_vz = 8
epsilon = 1e-2
bc = absorbing
t_final = 0.1
n_g = 8
n_f = 32
k_max = 8
tol = 1e-8
"""


def test_config_presets_overrides_and_errors(tmp_path):
    p = tmp_path / "a.cfg"
    p.write_text("preset = beams\nn_x = 50  # coarser\nworkers = 3\n")
    cfg = P.parse_config(p)
    assert (cfg.case, cfg.n_x, cfg.n_vx, cfg.epsilon, cfg.bc, cfg.workers) == \
        ("beams", 50, 256, 1e-5, "periodic", 3)
    p.write_text(CRIT11)
    cfg = P.parse_config(p)
    d = P.build_discretization(cfg)
    assert d.time.n_g == 8 and d.phase.space.dx == 0.1
    kin, flu = P.build_params(cfg, d)
    assert kin.force is None and kin.epsilon == 1e-2
    for bad, msg in (("n_x 3\n", ":1: expected key=value"), ("nope = 1\n", "unknown key"),
                     ("preset = sod\nn_x = many\n", ":2: bad value"),
                     ("case = sod\n", "required keys missing"), ("preset = jet\n", "unknown preset"),
                     ("preset = sod\nmode = magic\n", "unknown mode"),
                     ("preset = sod\ncfl_fluid = 1.5\n", "cfl_fluid"),
                     ("preset = sod\nalpha = 2\n", "alpha"),
                     ("preset = sod\ncoarse = navier\n", "coarse model"),
                     ("preset = sod\nx_scheme = weno\n", "x_scheme"),
                     ("preset = sod\nschedule = eager\n", "schedule")):
        p.write_text(bad)
        with pytest.raises(P.ConfigurationError, match=msg):
            P.parse_config(p)


def test_config_extension_keys(tmp_path):
    p = tmp_path / "x.cfg"
    p.write_text("preset = sod\nalpha = 1\ncoarse = drift_diffusion\nschedule = pipelined\n")
    cfg = P.parse_config(p)
    kin, flu = P.build_params(cfg, P.build_discretization(cfg))
    assert (kin.alpha, flu.model, cfg.schedule) == (1, "drift_diffusion", "pipelined")
    p.write_text("preset = sod\nx_scheme = muscl\n")
    kin, _ = P.build_params(P.parse_config(p), P.build_discretization(P.parse_config(p)))
    assert kin.scheme == "muscl"


def test_artifacts_round_trip_exactly(tmp_path):
    rng = np.random.default_rng(0)
    sp = P.build_spatial_grid(0.0, 2.0, 7)
    snaps = [P.MomentField(rng.random(7), rng.normal(size=(7, 3)), rng.random(7)) for _ in range(3)]
    paths = P.write_snapshots(snaps, sp, tmp_path)
    assert [p.name for p in paths] == ["snap_00000.csv", "snap_00001.csv", "snap_00002.csv"]
    for U, p in zip(snaps, paths):
        d = P.read_snapshot(p)
        assert np.array_equal(d["rho"], U.rho) and np.array_equal(d["uy"], U.u[:, 1])
        assert np.array_equal(d["x"], sp.centers)
    assert paths[0].read_text().splitlines()[0] == "x,rho,ux,uy,uz,theta"
    recs = [P.ConvergenceRecord(1, 0.1 + 0.2, 1e-3), P.ConvergenceRecord(2, 1e-17, 2.5)]
    P.write_convergence(recs, tmp_path)
    assert P.read_convergence(tmp_path / "convergence.csv") == recs
    P.write_timing(P.TimingReport(iterations=[1.0], speedup=2.0), tmp_path)
    assert '"speedup": 2.0' in (tmp_path / "timing.json").read_text()


def test_cli_exit_code_two_on_solver_error(tmp_path, capsys):
    p = tmp_path / "bad.cfg"
    p.write_text("preset = sod\nbc = reflective\n")
    assert cli_main(["run", "--config", str(p)]) == 2
    assert "unknown bc" in capsys.readouterr().err


def test_case_data():
    sp = P.build_spatial_grid(0.0, 2.0, 8)
    U = P.sod_moments(sp)
    assert list(U.rho) == [1.0] * 4 + [0.125] * 4
    B = P.blast_moments(sp)
    assert B.u[0, 0] == 1.0 and B.u[4, 0] == 0.0 and B.u[-1, 0] == -1.0
    assert P.external_force(np.array([0.0, 1.0, 2.0])).tolist() == [0.0, 0.0, 0.0]
    assert P.external_force(np.array([0.5]))[0] == pytest.approx(0.791015625)
    assert P.force_field("sod", sp) is None and P.force_field("beams", sp).shape == (8,)


# --------------------------------------------------------------------- GPU

@pytest.mark.gpu
def test_run_mode_parareal_and_fine_match_reference_artifacts(tmp_path):
    g = np.load(GOLD / "artifacts.npz")
    p = tmp_path / "c.cfg"
    p.write_text(CRIT11)
    cfg = P.parse_config(p)
    out = P.run_mode(cfg, tmp_path / "par")
    files = sorted(out.glob("snap_*.csv"))
    assert len(files) == 9
    cols = ("x", "rho", "ux", "uy", "uz", "theta")
    got = np.stack([np.stack([P.read_snapshot(f)[c] for c in cols]) for f in files])
    assert np.array_equal(got[:, 0], g["par"][:, 0])
    for n in range(9):
        for c in (1, 5):
            assert rel_inf(got[n, c], g["par"][n, c]) <= 1e-10
        scale = max(np.max(np.abs(g["par"][n, 2:5])), np.sqrt(np.max(g["par"][n, 5])))
        assert np.max(np.abs(got[n, 2:5] - g["par"][n, 2:5])) <= 1e-10 * scale
    recs = P.read_convergence(out / "convergence.csv")
    assert [r.k for r in recs] == list(g["k"])
    np.testing.assert_allclose([r.error for r in recs], g["err"], rtol=1e-8)
    from dataclasses import replace
    outf = P.run_mode(replace(cfg, mode="fine"), tmp_path / "fine")
    fine = np.stack([np.stack([P.read_snapshot(f)[c] for c in cols])
                     for f in sorted(outf.glob("snap_*.csv"))])
    for n in range(9):
        assert rel_inf(fine[n, 1], g["fine"][n, 1]) <= 1e-10
        assert rel_inf(fine[n, 5], g["fine"][n, 5]) <= 1e-10
    # determinism across runs: byte-identical artifacts
    out2 = P.run_mode(replace(cfg, workers=2), tmp_path / "par2")
    for a, b in zip(files, sorted(out2.glob("snap_*.csv"))):
        assert a.read_bytes() == b.read_bytes()


@pytest.mark.gpu
def test_run_comparison_writes_report(tmp_path):
    p = tmp_path / "c.cfg"
    p.write_text(CRIT11.replace("k_max = 8", "k_max = 2"))
    rep = P.run_comparison(P.parse_config(p), tmp_path / "cmp")
    assert rep.speedup > 0 and rep.parareal_seconds > 0 and len(rep.iterations) == 2
    for sub in ("fluid", "fine", "parareal"):
        assert len(list((tmp_path / "cmp" / sub).glob("snap_*.csv"))) == 9
    assert (tmp_path / "cmp" / "timing.json").exists()
    assert cli_main(["run", "--config", str(p), "--mode", "fluid", "--out", str(tmp_path / "cli")]) == 0
