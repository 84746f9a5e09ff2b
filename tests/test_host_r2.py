"""Host-side logic added in round 2 (no GPU): the multi-rank bench launcher's
checks, the executor / workers seam of the parareal driver, the CPU-baseline
sampler of the reference algorithm."""

import os
import sys
import warnings
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2502_02704_b200.configs import config  # noqa: E402


def test_bench_world_size_mismatch_fails_loudly(monkeypatch):
    import bench
    monkeypatch.setenv("WORLD_SIZE", "2")
    args = type("A", (), {"gpus": 4})()
    with pytest.raises(SystemExit) as info:
        bench.relaunch_if_needed(args)
    assert "WORLD_SIZE=2" in str(info.value)


def test_bench_matching_world_size_runs_in_place(monkeypatch):
    import bench
    monkeypatch.setenv("WORLD_SIZE", "4")
    bench.relaunch_if_needed(type("A", (), {"gpus": 4})())  # no relaunch, no error


def test_bench_relaunches_under_torchrun(monkeypatch):
    import bench
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    calls = []
    monkeypatch.setattr(bench.subprocess, "call", lambda cmd, env: calls.append((cmd, env)) or 0)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "3", "--steps", "2"])
    with pytest.raises(SystemExit) as info:
        bench.relaunch_if_needed(type("A", (), {"gpus": 3})())
    assert info.value.code == 0
    cmd, env = calls[0]
    assert "torch.distributed.run" in cmd and "--nproc-per-node=3" in cmd
    assert "--master-addr=127.0.0.1" in cmd and cmd[-4:] == ["--gpus", "3", "--steps", "2"]
    assert env["NCCL_DEBUG"] == "INFO"


def test_workers_and_executor_seam():
    from paper_2502_02704_b200 import parareal as PR
    from paper_2502_02704_b200.errors import ConfigurationError
    with warnings.catch_warnings(record=True) as got:
        warnings.simplefilter("always")
        ex = PR.make_executor(4, None, None, None)
    assert any(issubclass(x.category, RuntimeWarning) for x in got)
    PR._check_executor(ex)
    PR._check_executor(None)
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(1) as pool, pytest.raises(ConfigurationError):
        PR._check_executor(pool)


def test_cpu_sampler_slab_keeps_the_workload_spacing():
    from oracle.cpu_bench import slab_workload
    w = config(4)
    ws = slab_workload(w, 16)
    assert ws.nx == 16
    assert np.isclose((ws.x_max - ws.x_min) / ws.nx, (w.x_max - w.x_min) / w.nx, rtol=0, atol=1e-15)
    assert ws.x_min < 0.5 < ws.x_max  # centred on the Sod interface
    assert ws.window_steps() == w.window_steps()


def test_cpu_sampler_runs_whole_window_jumps():
    from dataclasses import replace
    from oracle.cpu_bench import window_rate, fine_rate
    w = replace(config(0), nv=(8, 8, 8))
    r = window_rate(w, 6, workers=2)
    assert r["cores"] == 2 and r["cell_updates"] == 2 * 6 * 512 * w.window_steps() and r["value"] > 0
    r1 = fine_rate(replace(config(1), nv=(8, 8, 8)), 8, 3)
    assert r1["cores"] == 1 and r1["cell_updates"] == 8 * 512 * 3
