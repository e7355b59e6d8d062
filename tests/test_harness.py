"""Harness and CLI parity with the reference's report format
(pkg/tests/test_bench.py, test_cli.py): report arithmetic, writers and
config handling on CPU; timed runs, sweeps and the solve/bench commands on
the GPU path (marked gpu)."""

import csv
import json

import pytest

from conftest import channel_cloud, lattice_cloud
from paper_2108_07031_b200 import SolverConfig, write_point_cloud
from paper_2108_07031_b200.cli import CONFIG_DEFAULTS, build_parser, main, read_config_file, resolve_config
from paper_2108_07031_b200.harness import (
    CSV_FIELDS,
    POINT_LEVELS,
    BenchmarkReport,
    SweepCell,
    speedup,
    summary_rows,
    sweep,
    timed_run,
    write_reports_json,
    write_summary_csv,
)


class TickClock:
    def __init__(self, step=1.0):
        self.t, self.step = 0.0, step

    def __call__(self):
        self.t += self.step
        return self.t


def cfg(**kw):
    base = dict(mach=0.63, aoa_deg=2.0, cfl=0.2, n_outer=5, n_inner=1)
    base.update(kw)
    return SolverConfig(**base)


# ------------------------------------------------------------------ CPU


def test_rdp_and_shares_hand_computed():
    rep = BenchmarkReport.from_timing(points=625000, iterations=1000, wall_seconds=10.0)
    assert rep.rdp == 1.6e-8
    rep = BenchmarkReport.from_timing(points=100, iterations=10, wall_seconds=8.0,
                                      stage_seconds={"flux_residual": 6.0, "residue": 1.0})
    assert rep.stage_shares == {"flux_residual": 0.75, "residue": 0.125}
    assert BenchmarkReport.from_timing(points=10, iterations=5, wall_seconds=0.0).rdp == 0.0


def test_report_validation_and_speedup():
    for kw in (dict(points=0, iterations=1, wall_seconds=1.0), dict(points=1, iterations=0, wall_seconds=1.0),
               dict(points=1, iterations=1, wall_seconds=-0.5)):
        with pytest.raises(ValueError):
            BenchmarkReport.from_timing(**kw)
    slow = BenchmarkReport.from_timing(points=2**20, iterations=2**10, wall_seconds=14.4090e-8 * 2**30)
    fast = BenchmarkReport.from_timing(points=2**20, iterations=2**10, wall_seconds=5.1200e-8 * 2**30)
    assert speedup(fast, slow) == 14.4090e-8 / 5.1200e-8
    stuck = BenchmarkReport.from_timing(points=1, iterations=1, wall_seconds=0.0)
    with pytest.raises(ValueError):
        speedup(stuck, fast)


def test_point_levels_include_reference_and_baseline_sizes():
    assert POINT_LEVELS["2.5k"] == (84, 30, 1.15, 20.0) and POINT_LEVELS["40k"] == (400, 100, 1.06, 20.0)
    assert POINT_LEVELS["40m"] == (12648, 3162, 1.001821, 20.0)


def test_summary_and_writers_round_trip(tmp_path):
    ok1 = BenchmarkReport.from_timing(points=1000, iterations=100, wall_seconds=7.0)
    ok2 = BenchmarkReport.from_timing(points=1000, iterations=100, wall_seconds=3.5)
    rows = summary_rows([SweepCell("a", ok1), SweepCell("broken", error="boom"), SweepCell("b", ok2)])
    assert [r["speedup"] for r in rows] == ["1", "failed", "2"]
    write_summary_csv(tmp_path / "s.csv", rows)
    with open(tmp_path / "s.csv", newline="") as fh:
        back = list(csv.DictReader(fh))
    assert list(back[0]) == list(CSV_FIELDS) and float(back[0]["rdp"]) == ok1.rdp and back[1]["speedup"] == "failed"
    write_reports_json(tmp_path / "r.json", [ok1, ok2])
    payload = json.loads((tmp_path / "r.json").read_text())
    assert len(payload) == 2 and payload[0]["rdp"] == ok1.rdp and payload[0]["host"]["cpus"] >= 1


def test_sweep_argument_validation():
    cloud = lattice_cloud(5, classify_boundary=True)
    with pytest.raises(ValueError):
        sweep(cfg(), cloud, "cfl", [0.1])
    with pytest.raises(ValueError):
        sweep(cfg(), None, "threads", [1])
    with pytest.raises(ValueError):
        timed_run(cfg(), cloud, warmup=5, clock=TickClock())


def test_config_file_and_precedence(tmp_path, monkeypatch):
    f = tmp_path / "run.cfg"
    f.write_text("# c\nmach = 0.7   # inline\n\niters = 250\ntol = none\n")
    assert read_config_file(f) == {"mach": 0.7, "iters": 250, "tol": None}
    f.write_text("mach = 0.7\n\nwarp = 9\n")
    with pytest.raises(ValueError, match=r"run\.cfg:3: unknown key 'warp'"):
        read_config_file(f)
    f.write_text("mach 0.7\n")
    with pytest.raises(ValueError, match=r"run\.cfg:1: expected 'key = value'"):
        read_config_file(f)
    f.write_text("mach = 0.7\ncfl = 0.35\n")
    args = build_parser().parse_args(["solve", "--grid", "g", "--out", "o", "--config", str(f), "--cfl", "0.1"])
    monkeypatch.setenv("KMF_THREADS", "3")
    merged = resolve_config(args)
    assert merged["mach"] == 0.7 and merged["cfl"] == 0.1 and merged["iters"] == CONFIG_DEFAULTS["iters"]
    assert merged["threads"] == 3


def test_generate_info_validate_and_errors(tmp_path, capsys):
    out = tmp_path / "g.txt"
    assert main(["generate", "--chord-points", "80", "--layers", "30", "--out", str(out)]) == 0
    assert "wrote 2400 points (80 wall, 80 outer)" in capsys.readouterr().out
    assert main(["info", "--grid", str(out)]) == 0
    text = capsys.readouterr().out
    assert "points: 2400" in text and "min spacing:" in text
    assert main(["validate", "--grid", str(out)]) == 2
    assert main(["info", "--grid", str(tmp_path / "missing.txt")]) == 1
    assert "error:" in capsys.readouterr().err
    assert main(["bench", "--out", str(tmp_path / "b")]) == 2


# ------------------------------------------------------------------ GPU


@pytest.mark.gpu
def test_timed_run_counts_only_post_warmup(gpu):
    cloud = lattice_cloud(7, h=0.5, classify_boundary=True)
    rep = timed_run(cfg(), cloud, warmup=2, clock=TickClock())
    assert rep.points == 49 and rep.iterations == 3 and rep.rdp == rep.wall_seconds / (3 * 49)
    assert rep.stage_shares["q_derivatives"] > 0 and rep.stage_shares["flux_residual"] > 0
    assert rep.config["mach"] == 0.63 and "gpu" in rep.host
    bare = timed_run(cfg(n_outer=3), cloud, warmup=0, clock=TickClock())
    assert bare.wall_seconds == rep.wall_seconds


@pytest.mark.gpu
def test_sweep_modes_points_and_failure_capture(gpu, small_naca):
    cloud = lattice_cloud(7, h=0.5, classify_boundary=True)
    out = sweep(cfg(n_outer=3), cloud, "mode", ["fused", "split4", "bogus"], warmup=0, clock=TickClock())
    assert [c.failed for c in out.cells] == [False, False, True] and out.any_failed
    assert [r["speedup"] for r in out.rows] == ["1", "1", "failed"]
    pts = sweep(cfg(n_outer=2), None, "points", [(80, 30, 1.15, 20.0)], warmup=0, clock=TickClock())
    assert not pts.any_failed and pts.cells[0].report.points == small_naca.n_points


@pytest.mark.gpu
def test_cli_solve_and_bench_outputs(gpu, tmp_path, capsys):
    grid = tmp_path / "channel.txt"
    write_point_cloud(channel_cloud(), grid)
    out = tmp_path / "run"
    assert main(["solve", "--grid", str(grid), "--out", str(out), "--iters", "5", "--aoa", "0"]) == 0
    assert "5 iterations, final residue" in capsys.readouterr().out
    sol = list(csv.DictReader(open(out / "solution.csv")))
    assert len(sol) == channel_cloud().n_points and set(sol[0]) == {"x", "y", "rho", "u1", "u2", "p"}
    assert len(list(csv.DictReader(open(out / "history.csv")))) == 5
    assert (out / "wall.csv").read_text().startswith("x,y,cp\n")
    assert "iters = 5" in (out / "config.txt").read_text()
    o1 = tmp_path / "run1"
    assert main(["solve", "--grid", str(grid), "--out", str(o1), "--iters", "3", "--order", "1"]) == 0
    assert "order = 1" in (o1 / "config.txt").read_text()
    assert len(list(csv.DictReader(open(o1 / "history.csv")))) == 3
    b = tmp_path / "bench"
    assert main(["bench", "--grid", str(grid), "--out", str(b), "--iters", "4", "--warmup", "1",
                 "--modes", "fused,split4"]) == 0
    rows = list(csv.DictReader(open(b / "summary.csv")))
    assert [r["level"] for r in rows] == ["fused/t1", "split4/t1"]
    assert len(json.loads((b / "reports.json").read_text())) == 2
