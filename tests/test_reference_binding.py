"""The reference's OWN harness and CLI on the B200 path.

`integration.route_reference` binds the imported reference package to this
one the way INTEGRATION.md's kmf/_b200.py does; the reference's
kmf.bench (BenchmarkReport, timed_run, sweep, writers) and kmf.cli then run
unchanged and write their own report formats from B200 runs.

The reference is imported from baseline/_ref (its offline install, which
travels to the GPU box; `__graft_entry__.build()` creates it) or, on the
CPU only, from /root/reference.
"""

from __future__ import annotations

import csv
import importlib
import json
import sys

import numpy as np
import pytest

from conftest import ROOT
from paper_2108_07031_b200 import _lib
from paper_2108_07031_b200 import SolverConfig, build_stencils, solve
from paper_2108_07031_b200.integration import route_reference, unroute
from paper_2108_07031_b200.solver import STAGE_NAMES

REF_INSTALL = ROOT / "baseline" / "_ref"


def _import_kmf(allow_source: bool):
    roots = [REF_INSTALL]
    if allow_source:
        roots.append(__import__("pathlib").Path("/root/reference/pkg/src"))
    for root in roots:
        if (root / "kmf" / "__init__.py").exists():
            sys.path.insert(0, str(root))
            try:
                for name in [m for m in sys.modules if m == "kmf" or m.startswith("kmf.")]:
                    del sys.modules[name]
                kmf = importlib.import_module("kmf")
                for sub in ("solver", "geometry", "bench", "cli", "validation"):
                    importlib.import_module(f"kmf.{sub}")
                return kmf
            finally:
                sys.path.remove(str(root))
    pytest.skip("reference package not installed (baseline/_ref: run __graft_entry__.build())")


@pytest.fixture
def kmf_cpu():
    kmf = _import_kmf(allow_source=True)
    yield kmf
    unroute(kmf)


@pytest.fixture
def kmf_gpu(gpu):
    kmf = _import_kmf(allow_source=False)  # never /root/reference on the GPU box
    route_reference(kmf)
    yield kmf
    unroute(kmf)


def test_route_and_unroute_rebind_every_holder(kmf_cpu):
    kmf = kmf_cpu
    orig = {m: getattr(m, "solve") for m in (kmf, kmf.solver, kmf.bench, kmf.cli)}
    route_reference(kmf)
    for m in orig:
        assert m.solve is not orig[m] and m.solve.__module__ == "paper_2108_07031_b200.integration"
    assert kmf.geometry.build_stencils.__module__ == "paper_2108_07031_b200.integration"
    unroute(kmf)
    for m, fn in orig.items():
        assert m.solve is fn


@pytest.mark.skipif(_lib.lib().kmf_device_count() > 0, reason="checks the no-GPU behaviour")
def test_routed_reference_has_no_cpu_fallback(kmf_cpu):
    kmf = kmf_cpu
    route_reference(kmf)
    cloud = kmf.geometry.generate_naca_cloud(80, 30, 1.15, 20.0)
    with pytest.raises(_lib.DeviceError):
        kmf.bench.timed_run(kmf.solver.SolverConfig(mach=0.63, n_outer=3), cloud, warmup=1)


@pytest.mark.gpu
def test_reference_timed_run_and_writers(kmf_gpu, tmp_path):
    kmf = kmf_gpu
    cloud = kmf.geometry.generate_naca_cloud(80, 30, 1.15, 20.0)
    cfg = kmf.solver.SolverConfig(mach=0.63, aoa_deg=2.0, n_outer=12)
    rep = kmf.bench.timed_run(cfg, cloud, warmup=2)
    assert isinstance(rep, kmf.bench.BenchmarkReport)
    assert rep.points == cloud.n_points and rep.iterations == 10
    assert 0.0 < rep.rdp < 1e-6  # the reference's numpy path: ~1e-4 s here
    assert set(rep.stage_shares) == set(STAGE_NAMES)
    assert rep.stage_shares["q_derivatives"] > 0 and rep.stage_shares["flux_residual"] > 0
    assert 0.0 < sum(rep.stage_shares.values()) <= 1.0 + 1e-9
    kmf.bench.write_reports_json(tmp_path / "reports.json", [rep])
    back = json.loads((tmp_path / "reports.json").read_text())
    assert back[0]["points"] == cloud.n_points and back[0]["config"]["mach"] == 0.63


@pytest.mark.gpu
def test_reference_sweep_over_modes(kmf_gpu):
    kmf = kmf_gpu
    cloud = kmf.geometry.generate_naca_cloud(80, 30, 1.15, 20.0)
    res = kmf.bench.sweep(kmf.solver.SolverConfig(mach=0.63, aoa_deg=2.0, n_outer=6), cloud, "mode",
                          ["fused", "split4"], warmup=1)
    assert not res.any_failed, [c.error for c in res.cells]
    assert [r["level"] for r in res.rows] == ["fused", "split4"] and float(res.rows[0]["speedup"]) == 1.0


@pytest.mark.gpu
def test_reference_cli_solve_and_bench(kmf_gpu, tmp_path):
    """`kmf generate` + `kmf solve` + `kmf bench` of the reference CLI, on the
    B200: the history it writes is this package's solve, bit for bit."""
    kmf = kmf_gpu
    grid = tmp_path / "grid.dat"
    assert kmf.cli.main(["generate", "--chord-points", "80", "--layers", "30", "--out", str(grid)]) == 0
    out = tmp_path / "run"
    assert kmf.cli.main(["solve", "--grid", str(grid), "--out", str(out), "--mach", "0.63", "--aoa", "2",
                         "--iters", "5"]) == 0
    with open(out / "history.csv") as fh:
        hist = np.array([float(r["residue"]) for r in csv.DictReader(fh)])
    cloud = kmf.geometry.read_point_cloud(str(grid))
    ref = solve(SolverConfig(mach=0.63, aoa_deg=2.0, n_outer=5), cloud, build_stencils(cloud), instrument=False)
    assert np.array_equal(hist, ref.residue_history)
    for name in ("solution.csv", "wall.csv", "config.txt"):
        assert (out / name).exists()
    bench_out = tmp_path / "bench"
    assert kmf.cli.main(["bench", "--grid", str(grid), "--out", str(bench_out), "--iters", "6", "--warmup", "2",
                         "--modes", "fused,split4"]) == 0
    reports = json.loads((bench_out / "reports.json").read_text())
    assert len(reports) == 2 and all(r["iterations"] == 4 for r in reports)
