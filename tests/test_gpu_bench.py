"""bench.py keeps the driver contract (one JSON line with the required keys)
on a small configuration, for both arms."""

import json
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

REQUIRED = ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
            "vs_baseline", "dtype", "data", "config", "e2e", "gpu_launches", "roofline", "roofline_fp64",
            "cpu_baseline", "clocks")


def run(*args):
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], capture_output=True, text=True,
                         timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_bench_ours_contract(gpu):
    d = run("--config", "c1", "--steps", "3", "--warmup", "3")
    for k in REQUIRED:
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3 and d["value"] > 0
    assert d["config"]["n_points"] == 40000 and "workload" in d["config"]
    assert d["e2e"]["h2d_bytes_per_step"] == 4 * 40000 * 8 and d["e2e"]["value"] > 0
    # per step: 4 stages x (first order + 3 sweeps + flux + boundary + update)
    # = 28 in second order; c1 is BASELINE's first-order config: 4 x 3 = 12
    assert d["config"]["order"] == 1 and d["gpu_launches"] == 3 * 12
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in d["roofline"]
    assert 0 < d["roofline"]["frac"] < 1
    cb = d["cpu_baseline"]
    assert cb["kind"] == "port" and cb["cores"] >= 1 and cb["value"] > 0 and cb["sample"]


def test_bench_reference_arm_contract(gpu):
    d = run("--impl", "reference", "--config", "c1", "--steps", "1", "--warmup", "0")
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "point-iterations/s"
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert d["cpu_baseline"]["value"] == d["value"]
