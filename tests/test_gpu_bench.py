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
    # = 28 in the reference's second-order scheme (c1)
    assert d["config"]["order"] == 2 and d["gpu_launches"] == 3 * 28
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in d["roofline"]
    assert 0 < d["roofline"]["frac"] < 1
    rq = d["roofline_qgrad"]
    for kern in ("first_order", "sweep"):
        assert 0 < rq[kern]["frac"] < 1.5 and rq[kern]["launch_us"] > 0
    assert "algorithmic_achieved" not in d["roofline_fp64"]
    cb = d["cpu_baseline"]
    assert cb["kind"] in ("reference", "port") and cb["cores"] >= 1 and cb["value"] > 0 and cb["sample"]
    if cb["kind"] == "reference":  # the reference package itself (baseline/_ref), the C port beside it
        assert "kmf" in cb["sample"] and d["cpu_baseline_port"]["kind"] == "port"


def test_bench_first_order_config(gpu):
    """c1o1: BASELINE configs[0]'s first-order scheme, labelled as such:
    4 stages x (flux + boundary + update) = 12 launches per step."""
    d = run("--config", "c1o1", "--steps", "3", "--warmup", "3", "--no-cpu-baseline")
    assert d["config"]["order"] == 1 and d["gpu_launches"] == 3 * 12 and d["roofline_qgrad"] is None
    assert "first order" in d["config"]["workload"]



@pytest.mark.parametrize("transport", ["peer", "nccl"])
def test_bench_two_ranks(gpu, transport):
    """--gpus 2 self-launches two ranks (torchrun); with one visible GPU the
    ranks share it (KMF_SHARE_GPU: IPC on one device / NCCL over sockets).
    Before timing, the partitioned residues must equal a single-GPU solve
    bit for bit; the line carries the transport and that check."""
    import os

    env = dict(os.environ, KMF_SHARE_GPU="1")
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--config", "c1", "--steps", "2",
                          "--warmup", "3", "--no-cpu-baseline", "--transport", transport],
                         capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["e2e"]["value"] > 0
    t = d["transport"]
    assert t["name"] == transport and t["fallback"] is None and t["check"]["bitwise_vs_single_gpu"]
    assert d["partition"]["scheme"] == "sectors" and len(d["partition"]["ranks"]) == 2
    assert d.get("shared_gpu") is True


def test_bench_peer_fallback_to_nccl(gpu):
    """A peer transport that fails its pre-timing check (here every peer
    wait gets a 1 ns deadline, so the first wait fails with KMF_EPEER) is
    replaced by NCCL on every rank, and the line records why."""
    import os

    env = dict(os.environ, KMF_SHARE_GPU="1", KMF_PEER_TIMEOUT_S="1e-9")
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--config", "c1", "--steps", "2",
                          "--warmup", "3", "--no-cpu-baseline", "--transport", "peer"],
                         capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    d = json.loads([l for l in out.stdout.splitlines() if l.startswith("{")][0])
    t = d["transport"]
    assert t["name"] == "nccl" and t["fallback"]["from"] == "peer" and t["check"]["bitwise_vs_single_gpu"]
    assert any(w and "did not arrive" in w for w in t["fallback"]["why"]), t
