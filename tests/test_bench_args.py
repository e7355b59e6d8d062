"""bench.py's launch contract on the CPU: --gpus N under a launcher with
another world size fails loudly instead of silently measuring a different
GPU count (the GPU path itself is tests/test_gpu_bench.py)."""

import os
import subprocess
import sys

from conftest import ROOT


def test_bench_gpus_mismatch_fails():
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--config", "c1", "--steps", "1"],
                         capture_output=True, text=True, timeout=300, cwd=ROOT, env=env)
    assert out.returncode != 0 and "WORLD_SIZE" in out.stderr


def test_bench_self_launch_command(monkeypatch):
    """Outside torchrun, --gpus N re-launches under torch.distributed.run with
    N ranks on 127.0.0.1 and NCCL's INFO log on stderr."""
    sys.path.insert(0, str(ROOT))
    import bench

    seen = {}

    def fake_call(cmd, env):
        seen["cmd"], seen["env"] = cmd, env
        return 0

    monkeypatch.setattr(bench.subprocess, "call", fake_call)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4", "--steps", "2"])
    args = type("A", (), {"gpus": 4})()
    assert bench.self_launch(args) == 0
    cmd = seen["cmd"]
    assert cmd[1:3] == ["-m", "torch.distributed.run"] and "--nproc-per-node=4" in cmd
    assert cmd[cmd.index("--master-addr") + 1] == "127.0.0.1" and cmd[-4:] == ["--gpus", "4", "--steps", "2"]
    assert seen["env"]["NCCL_DEBUG"] == "INFO" and seen["env"]["NCCL_DEBUG_FILE"] == "/dev/stderr"
