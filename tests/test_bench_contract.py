"""bench.py's output contract, on CPU: the reference arm (the oracle port on
the host cores) prints one JSON line with the keys the driver reads, for the
points workload and for the tube workload; the GPU arm is covered by the
round-end bench run itself."""

import json
import os
import subprocess
import sys

import pytest

from conftest import REPO

BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
             "scaling", "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"}


def run_bench(*args, timeout=600):
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="")
    res = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), *args], capture_output=True,
                         text=True, timeout=timeout, cwd=REPO, env=env)
    assert res.returncode == 0, res.stderr[-2000:]
    lines = [ln for ln in res.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1, res.stdout
    return json.loads(lines[0])


def test_reference_arm_points_workload():
    out = run_bench("--impl", "reference", "--workload", "c1", "--steps", "1", "--warmup", "0",
                    "--cpu-seconds", "2")
    assert BASE_KEYS <= set(out)
    assert out["impl"] == "reference" and out["unit"] == "points/s" and out["higher_is_better"] is True
    assert out["value"] > 0 and out["e2e"]["value"] == out["value"]
    assert out["e2e"]["h2d_bytes_per_step"] == 0 and out["e2e"]["d2h_bytes_per_step"] == 0
    cb = out["cpu_baseline"]
    assert cb["kind"] == "port" and cb["cores"] >= 1 and cb["value"] == out["value"]
    assert out["config"]["workload"].startswith("c1")


@pytest.mark.timeout(900)
def test_reference_arm_tube_workload():
    out = run_bench("--impl", "reference", "--workload", "tube", "--steps", "1", "--warmup", "0")
    assert BASE_KEYS <= set(out)
    assert out["unit"] == "ms" and out["higher_is_better"] is False and out["value"] > 0
    assert out["config"]["workload"].startswith("tube")


def test_reference_arm_under_torchrun_prints_once():
    """N > 1 launch (torchrun, 2 ranks): rank 0 alone runs the reference arm
    and prints one line; the other rank exits 0 without work."""
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29561", os.path.join(REPO, "bench.py"),
           "--impl", "reference", "--gpus", "2", "--workload", "c1", "--steps", "1", "--warmup", "0",
           "--cpu-seconds", "2"]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=REPO, env=env)
    assert res.returncode == 0, res.stderr[-2000:]
    lines = [ln for ln in res.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1, res.stdout
    out = json.loads(lines[0])
    assert out["impl"] == "reference" and out["n_gpus"] == 2 and out["value"] > 0
