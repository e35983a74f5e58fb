"""bench.py contract checks that need no GPU: the reference arm (the fp64 oracle on the
host cores) prints one JSON line with the contract's keys, and our arm fails
loudly (non-zero exit) instead of falling back to the CPU when no CUDA device is present."""
import json
import os
import subprocess
import sys

import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run(args, timeout=300):
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT,
                          capture_output=True, text=True, timeout=timeout)


def test_reference_arm_prints_contract_line():
    r = run(["--impl", "reference", "--steps", "1", "--warmup", "0", "--workload", "C1"])
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
                "cpu_baseline", "e2e", "gpu_launches"):
        assert key in line, key
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["d2h_bytes_per_step"] == 0
    assert line["cpu_baseline"]["kind"] == "oracle" and line["cpu_baseline"]["cores"] >= 1
    assert line["config"]["workload"] == "C1"


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU failure path")
def test_our_arm_fails_loudly_without_a_gpu():
    r = run(["--steps", "1", "--warmup", "0", "--no-extra", "--no-cpu-baseline",
             "--e2e-steps", "0"])
    assert r.returncode != 0
    assert '"value"' not in r.stdout


def test_gpus_n_starts_n_ranks_itself():
    """`bench.py --gpus 2` with no launcher environment starts the 2 ranks itself (the
    driver's torchrun form); the reference arm's line comes from rank 0 of a world of 2."""
    env = {k: v for k, v in os.environ.items()
           if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--impl",
                        "reference", "--steps", "1", "--warmup", "0", "--workload", "C1"],
                       cwd=ROOT, capture_output=True, text=True, timeout=300, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.strip().splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout  # rank 0 alone prints
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["world_size"] == 2 and line["impl"] == "reference"


def test_mismatched_world_is_rejected():
    """A launcher world that differs from --gpus exits non-zero instead of reporting a
    number for the wrong GPU count."""
    env = {**os.environ, "WORLD_SIZE": "3", "RANK": "0", "LOCAL_RANK": "0"}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--impl",
                        "reference", "--steps", "1", "--warmup", "0", "--workload", "C1"],
                       cwd=ROOT, capture_output=True, text=True, timeout=300, env=env)
    assert r.returncode != 0
    assert "WORLD_SIZE=3" in r.stderr
    assert '"value"' not in r.stdout
    env1 = {**os.environ, "WORLD_SIZE": "1", "RANK": "0", "LOCAL_RANK": "0"}
    r1 = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "4", "--impl",
                         "reference", "--steps", "1", "--warmup", "0", "--workload", "C1"],
                        cwd=ROOT, capture_output=True, text=True, timeout=300, env=env1)
    assert r1.returncode != 0 and '"value"' not in r1.stdout
