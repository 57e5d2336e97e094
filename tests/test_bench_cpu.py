"""bench.py contract pieces that run without a GPU: the reference arm (the
FP64 C port of the reference step on host cores) prints one JSON line with
the contract's keys; under torchrun only rank 0 prints; the device arm
fails loudly instead of falling back to the CPU."""

import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


def _bench(*args, env=None):
    e = dict(os.environ)
    e.update(env or {})
    return subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], capture_output=True, text=True,
                          cwd=ROOT, env=e, timeout=600)


def test_reference_arm_json_line():
    r = _bench("--impl", "reference", "--workload", "C1", "--steps", "2", "--warmup", "1",
               "--ref-step-seconds", "0.05")
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference"
    assert line["metric"].startswith("belief rollout-steps/s") and line["unit"] == "rollout-steps/s"
    assert line["value"] > 0 and line["higher_is_better"] is True and line["steps"] == 2
    assert line["config"]["workload"].startswith("C1")
    cb = line["cpu_baseline"]
    assert cb["kind"] == "port" and cb["cores"] >= 1 and cb["value"] == line["value"] and cb["sample"]
    assert line["e2e"] == {"value": line["value"], "unit": line["unit"], "h2d_bytes_per_step": 0,
                           "d2h_bytes_per_step": 0}


def test_reference_arm_only_rank0_prints():
    r = _bench("--impl", "reference", "--workload", "C1", "--steps", "1", "--warmup", "0",
               env={"RANK": "1", "WORLD_SIZE": "2", "LOCAL_RANK": "1"})
    assert r.returncode == 0 and r.stdout.strip() == ""


def test_device_arm_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    r = _bench("--steps", "1", "--warmup", "3", "--no-cpu-baseline")
    assert r.returncode != 0
    assert r.stdout.strip() == ""          # no JSON line, no CPU fallback number
