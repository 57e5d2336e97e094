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


@pytest.mark.parametrize("arm", ["reference", "port"])
def test_reference_arm_json_line(arm):
    """The stock reference package from baseline/_ref (numba, K-sharded over
    host processes) when installed, else / on request the FP64 C port."""
    sys.path.insert(0, str(ROOT))
    from baseline import reference_arm as ra
    if arm == "reference" and ra.available() is not None:
        pytest.skip(ra.available())
    r = _bench("--impl", "reference", "--workload", "C1", "--steps", "2", "--warmup", "1",
               "--ref-step-seconds", "0.05", env={"BSSMPPI_REFERENCE_ARM": arm})
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference"
    assert line["metric"].startswith("belief rollout-steps/s") and line["unit"] == "rollout-steps/s"
    assert line["value"] > 0 and line["higher_is_better"] is True and line["steps"] == 2
    assert line["config"]["workload"].startswith("C1")
    assert line["ms_per_step"] > 0
    cb = line["cpu_baseline"]
    assert cb["kind"] == arm and cb["cores"] >= 1 and cb["value"] == line["value"] and cb["sample"]
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


def test_algorithmic_work_table():
    """SURVEY.md 8d's per-particle-step work, pinned row by row: the
    roofline's `achieved` numbers are these counts x K M T / kernel time."""
    sys.path.insert(0, str(ROOT))
    import bench
    rows = {r[0].split(":")[0].split(" (")[0]: (r[2], r[3]) for r in bench.WORK_TABLE}
    assert bench.FLOP_PER_PARTICLE_STEP == 162 and bench.SFU_PER_PARTICLE_STEP == 16
    # rows that follow from the algebra alone
    assert rows["re-projection x = mu + L z"] == (2 * 10, 0)            # 10 multiply-adds of L (4x4 lower)
    assert rows["process noise"] == (3 + 3, 0)                           # 3 mul + 3 add
    assert rows["moments"] == (8 + 4 + 2 * 10, 0)                       # 8 adds, 4 sub, 10 FMA
    assert rows["tires"][1] == 2 + 4 + 4 + 2                             # atan2, atan, sin, sqrt
    assert rows["derivatives + curvature"][1] == 2 + 2                  # tanh x2, sin + cos
    assert all(r[1] for r in bench.WORK_TABLE)                           # every row cites the reference
