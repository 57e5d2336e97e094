"""Reference arm of bench.py: the UNMODIFIED reference package.

``belief_mppi`` 0.1.0 (arxiv 2408.00494's package, numba, FP64) is installed
once, offline, into ``baseline/_ref`` (git-ignored, shipped to the GPU box
with the working tree):

    python -m pip install --no-index --no-build-isolation --find-links /opt/wheelhouse \\
        --target baseline/_ref <copy of /root/reference/pkg> --no-deps

This module drives it through its own public API -- ``Controller(config,
cost, model, track, noise, seed, run_path).control_step(state)``
(controllers.py:343-410) with ``kind="bss"`` -- on the bench workload's
objects built by the reference's own constructors (``make_test_track``,
``VehicleParams``, ``NoiseModel``, ``MppiConfig``, ``CostSpec``).  Nothing of
this repo's kernels or host code is on that path.

The reference controller is serial (numba, no ``prange``); its own
parallelism is process-level (``sim.monte_carlo`` maps runs over a
``ProcessPoolExecutor``, sim.py:317-325).  The arm therefore K-shards one
iteration over P worker processes (one per host core): worker p owns a
``Controller`` on a K-slice with its own ``run_path``, and one bench step is
one ``control_step`` in every worker, timed by wall clock around the map.
"""

from __future__ import annotations

import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
REF = ROOT / "baseline" / "_ref"

_CTRL = None
_X0 = None


def available() -> str | None:
    """None if the installed reference imports, else the reason
    (BSSMPPI_REFERENCE_ARM=port forces bench.py's C-port fallback)."""
    if os.environ.get("BSSMPPI_REFERENCE_ARM") == "port":
        return "BSSMPPI_REFERENCE_ARM=port"
    if not (REF / "belief_mppi").is_dir():
        return f"{REF} not installed (see baseline/reference_arm.py)"
    try:
        _import()
    except Exception as e:   # numba / scipy missing, broken install
        return f"reference import failed: {e!r}"
    return None


def _import():
    for var in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS", "NUMBA_NUM_THREADS"):
        os.environ.setdefault(var, "1")
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/bssmppi_numba_cache")
    if str(REF) not in sys.path:
        sys.path.insert(0, str(REF))
    sys.path.insert(0, str(ROOT))
    import belief_mppi  # noqa: F401
    from belief_mppi import controllers, dynamics
    return controllers, dynamics


def build_controller(wl: dict, k_slice: int, index: int):
    """A reference ``Controller`` for ``k_slice`` rollouts of workload ``wl``
    (BASELINE config shapes; spline / ellipse tables from this repo's track
    generator fed through the reference's ``make_test_track``)."""
    rc, rd = _import()
    from paper_2408_00494_b200.tracks import named_track

    track = named_track(wl["track"], build=rd.make_test_track)
    model = rd.with_timestep(rd.VehicleParams(), wl["dt"], "euler")
    cfg = rc.MppiConfig(kind="bss", samples=int(k_slice), horizon=wl["T"], inner_samples=wl["M"],
                        sigma_eps=np.diag([0.2 ** 2, 0.5 ** 2]))
    noise = rd.NoiseModel(np.diag([wl["noise_std"] ** 2] * 3))
    s0 = float(np.random.default_rng(0).uniform(0.0, track.length))
    x0 = rd.VehicleState.rolling(5.0, model, s=s0).as_array()
    ctrl = rc.Controller(cfg, rc.CostSpec(), model, track, noise=noise, seed=0, run_path=(5, 0, index))
    return ctrl, x0


def _init(wl, k_slice, counter):
    global _CTRL, _X0
    with counter.get_lock():
        index = counter.value
        counter.value += 1
    _CTRL, _X0 = build_controller(wl, k_slice, index)
    _CTRL.control_step(_X0)                 # JIT (from the warm numba cache) + first iteration


def _step(_):
    t0 = time.perf_counter()
    _CTRL.control_step(_X0)
    return time.perf_counter() - t0


class ReferencePool:
    """P worker processes, each holding a reference Controller on a K-slice."""

    def __init__(self, wl: dict, step_seconds: float = 1.0, procs: int = 0):
        import multiprocessing as mp

        self.wl = wl
        self.procs = procs or os.cpu_count() or 1
        # compile once in this process (numba cache=True writes NUMBA_CACHE_DIR;
        # the workers load it) and calibrate the per-rollout cost
        ctrl, x0 = build_controller(wl, 4, 0)
        ctrl.control_step(x0)
        t0 = time.perf_counter()
        ctrl.control_step(x0)
        per_rollout = (time.perf_counter() - t0) / 4
        self.k_slice = int(max(1, min(-(-wl["K"] // self.procs), round(step_seconds / per_rollout))))
        ctx = mp.get_context("spawn")        # no CUDA / numba state inherited
        counter = ctx.Value("i", 0)
        self.pool = ctx.Pool(self.procs, initializer=_init, initargs=(wl, self.k_slice, counter))

    @property
    def rollouts_per_step(self) -> int:
        return self.k_slice * self.procs

    def step(self) -> float:
        """One K-sharded iteration (every worker one control_step); wall s."""
        t0 = time.perf_counter()
        self.pool.map(_step, range(self.procs), chunksize=1)
        return time.perf_counter() - t0

    def close(self):
        self.pool.close()
        self.pool.join()

    def sample(self) -> str:
        return (f"{self.procs} processes x K-slice {self.k_slice} (= {self.rollouts_per_step} of "
                f"K={self.wl['K']}) x M={self.wl['M']} x T={self.wl['T']} per step; "
                "stock belief_mppi 0.1.0 (numba, FP64) Controller.control_step kind='bss' "
                "from baseline/_ref, K-sharded like sim.monte_carlo's process pool")


def rate(wl: dict, seconds: float, procs: int = 0):
    """(rollout-steps/s, processes, sample) of the reference on ~``seconds``
    of K-sharded iterations (bench.py cpu_baseline)."""
    pool = ReferencePool(wl, step_seconds=min(1.0, seconds / 4), procs=procs)
    try:
        pool.step()                           # workers warm
        total, reps = 0.0, 0
        while total < seconds or reps == 0:
            total += pool.step()
            reps += 1
        ps = pool.rollouts_per_step * wl["M"] * wl["T"] * reps
        return ps / total, pool.procs, f"{reps} steps of " + pool.sample() + f", {total:.1f} s"
    finally:
        pool.close()
