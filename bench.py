#!/usr/bin/env python
"""bench.py -- BSS-MPPI optimisation-step throughput on B200.

Metric (BASELINE.json): belief rollout-steps/s (K*M*T per second), plus the
MPPI iteration latency (ms_per_step) and the FP32-roofline fraction of the
fused rollout kernel.  Workload: BASELINE config 3 (the throughput config
the north-star target is stated on): K=16384 control samples x M=256
disturbance realisations, T=50, dt=0.04, seeded random closed spline track
(half-width 2 m), Gaussian process noise std 0.05 on (vx, vy, r), control
noise std (0.2, 0.5).  Synthetic: the reference has no dataset; the track
and initial state are seeded.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1 runs under torchrun (one rank per GPU, NCCL): K is sharded across
ranks (weak in the number of GPUs per rollout, strong in total K: the
global workload is fixed), one all-reduce per iteration.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

# algorithmic work of one particle-step, counted from the
# reference formulation (FMA = 2 FLOP, add/sub/mul/div = 1; transcendental
# evaluations counted separately; per-(k,t) shared work excluded).
# (block, reference lines, FP32 FLOP, transcendentals)
WORK_TABLE = (
    ("re-projection x = mu + L z (lower-triangular 4x4)", "belief.py:264-272", 20, 0),
    ("process noise (diagonal F: 3 mul) + add to 3 channels", "belief.py:369, dynamics.py:571-572", 6, 0),
    ("tires: 2 atan2, 4 atan, 4 sin, 2 sqrt", "dynamics.py:375-395", 31, 12),
    ("derivatives + curvature: 2 tanh, sin + cos(e_psi)", "dynamics.py:409-437, 341-369", 49, 4),
    ("Euler update + angle / arc-length wraps", "dynamics.py:479-489", 24, 0),
    ("moments: mean 8 adds, cov 4 sub + 10 FMA", "belief.py:283-308", 32, 0),
)
FLOP_PER_PARTICLE_STEP = sum(r[2] for r in WORK_TABLE)   # 162
SFU_PER_PARTICLE_STEP = sum(r[3] for r in WORK_TABLE)    # 16
METRIC = "belief rollout-steps/s (K*M*T/s)"
UNIT = "rollout-steps/s"

WORKLOADS = {
    "C3": dict(K=16384, M=256, T=50, dt=0.04, track="spline0", noise_std=0.05),
    "C1": dict(K=256, M=32, T=20, dt=0.05, track="ellipse", noise_std=0.03),
    "C2": dict(K=4096, M=128, T=40, dt=0.05, track="ellipse", noise_std=0.05),
    "C5_4096x512": dict(K=4096, M=512, T=60, dt=0.04, track="spline0", noise_std=0.05),
    "C5_32768x64": dict(K=32768, M=64, T=60, dt=0.04, track="spline0", noise_std=0.05),
    "C5_131072x256": dict(K=131072, M=256, T=60, dt=0.04, track="spline0", noise_std=0.05),
    # config 4: extension beyond the reference (obstacles.py): Laplace(0.03) + U(+-0.05) slip,
    # shield beta = 0.2, 16 seeded obstacles with delta = 0.02 chance constraints
    "C4": dict(K=65536, M=64, T=50, dt=0.04, track="spline0", noise_std=None, laplace=(0.03, 0.05),
               cbf_rate=0.2, obstacles=16),
}


def build_problem_objects(wl):
    """(cfg, cost, model, track, noise, x0, obstacles) of a workload."""
    from paper_2408_00494_b200 import controllers as mc
    from paper_2408_00494_b200 import dynamics as md
    from paper_2408_00494_b200.constraints import SafetyParams
    from paper_2408_00494_b200.tracks import named_track

    track = named_track(wl["track"])
    model = md.with_timestep(md.VehicleParams(), wl["dt"], "euler")
    cfg = mc.MppiConfig(kind="bss", samples=wl["K"], horizon=wl["T"], inner_samples=wl["M"],
                        sigma_eps=np.diag([0.2 ** 2, 0.5 ** 2]))
    obstacles = None
    if wl.get("laplace"):
        from paper_2408_00494_b200.obstacles import LaplaceSlipNoise, place_obstacles
        noise = LaplaceSlipNoise(*wl["laplace"])
        obstacles = place_obstacles(track, wl["obstacles"], seed=0) if wl.get("obstacles") else None
    else:
        noise = md.NoiseModel(np.diag([wl["noise_std"] ** 2] * 3))
    cost = mc.CostSpec(safety=SafetyParams(wl.get("cbf_rate", 0.35), 2000.0))
    s0 = float(np.random.default_rng(0).uniform(0.0, track.length))
    x0 = md.VehicleState.rolling(5.0, model, s=s0).as_array()
    return cfg, cost, model, track, noise, x0, obstacles


# ----------------------------------------------------------------- clocks

class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 100 ms."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.path = None

    def start(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-i", str(self.device), "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        rows = [r.split(", ") for r in Path(self.path).read_text().splitlines() if r.strip()]
        os.unlink(self.path)
        sm = [float(r[1]) for r in rows if len(r) >= 9 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if len(r) >= 9 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows if len(r) >= 9 for i in range(4)
                          if r[5 + i].strip().lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "samples": len(rows), "reasons": reasons}


# ----------------------------------------------------------------- CPU arm

def cpu_rate(wl, seconds, threads=0, key=(1, 2)):
    """C oracle (FP64, all host threads, Philox noise) on a K-slice of the
    workload sized to ~``seconds``; returns (particle-steps/s, threads, sample)."""
    from oracle import c_oracle
    from paper_2408_00494_b200.controllers import RolloutContext, build_problem

    cfg, cost, model, track, noise, x0, obstacles = build_problem_objects(wl)
    ctx = RolloutContext(model, track, cost, noise=noise, obstacles=obstacles)
    nthr = threads or c_oracle.max_threads()
    plan = np.zeros((wl["T"], 2))

    def run(k):
        prob, keep = build_problem("bss", k, wl["T"], wl["M"], cfg.temperature, cfg.control_cost_weight,
                                   cfg.sigma_eps, cfg.precision, cfg.bounds, False, ctx)
        t0 = time.perf_counter()
        c_oracle.control_step(prob, x0, None, plan, key, (3, 4), threads=nthr)
        return time.perf_counter() - t0

    k = max(4 * nthr, 64)
    run(k)                                   # warm (thread pool, page faults)
    dt = run(k)
    k = int(min(wl["K"], max(nthr, k * seconds / max(dt, 1e-3))))
    reps, total = 0, 0.0
    while total < 0.8 * seconds or reps == 0:
        total += run(k)
        reps += 1
    ps = k * wl["M"] * wl["T"] * reps
    return ps / total, nthr, (f"{reps} x K-slice {k} of {wl['K']} (x M={wl['M']} x T={wl['T']}), "
                              f"{total:.1f} s")


def reference_arm(args, wl):
    """--impl reference: the UNMODIFIED reference package (belief_mppi 0.1.0,
    numba, installed in baseline/_ref) through its own Controller.control_step,
    K-sharded over one process per host core (baseline/reference_arm.py), on
    the same workload, metric and config.  Each step is a bounded K-slice of
    the iteration (``--ref-step-seconds`` per process); ``ms_per_step`` is the
    measured wall time of that sampled step.  Without the install it falls
    back to the FP64 C port of the same algorithm (oracle/, kind "port")."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from baseline import reference_arm as ra

    why = ra.available()
    if wl.get("laplace"):
        why = "config-4 Laplace/obstacle extension: the reference has no such path"
    if why is not None:
        return reference_arm_port(args, wl, why)
    pool = ra.ReferencePool(wl, step_seconds=args.ref_step_seconds)
    try:
        times = []
        for i in range(args.warmup + args.steps):
            dt = pool.step()
            if i >= args.warmup:
                times.append(dt)
    finally:
        pool.close()
    total = sum(times)
    per_step = pool.rollouts_per_step * wl["M"] * wl["T"]
    value = per_step * len(times) / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / len(times),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded spline track, seeded x0, the reference's numpy keyed noise)",
        "config": workload_config(args, wl),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": pool.procs, "kind": "reference",
                         "sample": pool.sample()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "note": (f"ms_per_step is the wall time of one sampled step ({pool.rollouts_per_step} of "
                 f"K={wl['K']} rollouts); a full-K iteration at this rate would take "
                 f"{1e3 * wl['K'] * wl['M'] * wl['T'] / value:.0f} ms"),
    }
    print(json.dumps(line))
    return 0


def reference_arm_port(args, wl, why):
    """Fallback reference arm: the FP64 C port (oracle/) on all host threads,
    full K per step (no extrapolation)."""
    from oracle import c_oracle
    from paper_2408_00494_b200.controllers import RolloutContext, build_problem

    cfg, cost, model, track, noise, x0, obstacles = build_problem_objects(wl)
    ctx = RolloutContext(model, track, cost, noise=noise, obstacles=obstacles)
    nthr = c_oracle.max_threads()
    prob, keep = build_problem("bss", wl["K"], wl["T"], wl["M"], cfg.temperature, cfg.control_cost_weight,
                               cfg.sigma_eps, cfg.precision, cfg.bounds, False, ctx)
    plan = np.zeros((wl["T"], 2))
    times = []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        vplus, _ = c_oracle.control_step(prob, x0, None, plan, (11, i), (12, i), threads=nthr)
        dt = time.perf_counter() - t0
        plan = np.concatenate([vplus[1:], vplus[-1:]])
        if i >= args.warmup:
            times.append(dt)
    total = sum(times)
    value = wl["K"] * wl["M"] * wl["T"] * len(times) / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / len(times),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded spline track, seeded x0, Philox noise)",
        "config": workload_config(args, wl),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": nthr, "kind": "port",
                         "sample": f"full K={wl['K']} per step; FP64 C port (oracle/): {why}"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


def workload_config(args, wl):
    extra = {}
    if wl.get("laplace"):
        extra = {"noise": f"Laplace({wl['laplace'][0]}) + U(+-{wl['laplace'][1]}) slip on vy",
                 "cbf_rate": wl["cbf_rate"], "obstacles": wl["obstacles"],
                 "extension": "beyond the reference (obstacles.py); parity vs extended C oracle"}
    return {"workload": f"{args.workload}: BSS-MPPI iteration K={wl['K']} x M={wl['M']} x "
                        f"T={wl['T']}, dt={wl['dt']}, track={wl['track']}",
            "K": wl["K"], "M": wl["M"], "T": wl["T"], "dt": wl["dt"], "track": wl["track"],
            "process_noise_std": wl["noise_std"], "control_noise_std": [0.2, 0.5], **extra,
            "global_batch": wl["K"], "seq_len": wl["T"], "parallelism": f"k-shard{args.gpus}",
            "l2": "flushed (256 MiB memset) between timed iterations"}


# ----------------------------------------------------------------- GPU arm

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="C3",
                    help="one of %s, or C5:K:M for the BASELINE config-5 sweep (T=60)" % sorted(WORKLOADS))
    ap.add_argument("--e2e-steps", type=int, default=50)
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--ref-step-seconds", type=float, default=0.5,
                    help="reference arm: wall seconds of one sampled K-sharded step")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.workload.startswith("C5:"):
        _, k, m = args.workload.split(":")
        wl = dict(K=int(k), M=int(m), T=60, dt=0.04, track="spline0", noise_std=0.05)
    else:
        wl = WORKLOADS[args.workload]
    if args.impl == "reference":
        return reference_arm(args, wl)

    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    # one rank per GPU; BSSMPPI_DIST_BACKEND=gloo lets the N>1 mechanics run
    # on a single GPU for testing (host-staged all-reduce, no waiting kernels)
    backend = os.environ.get("BSSMPPI_DIST_BACKEND", "nccl")
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
        else:
            dist.init_process_group(backend)

    from paper_2408_00494_b200 import _lib, streams
    from paper_2408_00494_b200 import controllers as mc

    cfg, cost, model, track, noise, x0, obstacles = build_problem_objects(wl)
    stream = torch.cuda.current_stream()
    if world > 1:
        from paper_2408_00494_b200.distributed import ShardedController
        ctrl = ShardedController(cfg, cost, model, track, noise=noise, seed=0, run_path=(5, 0),
                                 device=local, obstacles=obstacles)
    else:
        ctrl = mc.Controller(cfg, cost, model, track, noise=noise, seed=0, run_path=(5, 0),
                             device=local, stream=stream.cuda_stream, obstacles=obstacles)
    k_begin, k_count = ctrl._k_range()

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(v):
        if dist is None:
            return v
        t = torch.tensor([v], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- e2e through the public API: host x0/plan in, host v+ out ----
    for _ in range(args.warmup):
        ctrl.control_step(x0)
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n_e2e = max(1, min(args.e2e_steps, args.steps))
    e0.record(stream)
    t_wall = time.perf_counter()
    for _ in range(n_e2e):
        ctrl.control_step(x0)
    e1.record(stream)
    barrier()
    wall_e2e = (time.perf_counter() - t_wall) / n_e2e
    e2e_ms = max_over_ranks(e0.elapsed_time(e1) / n_e2e)

    # ---- device-resident throughput ----
    ctrl.upload_state(x0)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
    keys = [(streams.device_key(0, 5, 0, 2, 1000 + i), streams.device_key(0, 5, 0, 3, 1000 + i))
            for i in range(args.warmup + args.steps)]
    for i in range(args.warmup):
        ctrl.enqueue_iteration(*keys[i])
    ctrl.download()
    barrier()
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    step_ms, roll_ms = [], []
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    for i in range(args.steps):
        flush.zero_()
        ev[i][0].record(stream)
        ctrl.enqueue_iteration(*keys[args.warmup + i])
        ev[i][1].record(stream)
        _, d = ctrl.download()
        roll_ms.append(d["rollout_ms"])
    barrier()
    clock_info = clocks.stop()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    total_ms = max_over_ranks(sum(step_ms))
    ms_per_step = total_ms / args.steps
    KMT = wl["K"] * wl["M"] * wl["T"]
    value = KMT * args.steps / (total_ms * 1e-3)

    # ---- roofline of the dominant kernel (fused rollout) ----
    roll_avg = statistics.mean(roll_ms)
    flop = FLOP_PER_PARTICLE_STEP * k_count * wl["M"] * wl["T"]
    achieved = flop / (roll_avg * 1e-3) / 1e12
    peak = ctypes_ffma_peak(_lib, local)
    nominal = 148 * 128 * 2 * 1965e6 / 1e12
    try:
        mp = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
        nominal = 148 * 128 * 2 * float(mp.get("sm_max_mhz", 1965.0)) * 1e6 / 1e12
    except Exception:
        pass
    traffic = None
    tpath = ROOT / "profiles" / "rollout_traffic.json"
    if tpath.exists():
        tj = json.loads(tpath.read_text())
        traffic = tj.get(args.workload)
    G, block = ctrl.launch_shape()
    pipe = None
    ppath = ROOT / "profiles" / "rollout_pipes.json"
    if ppath.exists():
        pipe = json.loads(ppath.read_text()).get(args.workload)
    sfu_ops = SFU_PER_PARTICLE_STEP * k_count * wl["M"] * wl["T"]
    sfu_achieved = sfu_ops / (roll_avg * 1e-3) / 1e12
    sfu_peak = ctypes_mufu_peak(_lib, local)
    # north_star's roofline is the FP32 one: 162 algorithmic FLOP per
    # particle-step / the rollout kernel's CUDA-event time vs the
    # FFMA peak; the kernel is FMA-pipe bound (ncu evidence in fma_pipe)
    roofline = {
        "bound": "fp32", "kernel": f"bss_rollout_kernel<{G},false,false,{block}>",
        "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak if peak else None,
        "traffic": traffic,
        "peak_source": "FFMA microbenchmark measured in this run (MEASURED_PEAKS.json has no FP32 "
                       "figure); nominal 148 SM x 128 FMA x 2 x sm_max_mhz = "
                       f"{nominal:.1f} TFLOP/s",
        "frac_of_nominal": achieved / nominal,
        "algorithmic_flop_per_launch": flop, "flop_per_particle_step": FLOP_PER_PARTICLE_STEP,
        "particle_steps_per_launch": k_count * wl["M"] * wl["T"],
        "rollout_ms": roll_avg, "rollout_share_of_step": roll_avg / statistics.mean(step_ms),
        "fma_pipe": pipe,
        "sfu_transcendentals": {
            "what": "algorithmic transcendentals / MUFU peak -- not a bound: the atan, tire-sine and "
                    "heading sin/cos evaluations run as FMA-pipe polynomials, the MUFU work is mostly "
                    "Box-Muller",
            "achieved": sfu_achieved, "peak": sfu_peak, "unit": "Tops/s",
            "frac": sfu_achieved / sfu_peak if sfu_peak else None,
            "ops_per_particle_step": SFU_PER_PARTICLE_STEP},
    }

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32 (FP64 weighted update)",
        "data": "synthetic (seeded spline track, seeded x0, in-kernel Philox4x32 noise)",
        "config": workload_config(args, wl),
        "e2e": {"value": KMT / (e2e_ms * 1e-3), "unit": UNIT, "ms_per_step": e2e_ms,
                "wall_ms_per_step": wall_e2e * 1e3,
                "h2d_bytes_per_step": (24 + 2 * wl["T"]) * 4,
                "d2h_bytes_per_step": (2 * wl["T"] + 5) * 8,
                "path": "Controller.control_step (host numpy state/plan -> C ABI -> host v+)"},
        "roofline": roofline,
        "clocks": clock_info,
        # rollout + update partials + combine; a single-context K <= 1024
        # iteration runs the one-launch update (csrc/update.cuh kSmallK)
        "gpu_launches": (2 if world == 1 and k_count <= 1024 else 3) * args.steps,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        from baseline import reference_arm as ra
        if ra.available() is None and not wl.get("laplace"):
            rate, cores, sample = ra.rate(wl, args.cpu_seconds)
            line["cpu_baseline"] = {"value": rate, "unit": UNIT, "cores": cores, "kind": "reference",
                                    "sample": sample}
        rate, cores, sample = cpu_rate(wl, args.cpu_seconds / 3)
        port = {"value": rate, "unit": UNIT, "cores": cores, "kind": "port",
                "sample": sample + "; FP64 C port of the reference step (oracle/, OpenMP)"}
        line.setdefault("cpu_baseline", port)
        if line["cpu_baseline"] is not port:
            line["cpu_port"] = port
    if rank == 0:
        print(json.dumps(line))
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def ctypes_mufu_peak(_lib, device):
    out = _lib.C.c_double(0.0)
    _lib.check(_lib.load().bssmppi_mufu_peak(device, _lib.C.byref(out)))
    return out.value


def ctypes_ffma_peak(_lib, device):
    out = _lib.C.c_double(0.0)
    _lib.check(_lib.load().bssmppi_ffma_peak(device, _lib.C.byref(out)))
    return out.value


if __name__ == "__main__":
    sys.exit(main())
