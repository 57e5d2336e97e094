"""BASELINE config 2: 200-step closed loop on the ellipse, K=4096 x M=128,
T=40, dt=0.05, warm start, Gaussian process noise std ~ U[0.01, 0.1] per run
(seeded).  Runs the device controller (Philox) and, with --oracle, the same
loop driven by the FP64 C port of the reference step (same Philox keys, host
cores) as the oracle trajectory; reports per-step latency and the
constraint-violation rate (|e_y| > collision threshold) of both."""
import argparse, json, sys, time
sys.path.insert(0, ".")
import numpy as np
from paper_2408_00494_b200 import controllers as mc, dynamics as md, sim, streams
from paper_2408_00494_b200.tracks import named_track


class OracleController:
    """The C oracle as a closed-loop controller (test/measurement infra)."""

    def __init__(self, cfg, run_path):
        from oracle import c_oracle
        self.c = c_oracle
        self.cfg, self.seed, self.run_path = cfg, cfg.master_seed, tuple(run_path)
        ctx = mc.RolloutContext(cfg.model_params(), cfg.track, cfg.cost, noise=cfg.noise)
        m = cfg.controller
        self.prob, self._keep = mc.build_problem("bss", m.samples, m.horizon, m.inner_samples, m.temperature,
                                                 m.control_cost_weight, m.sigma_eps, m.precision, m.bounds,
                                                 False, ctx)
        self.plan = np.zeros((m.horizon, 2))
        self.iteration = 0
        self.last_diagnostics = {}

    def control_step(self, x):
        base = streams.base_key(self.seed, *self.run_path)
        kc = self.c.iteration_key(base, 2, self.iteration)
        kb = self.c.iteration_key(base, 3, self.iteration)
        t0 = time.perf_counter()
        vplus, _ = self.c.control_step(self.prob, x, None, self.plan, kc, kb)
        self.last_diagnostics = {"device_ms": 1e3 * (time.perf_counter() - t0)}
        self.plan = np.concatenate([vplus[1:], vplus[-1:]])
        self.iteration += 1
        return vplus[0].copy(), self.plan

    def close(self):
        pass


def config(seed, steps):
    std = float(np.random.default_rng(seed).uniform(0.01, 0.1))
    cfg = mc.MppiConfig(kind="bss", samples=4096, horizon=40, inner_samples=128,
                        sigma_eps=np.diag([0.2 ** 2, 0.5 ** 2]))
    return sim.ExperimentConfig(controller=cfg, track=named_track("ellipse"),
                                noise=md.NoiseModel(np.diag([std ** 2] * 3)), master_seed=seed,
                                max_steps=steps, init_speed=5.0, collision_threshold=1.2), std


def summarize(rec):
    lat = rec.latency_ms
    return dict(steps=rec.steps, crashed=rec.crashed, collisions=rec.collisions,
                violation_rate=rec.violation_rate, mean_speed=rec.mean_speed, lap_time=rec.lap_time,
                latency_ms_p50=float(np.median(lat)), latency_ms_p99=float(np.percentile(lat, 99)),
                latency_ms_mean=float(lat.mean()), device_ms_p50=float(np.median(rec.device_ms)))


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--seeds", type=int, nargs="+", default=[0, 1, 2])
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--oracle", action="store_true")
    ap.add_argument("--out", default="gpurun_out/closed_loop_c2.json")
    a = ap.parse_args()
    runs = []
    for seed in a.seeds:
        cfg, std = config(seed, a.steps)
        g = sim.run_closed_loop(cfg, 0)
        row = dict(seed=seed, noise_std=std, gpu=summarize(g))
        if a.oracle:
            o = sim.run_closed_loop(cfg, 0, controller_factory=OracleController)
            row["oracle"] = summarize(o)
            n = min(g.steps, o.steps)
            d = np.abs(g.trajectory[:n, :8] - o.trajectory[:n, :8])
            row["traj_max_abs_diff_first10"] = float(d[:10].max())
            row["first_step_u_diff_gt_1e-3"] = int(np.argmax(np.abs(g.trajectory[:n, 8:] - o.trajectory[:n, 8:]).max(1) > 1e-3))
        runs.append(row)
        print(json.dumps(row), flush=True)
    json.dump({"config": "C2: ellipse, K=4096 M=128 T=40 dt=0.05, plant RK4 0.01, 200 steps, "
                         "noise std ~ U[0.01,0.1] per seed, init vx=5, collision threshold 1.2 m",
               "runs": runs}, open(a.out, "w"), indent=1)
