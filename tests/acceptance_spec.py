"""The reference acceptance suite's closed-loop batches (test_acceptance.py:
37-57 fixture, criteria 07-10 at :204-247), shared by the golden generator
(tests/golden/make_acceptance.py, reference controller, build container) and
the GPU analogue (tests/test_gpu_acceptance.py, the reference's own harness
driving this repo's Controller).

A batch is (kind, q_ey, inner, penalty) on ``sim.default_experiment`` (the
noisy stadium experiment, sim.py:355-372) with RUNS seeded runs.
"""

from dataclasses import replace

RUNS = 20

BATCHES = [
    ("mppi", None, None, None),
    ("smppi", None, None, None),
    ("bss", None, None, None),
    ("smppi", 0.1, None, None),
    ("smppi", 40.0, None, None),
    ("bss", 0.1, None, None),
    ("bss", 40.0, None, None),
    ("bss", None, 2, None),
    ("bss", None, 64, None),
    ("bss", None, None, 0.0),
]


def key(batch):
    kind, q_ey, inner, penalty = batch
    return f"{kind}|q_ey={q_ey}|N={inner}|C={penalty}"


def config(sim, batch, runs=RUNS, workers=1):
    """``sim``: the reference ``belief_mppi.sim`` module."""
    kind, q_ey, inner, penalty = batch
    cfg = sim.default_experiment(kind, runs=runs, workers=workers)
    if q_ey is not None:
        cfg = sim.apply_axis(cfg, "q_ey", q_ey)
    if inner is not None:
        cfg = sim.apply_axis(cfg, "N", inner)
    if penalty is not None:
        cfg = replace(cfg, cost=replace(cfg.cost, safety=replace(cfg.cost.safety, penalty=penalty)))
    return cfg


def summary(report):
    return dict(
        crash_ratio=report.crash_ratio, mean_satisfaction=report.mean_satisfaction,
        collision_ratio=report.collision_ratio, completion_ratio=report.completion_ratio,
        mean_speed=report.mean_speed,
        crashed=[bool(r.crashed) for r in report.records],
        satisfaction=[r.satisfaction_rate for r in report.records],
        steps=[int(r.steps) for r in report.records])
