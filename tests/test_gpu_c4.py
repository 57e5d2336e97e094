"""BASELINE config 4 (extension beyond the reference, obstacles.py) on the
device vs the extended FP64 C oracle driving the same Philox counters:
K=65536 x M=64 x T=50, Laplace(0.03) + U(+-0.05) slip noise, shield beta=0.2,
16 seeded obstacles with delta=0.02 chance constraints."""

import numpy as np
import pytest

from helpers import death_mismatches_weightless
from oracle import c_oracle
from paper_2408_00494_b200 import controllers as mc
from paper_2408_00494_b200 import dynamics as md
from paper_2408_00494_b200.constraints import SafetyParams
from paper_2408_00494_b200.obstacles import LaplaceSlipNoise, Obstacles, place_obstacles
from paper_2408_00494_b200.tracks import named_track

pytestmark = pytest.mark.gpu


def _c4(K=65536, M=64, T=50, obstacles=True):
    track = named_track("spline0")
    model = md.with_timestep(md.VehicleParams(), 0.04, "euler")
    cost = mc.CostSpec(safety=SafetyParams(0.2, 2000.0))
    obs = place_obstacles(track, 16, seed=0) if obstacles else None
    ctx = mc.RolloutContext(model, track, cost, noise=LaplaceSlipNoise(0.03, 0.05), obstacles=obs)
    cfg = mc.MppiConfig(kind="bss", samples=K, horizon=T, inner_samples=M,
                        sigma_eps=np.diag([0.2 ** 2, 0.5 ** 2]))
    return cfg, ctx, track, model


def _batch(cfg, T, seed):
    rng = np.random.default_rng(seed)
    nominal = np.tile([0.0, 0.35], (T, 1))
    eps = rng.standard_normal((cfg.samples, T, 2)) @ md.psd_factor(cfg.sigma_eps).T
    u = np.clip(nominal[None] + eps, [-0.35, -1.0], [0.35, 1.0])
    return nominal, u, eps


def test_c4_device_vs_extended_oracle():
    cfg, ctx, track, model = _c4()
    T = cfg.horizon
    x0 = md.VehicleState.rolling(5.0, model, s=40.0).as_array()
    nominal, u, eps = _batch(cfg, T, 4)
    kb = (2024, 11)
    gpu = mc.rollout_bss(x0, np.zeros((4, 4)), mc.RolloutBatch(u, eps), nominal, ctx, mc.DeviceKey(kb),
                         cfg.inner_samples, precision=cfg.precision, cost_weight=cfg.control_cost_weight)
    prob, keep = mc.build_problem("bss", cfg.samples, T, cfg.inner_samples, 1.0, cfg.control_cost_weight,
                                  cfg.sigma_eps, cfg.precision, cfg.bounds, False, ctx)
    ref, _ = c_oracle.rollout(prob, x0, np.zeros((4, 4)), nominal, u=u, eps=eps, key_belief=kb)
    fin = np.isfinite(ref) & np.isfinite(gpu)
    n_mism, weightless = death_mismatches_weightless(gpu, ref)
    print(f"C4: dead in one of device / oracle only: {n_mism} of {cfg.samples}")
    assert n_mism <= 1e-3 * cfg.samples and weightless
    rel = np.abs(gpu[fin] - ref[fin]) / np.abs(ref[fin])
    w = fin & (ref - ref[fin].min() <= 100.0)
    werr = np.max(np.abs(gpu[w] - ref[w]) / ref[w])
    print(f"C4: weighted rel err {werr:.2e}, frac<1e-3 {np.mean(rel < 1e-3):.5f}, median {np.median(rel):.1e}")
    assert werr < 1e-3 and np.mean(rel < 1e-3) > 0.99
    # the obstacles matter: the same batch without them is cheaper
    cfg0, ctx0, _, _ = _c4(obstacles=False)
    free = mc.rollout_bss(x0, np.zeros((4, 4)), mc.RolloutBatch(u, eps), nominal, ctx0, mc.DeviceKey(kb),
                          cfg.inner_samples, precision=cfg.precision, cost_weight=cfg.control_cost_weight)
    both = fin & np.isfinite(free)
    assert np.mean(gpu[both] >= free[both] - 1e-3 * np.abs(free[both])) > 0.999
    assert np.mean(gpu[both] > free[both] * (1 + 1e-4)) > 0.01


def test_far_obstacles_bit_identical_on_device():
    cfg, ctx, track, model = _c4(K=1024, M=64, T=30, obstacles=False)
    far = mc.RolloutContext(ctx.model, ctx.track, ctx.cost, noise=ctx.noise,
                            obstacles=Obstacles(np.array([[1e4, 1e4], [-1e4, 5e3]]), np.array([1.0, 0.7])))
    x0 = md.VehicleState.rolling(5.0, model, s=10.0).as_array()
    nominal, u, eps = _batch(cfg, 30, 7)
    a = mc.rollout_bss(x0, None, mc.RolloutBatch(u, eps), nominal, ctx, mc.DeviceKey((1, 2)), 64)
    b = mc.rollout_bss(x0, None, mc.RolloutBatch(u, eps), nominal, far, mc.DeviceKey((1, 2)), 64)
    np.testing.assert_array_equal(a, b)


def test_c4_controller_runs_and_reference_noise_rejected():
    cfg, ctx, track, model = _c4(K=4096, M=64, T=50)
    with pytest.raises(ValueError):
        mc.Controller(cfg, ctx.cost, model, track, noise=ctx.noise, obstacles=ctx.obstacles,
                      noise_source="reference")
    ctrl = mc.Controller(cfg, ctx.cost, model, track, noise=ctx.noise, obstacles=ctx.obstacles, seed=1)
    u0, plan = ctrl.control_step(md.VehicleState.rolling(5.0, model, s=40.0).as_array())
    assert np.all(np.isfinite(u0)) and ctrl.last_diagnostics["n_finite"] > 0
