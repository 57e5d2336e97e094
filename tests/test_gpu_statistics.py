"""Philox performance mode vs the reference's noise, statistically, at the
BASELINE config-3 shape (SURVEY.md 8c "Perf-mode (Philox) parity"): the same
control batch, R independent belief-noise draws on each side -- in-kernel
Philox4x32-7 (one block per particle-step) on the device, numpy
``standard_normal`` (the reference's generator, controllers.py:285-287) fed
to the FP64 C oracle -- and per-rollout mean cost and per-step sigma_y
(belief.py:297-308) must agree within 3 combined standard errors.

Shape: spline track, M = 256, T = 50, dt = 0.04, process noise std 0.05 (C3),
on a 256-rollout slice of K run at the production lane-group width G = 8
(32 particles per lane, what the K = 16384 launch uses)."""

import math

import numpy as np
import pytest

from helpers import unpack_moments

from oracle import c_oracle
from paper_2408_00494_b200 import controllers as mc
from paper_2408_00494_b200 import dynamics as md
from paper_2408_00494_b200.tracks import named_track

pytestmark = pytest.mark.gpu

K, M, T, DT, R = 256, 256, 50, 0.04, 16


@pytest.fixture(scope="module")
def draws():
    track = named_track("spline0")
    model = md.with_timestep(md.VehicleParams(), DT, "euler")
    noise = md.NoiseModel(np.diag([0.05 ** 2] * 3))
    cfg = mc.MppiConfig(kind="bss", samples=K, horizon=T, inner_samples=M,
                        sigma_eps=np.diag([0.2 ** 2, 0.5 ** 2]))
    ctx = mc.RolloutContext(model, track, mc.CostSpec(), noise=noise)
    x0 = md.VehicleState.rolling(5.0, model, s=17.0).as_array()
    rng = np.random.default_rng(2024)
    nominal = np.tile([0.02, 0.3], (T, 1))
    eps = rng.standard_normal((K, T, 2)) @ md.psd_factor(cfg.sigma_eps).T
    u = np.clip(nominal[None] + eps, [-0.35, -1.0], [0.35, 1.0])
    prob, keep = mc.build_problem("bss", K, T, M, 1.0, cfg.control_cost_weight, cfg.sigma_eps,
                                  cfg.precision, cfg.bounds, False, ctx)
    gc, gs, oc, os_ = [], [], [], []
    for r in range(R):
        c, mom = mc.rollout_bss(x0, np.zeros((4, 4)), mc.RolloutBatch(u, eps), nominal, ctx,
                                mc.DeviceKey((5000 + r, 11)), M, precision=cfg.precision,
                                cost_weight=cfg.control_cost_weight, moments=True, group_width=8)
        gc.append(c)
        gs.append(np.sqrt(np.clip(unpack_moments(mom)[1][..., 3, 3], 0, None)))
        z = np.random.default_rng(r).standard_normal((T, K, M, 7))
        c, _, mom = c_oracle.rollout(prob, x0, np.zeros((4, 4)), nominal, u=u, eps=eps, z=z, moments=True)
        oc.append(c)
        os_.append(np.sqrt(np.clip(unpack_moments(mom)[1][..., 3, 3], 0, None)))
    return tuple(np.stack(a) for a in (gc, gs, oc, os_))


def _z(a, b):
    """Standardised difference of the means over axis 0 (R draws each)."""
    se = np.sqrt(a.var(0, ddof=1) / a.shape[0] + b.var(0, ddof=1) / b.shape[0])
    with np.errstate(divide="ignore", invalid="ignore"):
        return np.where(se > 0, (a.mean(0) - b.mean(0)) / se, 0.0)


def _keep(gc, oc):
    # rollouts alive in every draw on both sides and on the track on average
    # (the C_obs = 1e4 lane-exit indicator makes off-track costs bimodal)
    return np.all(np.isfinite(gc), 0) & np.all(np.isfinite(oc), 0) & (oc.mean(0) < 5e3) & (gc.mean(0) < 5e3)


def test_mean_cost_per_rollout(draws):
    gc, _, oc, _ = draws
    keep = _keep(gc, oc)
    z = _z(gc[:, keep], oc[:, keep])
    n = keep.sum()
    print(f"per-rollout mean cost: {n} rollouts, |z| < 3: {np.mean(np.abs(z) < 3):.4f}, "
          f"max |z| {np.abs(z).max():.2f}, mean z {z.mean():+.3f}")
    # power: >= 64 on-track rollouts x R draws (random controls around a
    # fixed nominal leave about half of K on the track)
    assert n >= K // 4
    assert np.mean(np.abs(z) < 3.0) >= 0.97          # 0.9973 expected
    assert np.abs(z).max() < 5.0
    assert abs(z.mean()) < 4.0 / math.sqrt(n)          # no common bias


def test_sigma_y_per_step(draws):
    gc, gs, oc, os_ = draws
    keep = _keep(gc, oc)
    a, b = gs[:, :, keep], os_[:, :, keep]             # (R, T, k)
    z = _z(a, b)                                       # (T, k)
    zt = z.mean(1) * math.sqrt(z.shape[1])             # pooled over rollouts, per step
    print(f"sigma_y per (t, k): |z| < 3: {np.mean(np.abs(z) < 3):.4f}; per-step pooled max |z| "
          f"{np.abs(zt).max():.2f}; mean sigma_y ratio device/oracle at t=T-1 "
          f"{a[:, -1].mean() / b[:, -1].mean():.5f}")
    assert np.mean(np.abs(z) < 3.0) >= 0.97
    # per-step pooled z (rollouts draw independent noise, so z_t ~ N(0, 1)
    # under parity): SE of the pooled mean sigma_y is ~0.1 %, so this
    # bounds a generator bias at ~0.4 %; 4 sigma over 50 steps: 0.3 % false alarms
    assert np.abs(zt).max() < 4.0
