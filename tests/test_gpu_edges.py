"""Edge shapes on the device against the FP64 C oracle driving the same
Philox counters: a single rollout / particle pair / step, ragged lane
groups, the ABI maxima (inner_samples 8192, horizon 512) and the persist
variant's shared-memory limits (the group widens until a block's clouds
fit; M = 1792 is the largest persist cloud)."""

import numpy as np
import pytest

from oracle import c_oracle
from paper_2408_00494_b200 import _lib
from paper_2408_00494_b200 import controllers as mc
from paper_2408_00494_b200 import dynamics as md
from paper_2408_00494_b200.tracks import named_track

pytestmark = pytest.mark.gpu


def _run(K, M, T, persist=False, dt=0.05, seed=0):
    track = named_track("ellipse")
    model = md.with_timestep(md.VehicleParams(), dt, "euler")
    noise = md.NoiseModel(np.diag([0.04 ** 2] * 3))
    cfg = mc.MppiConfig(kind="bss", samples=K, horizon=T, inner_samples=M,
                        sigma_eps=np.diag([0.2 ** 2, 0.5 ** 2]), persist_particles=persist)
    ctx = mc.RolloutContext(model, track, mc.CostSpec(), noise=noise)
    x0 = md.VehicleState.rolling(5.0, model, s=23.0).as_array()
    rng = np.random.default_rng(seed + K + M + T)
    nominal = np.tile([0.01, 0.3], (T, 1))
    eps = rng.standard_normal((K, T, 2)) @ md.psd_factor(cfg.sigma_eps).T
    u = np.clip(nominal[None] + eps, [-0.35, -1.0], [0.35, 1.0])
    kb = (2718281828, 3141592653)
    gpu = mc.rollout_bss(x0, np.zeros((4, 4)), mc.RolloutBatch(u, eps), nominal, ctx, mc.DeviceKey(kb), M,
                         precision=cfg.precision, cost_weight=cfg.control_cost_weight,
                         persist_particles=persist)
    prob, _keep = mc.build_problem("bss", K, T, M, 1.0, cfg.control_cost_weight, cfg.sigma_eps,
                                   cfg.precision, cfg.bounds, persist, ctx)
    ref, _ = c_oracle.rollout(prob, x0, np.zeros((4, 4)), nominal, u=u, eps=eps, key_belief=kb)
    return gpu, ref


@pytest.mark.parametrize("K,M,T,persist", [
    (1, 2, 1, False),            # one rollout, the smallest cloud, one step
    (3, 3, 2, False),            # M < 4: Cholesky rank capped at M - 1
    (33, 7, 3, False),           # ragged K (33 groups of 8) and M (7 of 8 lanes busy)
    (2, 8192, 3, False),         # ABI maximum inner_samples (256 particles per lane)
    (16, 4, 512, False),         # ABI maximum horizon
    (16384, 512, 3, True),       # persist at large K: the group is not narrowed (G = 32, 64 KB of clouds per block)
    (2, 1792, 2, True),          # the largest persist cloud (G = 32 block)
], ids=["K1M2T1", "M3", "ragged", "Mmax", "Tmax", "persist_wide", "persist_max"])
def test_edge_shape_costs_match_oracle(K, M, T, persist):
    """North-star cost bound: 1e-3 relative on every rollout with
    non-negligible weight (S - min S <= 100 lambda); over short horizons on
    every rollout.  Over the 512-step horizon FP32 and FP64 trajectories of
    off-track rollouts separate chaotically, so only the
    weighted ones are bounded there."""
    gpu, ref = _run(K, M, T, persist)
    fin = np.isfinite(ref)
    assert np.array_equal(np.isfinite(gpu), fin)
    rel = np.abs(gpu[fin] - ref[fin]) / np.abs(ref[fin])
    weighted = ref[fin] - ref[fin].min() <= 100.0
    assert rel[weighted].max() < 1e-3, (rel, ref[fin])
    if T <= 50:
        assert rel.max() < 1e-3, rel.max()
        assert np.median(rel) < 1e-5


def test_limits_are_refused():
    """Beyond the maxima the library refuses (BSSMPPI_ERR_UNSUPPORTED, the
    reference's NotImplementedError) instead of launching."""
    for K, M, T, persist, what in [(4, 8193, 3, False, b"inner_samples"), (4, 4, 513, False, b"horizon"),
                                   (4, 1793, 3, True, b"persist")]:
        with pytest.raises(NotImplementedError, match="status 4") as ei:
            _run(K, M, T, persist)
        assert isinstance(ei.value, _lib.BssMppiError)
        assert what in _lib.load().bssmppi_last_error()


@pytest.mark.parametrize("tire", [dict(c_lat_front=2.5, c_lat_rear=2.2),            # C > 2: interior zero of the force
                                  dict(b_lat_front=12.0, b_lat_rear=9.0),          # stiff: > 330 table rows (global copy)
                                  dict(b_lat_front=1.5, c_lat_front=0.8)],
                         ids=["wideC", "stiffB", "soft"])
def test_tire_table_shapes_match_oracle(tire):
    """The lateral forces come from the per-context tire table (any B, C):
    belief rollouts for tires the old polynomial sine could not take (C > 2)
    and for stiff tires whose table exceeds the kernels' shared copy (read
    from global memory instead) match the FP64 C oracle at the north-star
    cost bound."""
    from dataclasses import replace
    K, M, T = 256, 32, 20
    track = named_track("ellipse")
    model = replace(md.with_timestep(md.VehicleParams(), 0.05, "euler"), **tire)
    noise = md.NoiseModel(np.diag([0.04 ** 2] * 3))
    cfg = mc.MppiConfig(kind="bss", samples=K, horizon=T, inner_samples=M, sigma_eps=np.diag([0.2 ** 2, 0.5 ** 2]))
    ctx = mc.RolloutContext(model, track, mc.CostSpec(), noise=noise)
    x0 = md.VehicleState.rolling(5.0, model, s=23.0).as_array()
    rng = np.random.default_rng(11)
    nominal = np.tile([0.05, 0.3], (T, 1))
    eps = rng.standard_normal((K, T, 2)) @ md.psd_factor(cfg.sigma_eps).T
    u = np.clip(nominal[None] + eps, [-0.35, -1.0], [0.35, 1.0])
    kb = (27182818, 31415926)
    gpu = mc.rollout_bss(x0, np.zeros((4, 4)), mc.RolloutBatch(u, eps), nominal, ctx, mc.DeviceKey(kb), M,
                         precision=cfg.precision, cost_weight=cfg.control_cost_weight)
    prob, _keep = mc.build_problem("bss", K, T, M, 1.0, cfg.control_cost_weight, cfg.sigma_eps, cfg.precision,
                                   cfg.bounds, False, ctx)
    ref, _ = c_oracle.rollout(prob, x0, np.zeros((4, 4)), nominal, u=u, eps=eps, key_belief=kb)
    fin = np.isfinite(ref)
    assert np.array_equal(np.isfinite(gpu), fin)
    rel = np.abs(gpu[fin] - ref[fin]) / np.abs(ref[fin])
    assert rel.max() < 1e-3, rel.max()
    assert np.median(rel) < 1e-5


def test_step_array_steering_beyond_the_table():
    """step_array takes arbitrary controls: slip angles past the tire table's
    domain (steering far outside the controller bounds) fall back to the
    libdevice magic formula, so the step still matches the FP64 oracle."""
    from oracle import bss_oracle as orc
    track = named_track("ellipse")
    model = md.with_timestep(md.VehicleParams(), 0.05, "euler")
    rng = np.random.default_rng(5)
    n = 2048
    x = np.zeros((n, 8))
    x[:, 0] = rng.uniform(-3, 7, n)
    x[:, 1] = rng.normal(0, 0.5, n)
    x[:, 2] = rng.normal(0, 0.8, n)
    x[:, 3] = x[:, 0] / 0.095
    x[:, 4] = x[:, 0] / 0.095
    x[:, 5] = rng.normal(0, 0.3, n)
    x[:, 6] = rng.uniform(-1.0, 1.0, n)
    x[:, 7] = rng.uniform(0, track.length, n)
    u = np.stack([rng.uniform(-3.0, 3.0, n), rng.uniform(-1, 1, n)], 1)   # |steering| up to 3 rad
    ctx = mc.RolloutContext(model, track, mc.CostSpec())
    prob, _keep = mc.build_problem("mppi", 1, 1, 1, 1.0, 0.0, np.eye(2), None, mc.ControlBounds(), False, ctx)
    dc = mc.DeviceContext(prob)
    out = np.empty_like(x)
    ok = np.empty(n, dtype=np.uint8)
    _lib.check(dc.lib.bssmppi_step_array(dc.h, n, _lib.dptr(x), _lib.dptr(u), None, _lib.dptr(out),
                                         ok.ctypes.data_as(_lib.C.POINTER(_lib.C.c_uint8))))
    ref, ref_ok = orc.step_euler(x, u, orc.phys(model), track, model.dt)
    assert np.array_equal(ok.astype(bool), ref_ok)
    scale = np.array([5, 1, 1, 50, 50, 1, 1, track.length])
    err = np.abs(out - ref) / scale
    assert err.max() < 5e-6, err.max()
    dc.close()
