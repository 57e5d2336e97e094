"""Full-size parity (BASELINE C3 / C5 shapes) where the reference's numpy
noise arrays would be multi-GB: the device (Philox mode) against the FP64 C
oracle driving the SAME Philox4x32 counters on the host (oracle/bss_oracle.c,
pinned to the reference by tests/test_c_oracle.py).  The two differ only by
FP32 vs FP64 arithmetic and the device Box-Muller (MUFU radius, tabulated
angles) vs libm (~1e-7 on the normals).
These shapes exercise the narrowed lane groups of large K (G = 8 at C3, 4 at
C5 32768 x 64, 2 at the C4 shape 65536 x 64) and the 512-thread one-wave
launches (C2; a ragged 2047-rollout shard whose last block is partial)."""

import numpy as np
import pytest

from helpers import channel_spread, death_mismatches_weightless, moments_err_arrays, unpack_moments

from oracle import c_oracle
from paper_2408_00494_b200 import _lib
from paper_2408_00494_b200 import controllers as mc
from paper_2408_00494_b200 import dynamics as md
from paper_2408_00494_b200.tracks import named_track

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("K,M,T,dt", [(16384, 256, 50, 0.04), (32768, 64, 60, 0.04), (4096, 128, 40, 0.05),
                                     (2047, 256, 20, 0.05), (65536, 64, 50, 0.04)],
                         ids=["C3", "C5_32768x64", "C2", "ragged_one_wave", "C4_shape_G2"])
def test_fullsize_philox_costs_and_update(K, M, T, dt):
    track = named_track("spline0" if dt == 0.04 else "ellipse")
    model = md.with_timestep(md.VehicleParams(), dt, "euler")
    noise = md.NoiseModel(np.diag([0.05 ** 2] * 3))
    cfg = mc.MppiConfig(kind="bss", samples=K, horizon=T, inner_samples=M,
                        sigma_eps=np.diag([0.2 ** 2, 0.5 ** 2]))
    ctx = mc.RolloutContext(model, track, mc.CostSpec(), noise=noise)
    x0 = md.VehicleState.rolling(5.0, model, s=17.0).as_array()
    rng = np.random.default_rng(K + M)
    nominal = np.tile([0.02, 0.3], (T, 1))
    eps = rng.standard_normal((K, T, 2)) @ md.psd_factor(cfg.sigma_eps).T
    u = np.clip(nominal[None] + eps, [-0.35, -1.0], [0.35, 1.0])
    kb = (123456789, 987654321)
    gpu, gmom = mc.rollout_bss(x0, np.zeros((4, 4)), mc.RolloutBatch(u, eps), nominal, ctx, mc.DeviceKey(kb),
                               M, precision=cfg.precision, cost_weight=cfg.control_cost_weight, moments=True)
    prob, keep = mc.build_problem("bss", K, T, M, 1.0, cfg.control_cost_weight, cfg.sigma_eps,
                                  cfg.precision, cfg.bounds, False, ctx)
    ref, _, rmom = c_oracle.rollout(prob, x0, np.zeros((4, 4)), nominal, u=u, eps=eps, key_belief=kb,
                                    moments=True)
    fin = np.isfinite(ref)
    n_mism, weightless = death_mismatches_weightless(gpu, ref)
    print(f"K={K} M={M}: dead in one of device / oracle only: {n_mism} of {K}")
    assert n_mism <= 1e-3 * K and weightless
    both = fin & np.isfinite(gpu)
    rel = np.abs(gpu[both] - ref[both]) / np.abs(ref[both])
    weighted = both & (ref - ref[fin].min() <= 100.0)
    print(f"K={K} M={M}: weighted rel err max {np.max(np.abs(gpu[weighted] - ref[weighted]) / ref[weighted]):.2e}, "
          f"all: frac<1e-3 {np.mean(rel < 1e-3):.5f}, median {np.median(rel):.1e}")
    assert np.max(np.abs(gpu[weighted] - ref[weighted]) / np.abs(ref[weighted])) < 1e-3
    assert np.mean(rel < 1e-3) > 0.99
    # per-step belief moments at the production lane-group width (C3: G = 8,
    # 32 particles per lane; C5 32768x64: G = 4, 16 per lane): the device's
    # shifted one-pass sums vs the C oracle's tree mean + two-pass
    # covariance (belief.py:275-308), on rollouts alive in both
    G = _lib.load().bssmppi_group_width(M, K)
    em, ec = moments_err_arrays(*unpack_moments(gmom), *unpack_moments(rmom), channel_spread(noise.factor))
    per_k = np.maximum(em.max(axis=(0, 2)), ec.max(axis=(0, 2, 3)))
    print(f"  G={G} ({-(-M // G)} particles per lane): moments max {per_k[weighted].max():.2e} (weighted), "
          f"frac alive <= 1e-4 {np.mean(per_k[both] <= 1e-4):.5f}, median {np.median(per_k[both]):.1e}")
    assert per_k[weighted].max() <= 1e-4
    assert np.mean(per_k[both] <= 1e-4) > 0.99
    v_gpu = mc.mppi_update(mc.RolloutBatch(u, eps, gpu), 1.0, mc.ControlBounds()).controls
    v_ref = c_oracle.update(ref, u, 1.0, [-0.35, -1.0], [0.35, 1.0])
    top2 = np.sort(ref[fin])[:2]
    if top2[1] - top2[0] > 1e-3 * top2[0]:
        np.testing.assert_allclose(v_gpu, v_ref, atol=1e-4)
