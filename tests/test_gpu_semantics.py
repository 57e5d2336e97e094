"""GPU analogues of the reference's own unit tests (pkg/tests/test_controllers.py,
test_belief.py, test_dynamics.py) plus the device generator and the K-shard
path.  Same-precision comparisons run within FP32 on the device."""

import math

import numpy as np
import pytest

from cases import update_batch
from helpers import Inputs

from oracle import bss_oracle as orc
from oracle import c_oracle
from paper_2408_00494_b200 import _lib
from paper_2408_00494_b200 import controllers as mc
from paper_2408_00494_b200 import dynamics as md
from paper_2408_00494_b200 import streams
from paper_2408_00494_b200.constraints import SafetyParams
from paper_2408_00494_b200.tracks import named_track

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def oval():
    return named_track("oval")


@pytest.fixture(scope="module")
def model():
    return md.with_timestep(md.VehicleParams(), 0.05, "euler")


def quiet_cost(**kw):
    d = dict(q_diag=np.zeros(8), obstacle_penalty=0.0, safety=SafetyParams(0.5, 0.0))
    d.update(kw)
    return mc.CostSpec(**d)


# ------------------------------------------------------------ generator

def test_philox_device_known_answers():
    lib = _lib.load()
    out = (_lib.C.c_uint32 * 4)()
    for ctr, key, exp in [([0, 0, 0, 0], [0, 0], [0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8]),
                          ([0xFFFFFFFF] * 4, [0xFFFFFFFF] * 2,
                           [0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD]),
                          ([0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344], [0xA4093822, 0x299F31D0],
                           [0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1])]:
        _lib.check(lib.bssmppi_philox4x32((_lib.C.c_uint32 * 4)(*ctr), (_lib.C.c_uint32 * 2)(*key), 10, out))
        assert list(out) == exp
    # the 7-round belief generator agrees with the C port bit for bit
    rng = np.random.default_rng(1)
    for _ in range(16):
        ctr = [int(v) for v in rng.integers(0, 2 ** 32, 4)]
        key = [int(v) for v in rng.integers(0, 2 ** 32, 2)]
        _lib.check(lib.bssmppi_philox4x32((_lib.C.c_uint32 * 4)(*ctr), (_lib.C.c_uint32 * 2)(*key), 7, out))
        assert list(out) == c_oracle.philox(ctr, key, rounds=7)


def test_belief_normals_statistics():
    lib = _lib.load()
    n = 1 << 18
    z = np.empty((n, 7), dtype=np.float32)
    _lib.check(lib.bssmppi_belief_normals(_lib.key_arr((12345, 678)), 3, 77, n, _lib.fptr(z)))
    se = 1.0 / math.sqrt(n)
    assert np.all(np.abs(z.mean(0)) < 5 * se)
    assert np.all(np.abs(z.var(0) - 1.0) < 5 * math.sqrt(2.0) * se)
    c = np.corrcoef(z.T.astype(np.float64))
    assert np.all(np.abs(c[np.triu_indices(7, 1)]) < 5 * se)
    # tails: P(|z| > 3) = 0.0027
    assert abs(np.mean(np.abs(z) > 3.0) - 0.0027) < 0.0006
    # adjacent counters (m, m+1) are uncorrelated, and uniform bins are flat
    a, b = z[:-1].astype(np.float64), z[1:].astype(np.float64)
    lag = np.mean(a * b, 0)
    assert np.all(np.abs(lag) < 5 * se)
    from scipy.stats import chi2, norm
    u = norm.cdf(z[:, 0].astype(np.float64))
    hist = np.bincount(np.minimum((u * 64).astype(int), 63), minlength=64)
    stat = ((hist - n / 64) ** 2 / (n / 64)).sum()
    assert stat < chi2.ppf(0.9999, 63)
    z2 = np.empty_like(z)
    _lib.check(lib.bssmppi_belief_normals(_lib.key_arr((12345, 678)), 3, 77, n, _lib.fptr(z2)))
    assert np.array_equal(z, z2)


def test_belief_normals_match_oracle():
    """Device Box-Muller (MUFU lg2/sqrt/sin/cos on the raw form, kBmNeg
    scale) equals the FP64 oracle's bm() on the same Philox words."""
    lib = _lib.load()
    n = 1 << 14
    z = np.empty((n, 7), dtype=np.float32)
    _lib.check(lib.bssmppi_belief_normals(_lib.key_arr((12345, 678)), 3, 77, n, _lib.fptr(z)))
    ref = c_oracle.belief_normals((12345, 678), 3, 77, n)
    err = np.abs(z - ref)
    assert err.max() < 3e-5, err.max()
    assert np.median(err) < 1e-6, np.median(err)


# ------------------------------------------------------------ dynamics

def test_step_array_matches_oracle(oval, model):
    rng = np.random.default_rng(0)
    n = 4096
    x = np.zeros((n, 8))
    x[:, 0] = rng.uniform(0.5, 7, n)
    x[:, 1] = rng.normal(0, 0.3, n)
    x[:, 2] = rng.normal(0, 0.5, n)
    x[:, 3] = x[:, 0] / 0.095 * rng.uniform(0.8, 1.3, n)
    x[:, 4] = x[:, 0] / 0.095 * rng.uniform(0.8, 1.3, n)
    x[:, 5] = rng.normal(0, 0.3, n)
    x[:, 6] = rng.uniform(-1.8, 1.8, n)
    x[:, 7] = rng.uniform(0, oval.length, n)
    u = np.stack([rng.uniform(-0.35, 0.35, n), rng.uniform(-1, 1, n)], 1)
    ctx = mc.RolloutContext(model, oval, mc.CostSpec())
    prob, keep = mc.build_problem("mppi", 1, 1, 1, 1.0, 0.0, np.eye(2), None, mc.ControlBounds(),
                                  False, ctx)
    dc = mc.DeviceContext(prob)
    out = np.empty_like(x)
    ok = np.empty(n, dtype=np.uint8)
    _lib.check(dc.lib.bssmppi_step_array(dc.h, n, _lib.dptr(x), _lib.dptr(u), None, _lib.dptr(out),
                                         ok.ctypes.data_as(_lib.C.POINTER(_lib.C.c_uint8))))
    ref, ref_ok = orc.step_euler(x, u, orc.phys(model), oval, model.dt)
    assert np.array_equal(ok.astype(bool), ref_ok)
    scale = np.array([5, 1, 1, 50, 50, 1, 1, oval.length])
    err = np.abs(out - ref) / scale
    assert err.max() < 2e-6, err.max()
    dc.close()


def test_step_array_reverse_zero_slip(oval, model):
    """Reverse driving with zero lateral velocity and yaw rate: both slip
    angles are atan2(+0, vx < 0) = +pi in the reference (dynamics.py:381-382),
    so the device must keep the IEEE sign of vy + l r (signed zeros
    included) rather than derive it from the product with 1/vx."""
    n = 4
    x = np.zeros((n, 8))
    x[:, 0] = [-2.0, -0.8, -3.5, -2.0]
    x[:, 3] = x[:, 0] / 0.095
    x[:, 4] = x[:, 0] / 0.095
    x[:, 6] = [0.2, -0.1, 0.0, 0.3]
    x[:, 7] = [20.0, 5.0, 40.0, 1.0]
    x[3, 1] = 1e-3                      # one non-degenerate row
    u = np.tile([0.05, -0.5], (n, 1))
    ctx = mc.RolloutContext(model, oval, mc.CostSpec())
    prob, keep = mc.build_problem("mppi", 1, 1, 1, 1.0, 0.0, np.eye(2), None, mc.ControlBounds(),
                                  False, ctx)
    dc = mc.DeviceContext(prob)
    out = np.empty_like(x)
    ok = np.empty(n, dtype=np.uint8)
    _lib.check(dc.lib.bssmppi_step_array(dc.h, n, _lib.dptr(x), _lib.dptr(u), None, _lib.dptr(out),
                                         ok.ctypes.data_as(_lib.C.POINTER(_lib.C.c_uint8))))
    dc.close()
    ref, ref_ok = orc.step_euler(x, u, orc.phys(model), oval, model.dt)
    assert np.array_equal(ok.astype(bool), ref_ok)
    scale = np.array([5, 1, 1, 50, 50, 1, 1, oval.length])
    assert (np.abs(out - ref) / scale).max() < 2e-6


def _f32_track_s(s, L, closed):
    """float32 emulation of the device arc-length wrap (vehicle.cuh track_s:
    Python floor-mod on a closed track, exact on [-L, 2L) and fmodf beyond;
    clamp on an open one)."""
    f = np.float32
    s, L = f(s), f(L)
    if not closed:   # reference: s < 0 -> 0, s > L -> L, NaN passes (dynamics.py:488-491)
        return s if np.isnan(s) else f(min(max(s, f(0)), L))
    if not np.isfinite(s):
        return f(np.nan)
    if f(0) <= s < L:
        return s
    if L <= s < f(2) * L:
        return f(s - L)
    if -L <= s < f(0):
        return f(s + L)
    r = f(np.fmod(s, L))
    return f(r + L) if r < 0 else r


@pytest.mark.parametrize("closed", [True, False])
def test_step_array_rare_events(model, closed):
    """The step's rare-event screen (vehicle.cuh common_case + rare_fixup,
    wrap_pi) at its exact boundaries: with vx = vy = r = 0 the arc length and
    heading pass through the Euler update unchanged, so the device output is
    the wrap of the float32 input (dynamics.py:479-496 semantics)."""
    segs = named_track("oval")
    if closed:
        track = segs
    else:
        track = md.Track(segs.s, segs.kappa, segs.half_width, closed=False, length=segs.s[-1] + 1.0)
    f = np.float32
    L = f(track.length)
    ulp = np.spacing(L)
    s_in = [0.0, 1e-30, L / 2, L - ulp, L, L + ulp, f(1.5) * L, -ulp, f(-1.0), f(-0.5) * L,
            f(2.5) * L, f(-3.25) * L, np.inf, np.nan]
    pi = f(np.pi)
    e_in = [0.0, np.nextafter(pi, f(0)), pi, np.nextafter(pi, f(4)), -pi, np.nextafter(-pi, f(0)),
            f(4.0), f(-4.0), f(1e3)]
    rows = [(sv, 0.0) for sv in s_in] + [(10.0, ev) for ev in e_in]
    n = len(rows)
    x = np.zeros((n, 8))
    x[:, 7] = [r[0] for r in rows]
    x[:, 5] = [r[1] for r in rows]
    x[:, 6] = 0.1
    u = np.zeros((n, 2))
    ctx = mc.RolloutContext(model, track, mc.CostSpec())
    prob, keep = mc.build_problem("mppi", 1, 1, 1, 1.0, 0.0, np.eye(2), None, mc.ControlBounds(),
                                  False, ctx)
    dc = mc.DeviceContext(prob)
    out = np.empty_like(x)
    ok = np.empty(n, dtype=np.uint8)
    _lib.check(dc.lib.bssmppi_step_array(dc.h, n, _lib.dptr(x), _lib.dptr(u), None, _lib.dptr(out),
                                         ok.ctypes.data_as(_lib.C.POINTER(_lib.C.c_uint8))))
    dc.close()
    for i, (sv, ev) in enumerate(rows):
        exp_s = _f32_track_s(sv, L, closed)
        if np.isnan(exp_s):        # non-finite -> 0 and the step is not ok
            assert out[i, 7] == 0.0 and not ok[i], (sv, out[i])
            continue
        assert f(out[i, 7]) == exp_s, (sv, out[i, 7], exp_s)
        e = f(ev)
        exp_e = e if -pi < e <= pi else f(pi - _f32_track_s(f(pi - e), f(2 * np.pi), True))
        assert f(out[i, 5]) == exp_e, (ev, out[i, 5], exp_e)
        assert -pi <= out[i, 5] <= pi
        assert ok[i]


# ------------------------------------------------------------ update law
# (reference test_controllers.py:86-147)

def test_uniform_costs_give_mean():
    rng = np.random.default_rng(0)
    controls = rng.uniform(-0.2, 0.2, size=(16, 4, 2))
    plan = mc.mppi_update(mc.RolloutBatch(controls, np.zeros_like(controls), np.full(16, 5.0)), 1.0,
                          mc.ControlBounds())
    assert np.allclose(plan.controls, controls.mean(axis=0), atol=1e-15)


def test_baseline_shift_bit_invariance():
    rng = np.random.default_rng(9)
    costs = rng.integers(0, 2 ** 20, 64).astype(float) / 2 ** 10
    controls = rng.uniform(-0.3, 0.3, size=(64, 6, 2))
    base = mc.mppi_update(mc.RolloutBatch(controls, np.zeros_like(controls), costs), 0.7,
                          mc.ControlBounds())
    for shift in (1.0, -256.0, 4096.0, 1e6):
        shifted = mc.mppi_update(mc.RolloutBatch(controls, np.zeros_like(controls), costs + shift), 0.7,
                                 mc.ControlBounds())
        assert np.array_equal(base.controls, shifted.controls)


def test_temperature_collapse_to_argmin():
    rng = np.random.default_rng(12)
    costs = rng.uniform(1.0, 100.0, 128)
    controls = rng.uniform(-0.3, 0.3, size=(128, 5, 2))
    plan = mc.mppi_update(mc.RolloutBatch(controls, np.zeros_like(controls), costs), 1e-9,
                          mc.ControlBounds())
    assert np.max(np.abs(plan.controls - controls[np.argmin(costs)])) < 1e-6


def test_infinite_costs_ignored_and_all_invalid_raises():
    controls = np.zeros((3, 2, 2))
    controls[0] += 0.1
    plan = mc.mppi_update(mc.RolloutBatch(controls, np.zeros_like(controls), np.array([np.inf, np.inf, 4.0])),
                          1.0, mc.ControlBounds())
    assert np.array_equal(plan.controls, controls[2])
    with pytest.raises(mc.AllRolloutsInvalid):
        mc.mppi_update(mc.RolloutBatch(controls, np.zeros_like(controls), np.full(3, np.inf)), 1.0,
                       mc.ControlBounds())


def test_sample_controls_semantics():
    plan = mc.ControlPlan(np.tile([0.1, 0.4], (5, 1)))
    batch = mc.sample_controls(plan, np.zeros((2, 2)), 8, streams.substream(0), mc.ControlBounds())
    assert np.array_equal(batch.controls, np.tile(plan.controls, (8, 1, 1)))
    assert not np.any(batch.perturbations)
    b = mc.ControlBounds()
    plan = mc.ControlPlan(np.tile([b.delta_max, b.throttle_max], (3, 1)))
    batch = mc.sample_controls(plan, np.diag([0.04, 0.04]), 64, streams.substream(1), b)
    assert batch.controls[..., 0].max() <= b.delta_max
    assert (plan.controls[None] + batch.perturbations).max() > b.throttle_max
    # identical to the reference's numpy draw
    ref = streams.substream(1).standard_normal((64, 3, 2)) @ md.psd_factor(np.diag([0.04, 0.04])).T
    np.testing.assert_allclose(batch.perturbations, ref, atol=1e-15)


# ------------------------------------------------------------ rollouts
# (reference test_controllers.py:150-307)

def _batch(c):
    c = np.asarray(c, dtype=float)
    return mc.RolloutBatch(c, np.zeros_like(c))


def test_invalid_rollout_gets_inf(oval, model):
    ctx = mc.RolloutContext(model, oval, quiet_cost())
    x0 = md.VehicleState.rolling(3.0, model, s=25.0, e_y=6.5).as_array()
    total = mc.rollout_mppi(x0, _batch(np.zeros((2, 3, 2))), np.zeros((3, 2)), ctx)
    assert np.all(np.isinf(total))


def test_zero_weights_zero_cost(oval, model):
    ctx = mc.RolloutContext(model, oval, quiet_cost())
    x0 = md.VehicleState.rolling(3.0, model, s=1.0).as_array()
    total = mc.rollout_mppi(x0, _batch(np.full((4, 6, 2), 0.1)), np.zeros((6, 2)), ctx)
    assert np.array_equal(total, np.zeros(4))


def test_bss_reduces_to_smppi_without_uncertainty(oval, model):
    """Bit-exact on the device (the reference asserts 1e-9 in FP64)."""
    cost = mc.CostSpec(q_diag=np.array([1.0, 0, 0.1, 0, 0, 2.0, 0.5, 0]), safety=SafetyParams(0.5, 3000.0))
    ctx = mc.RolloutContext(model, oval, cost, noise=md.NoiseModel(np.zeros((3, 3))))
    x0 = md.VehicleState.rolling(4.0, model, s=16.0, e_y=0.8).as_array()
    batch = _batch(np.random.default_rng(3).uniform(-0.2, 0.4, size=(8, 10, 2)))
    det = mc.rollout_smppi(x0, batch, np.zeros((10, 2)), ctx)
    for n in (2, 16, 5, 64):
        belief = mc.rollout_bss(x0, np.zeros((4, 4)), batch, np.zeros((10, 2)), ctx,
                                rng=streams.substream(77), inner_samples=n)
        assert np.array_equal(belief, det)
        belief = mc.rollout_bss(x0, np.zeros((4, 4)), batch, np.zeros((10, 2)), ctx,
                                rng=mc.DeviceKey((1, 2)), inner_samples=n)
        assert np.array_equal(belief, det)


def test_zero_cov_zero_noise_moments_collapse(oval, model):
    """belief.py:282-284 guarantee: moments == deterministic step, cov == 0."""
    ctx = mc.RolloutContext(model, oval, mc.CostSpec(), noise=md.NoiseModel(np.zeros((3, 3))))
    x0 = md.VehicleState.rolling(3.0, model, s=4.0, e_y=0.5).as_array()
    u = np.tile([[0.05, 0.3]], (1, 6, 1))
    costs, mom = mc.rollout_bss(x0, np.zeros((4, 4)), _batch(u), np.zeros((6, 2)), ctx,
                                rng=streams.substream(9), inner_samples=16, moments=True)
    assert not np.any(mom[:, 0, 8:])
    prob, keep = mc.build_problem("mppi", 1, 1, 1, 1.0, 0.0, np.eye(2), None, mc.ControlBounds(), False, ctx)
    dc = mc.DeviceContext(prob)
    x = x0.copy()
    for t in range(6):
        out = np.empty(8)
        ok = np.empty(1, dtype=np.uint8)
        _lib.check(dc.lib.bssmppi_step_array(dc.h, 1, _lib.dptr(x), _lib.dptr(np.array([0.05, 0.3])), None,
                                             _lib.dptr(out), ok.ctypes.data_as(_lib.C.POINTER(_lib.C.c_uint8))))
        assert np.array_equal(mom[t, 0, :8].astype(np.float64), out)
        x = out.astype(np.float32).astype(np.float64)
    dc.close()


def test_persistent_particles_match_when_degenerate(oval, model):
    cost = mc.CostSpec(safety=SafetyParams(0.35, 3000.0))
    ctx = mc.RolloutContext(model, oval, cost, noise=md.NoiseModel(np.zeros((3, 3))))
    x0 = md.VehicleState.rolling(4.0, model, s=16.0, e_y=0.8).as_array()
    batch = _batch(np.random.default_rng(3).uniform(-0.2, 0.4, size=(8, 10, 2)))
    plain = mc.rollout_bss(x0, np.zeros((4, 4)), batch, np.zeros((10, 2)), ctx, rng=streams.substream(21),
                           inner_samples=8)
    persist = mc.rollout_bss(x0, np.zeros((4, 4)), batch, np.zeros((10, 2)), ctx, rng=streams.substream(21),
                             inner_samples=8, persist_particles=True)
    assert np.array_equal(plain, persist)


def test_bss_penalizes_uncertainty(oval, model):
    cost = quiet_cost(safety=SafetyParams(0.3, 3000.0))
    x0 = md.VehicleState.rolling(5.0, model, s=14.0, e_y=1.4, e_psi=0.05).as_array()
    batch = _batch(np.zeros((1, 20, 2)))
    quiet = mc.rollout_bss(x0, np.zeros((4, 4)), batch, np.zeros((20, 2)),
                           mc.RolloutContext(model, oval, cost, noise=md.NoiseModel(np.zeros((3, 3)))),
                           rng=streams.substream(5), inner_samples=64)
    noisy = mc.rollout_bss(x0, np.zeros((4, 4)), batch, np.zeros((20, 2)),
                           mc.RolloutContext(model, oval, cost,
                                             noise=md.NoiseModel(np.diag([0.15 ** 2, 0.15 ** 2, 0.35 ** 2]))),
                           rng=streams.substream(5), inner_samples=64)
    assert noisy[0] > quiet[0]


# ------------------------------------------------------------ control step
# (reference test_controllers.py:310-366)

def test_degenerate_returns_nominal(oval, model):
    cfg = mc.MppiConfig(kind="mppi", samples=1, horizon=6, temperature=1.0, sigma_eps=np.zeros((2, 2)))
    ctrl = mc.Controller(cfg, quiet_cost(), model, oval, seed=0)
    nominal = np.tile([0.05, 0.2], (6, 1))
    ctrl.plan = mc.ControlPlan(nominal.copy())
    u0, plan = ctrl.control_step(md.VehicleState.rolling(3.0, model).as_array())
    assert np.allclose(u0, [0.05, 0.2], atol=1e-7)
    assert np.allclose(plan.controls, nominal, atol=1e-7)


@pytest.mark.parametrize("noise_source", ["philox", "reference"])
def test_identical_seeds_identical_controls(oval, model, noise_source):
    cfg = mc.MppiConfig(kind="bss", samples=64, horizon=8, temperature=5.0, inner_samples=32)
    x0 = md.VehicleState.rolling(3.0, model, s=3.0).as_array()
    noise = md.NoiseModel(np.diag([0.05, 0.05, 0.1]) ** 2)
    outs = []
    for _ in range(2):
        ctrl = mc.Controller(cfg, mc.CostSpec(), model, oval, noise=noise, seed=42, run_path=(1,),
                             noise_source=noise_source)
        outs.append((ctrl.control_step(x0)[0], ctrl.control_step(x0)[0]))
    assert np.array_equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1])


def test_bss_matches_smppi_closed_loop_without_noise(oval, model):
    """30-step closed loop, zero noise: BSS == S-MPPI (reference: 1e-9)."""
    zero = md.NoiseModel(np.zeros((3, 3)))
    x_s = md.VehicleState.rolling(3.0, model, s=1.0).as_array()
    x_b = x_s.copy()
    smppi = mc.Controller(mc.MppiConfig(kind="smppi", samples=48, horizon=10, temperature=5.0),
                          mc.CostSpec(), model, oval, noise=zero, seed=11)
    bss = mc.Controller(mc.MppiConfig(kind="bss", samples=48, horizon=10, temperature=5.0, inner_samples=2),
                        mc.CostSpec(), model, oval, noise=zero, seed=11)
    for _ in range(30):
        u_s, _ = smppi.control_step(x_s)
        u_b, _ = bss.control_step(x_b)
        assert np.max(np.abs(u_s - u_b)) < 1e-9
        x_s, _ = orc.step_euler(x_s, u_s, orc.phys(model), oval, model.dt)
        x_b, _ = orc.step_euler(x_b, u_b, orc.phys(model), oval, model.dt)


def test_speed_tracking_on_straight(model):
    track = md.make_test_track([(500.0, 0.0), (math.pi * 6, 1 / 6), (500.0, 0.0), (math.pi * 6, 1 / 6)], 2.0)
    ctrl = mc.Controller(mc.MppiConfig(kind="mppi", samples=512, horizon=20, temperature=2.0),
                         mc.CostSpec(), model, track, seed=7)
    x = md.VehicleState.rolling(2.0, model).as_array()
    for _ in range(100):
        u0, _ = ctrl.control_step(x)
        x, ok = orc.step_euler(x, u0, orc.phys(model), track, model.dt)
        assert ok
    assert 5.0 <= x[0] <= 7.0


# ------------------------------------------------------------ Philox mode vs oracle (statistical)

def test_philox_mode_statistical_parity():
    """Same control batch; R independent belief-noise draws on each side:
    per-rollout mean cost of GPU-Philox and the FP64 oracle (numpy normals)
    agree within 4 combined standard errors."""
    inp = Inputs("c1_s0")
    K = 48
    u, eps = inp.u[:K], inp.eps[:K]
    R = 24
    gpu = np.stack([mc.rollout_bss(inp.x0, inp.cov0, mc.RolloutBatch(u, eps), inp.plan, inp.ctx,
                                   mc.DeviceKey((1000 + r, 7)), inp.M, precision=inp.cfg.precision,
                                   cost_weight=inp.cfg.control_cost_weight) for r in range(R)])
    ora = np.stack([orc.rollout_bss(inp.prob, inp.x0, inp.cov0, u, eps, inp.plan,
                                    np.random.default_rng(r).standard_normal((inp.T, K, inp.M, 7)),
                                    inp.cfg.precision, inp.cfg.control_cost_weight) for r in range(R)])
    keep = np.all(np.isfinite(gpu), 0) & np.all(np.isfinite(ora), 0) & (ora.mean(0) < 5e3)
    se = np.sqrt(gpu[:, keep].var(0, ddof=1) / R + ora[:, keep].var(0, ddof=1) / R) + 1e-9
    z = (gpu[:, keep].mean(0) - ora[:, keep].mean(0)) / se
    assert keep.sum() > K // 2
    assert np.all(np.abs(z) < 4.5), np.abs(z).max()
    assert abs(z.mean()) < 4.0 / math.sqrt(keep.sum()) + 0.5


# ------------------------------------------------------------ K-sharding, determinism

def _c3_like(K=2048, M=256, T=50):
    from paper_2408_00494_b200.tracks import named_track as nt
    model = md.with_timestep(md.VehicleParams(), 0.04, "euler")
    cfg = mc.MppiConfig(kind="bss", samples=K, horizon=T, inner_samples=M,
                        sigma_eps=np.diag([0.2 ** 2, 0.5 ** 2]))
    return cfg, mc.CostSpec(), model, nt("spline0"), md.NoiseModel(np.diag([0.05 ** 2] * 3))


def test_shard_partials_combine_equals_single_context():
    """Two K-shards (run one after the other on this GPU, global-k Philox
    counters) combined from their partial records give the single-context
    v+ to FP64 rounding, and identical diagnostics."""
    cfg, cost, model, track, noise = _c3_like(K=1024, M=64, T=30)
    ctx = mc.RolloutContext(model, track, cost, noise=noise)
    x0 = md.VehicleState.rolling(5.0, model, s=20.0).as_array()
    plan = np.zeros((cfg.horizon, 2))
    kc, kb = _lib.key_arr((5, 6)), _lib.key_arr((7, 8))
    full = mc.Controller(cfg, cost, model, track, noise=noise)
    dev = full._device_ctx()
    v_full = np.empty((cfg.horizon, 2))
    d_full = _lib.Diag()
    _lib.check(dev.lib.bssmppi_control_step(dev.h, _lib.dptr(x0), None, _lib.dptr(plan), kc, kb, None, None,
                                            _lib.dptr(v_full), _lib.C.byref(d_full)))
    import torch
    R = _lib.load().bssmppi_partial_len(cfg.horizon)
    buf = torch.zeros((3, R), dtype=torch.float64, device="cuda")
    ctxs = []
    for slot, (b, n) in enumerate([(0, 300), (300, 500), (800, 224)]):
        prob, keep = mc.build_problem("bss", cfg.samples, cfg.horizon, cfg.inner_samples, cfg.temperature,
                                      cfg.control_cost_weight, cfg.sigma_eps, cfg.precision, cfg.bounds,
                                      False, ctx, b, n)
        dc = mc.DeviceContext(prob)
        _lib.check(dc.lib.bssmppi_step_partials(dc.h, _lib.dptr(x0), None, _lib.dptr(plan), kc, kb, None, None,
                                                _lib.C.c_void_p(buf.data_ptr()), slot))
        ctxs.append(dc)
    v = np.empty((cfg.horizon, 2))
    d = _lib.Diag()
    _lib.check(ctxs[0].lib.bssmppi_update_combine(ctxs[0].h, _lib.C.c_void_p(buf.data_ptr()), 3,
                                                  _lib.dptr(v), _lib.C.byref(d)))
    np.testing.assert_allclose(v, v_full, atol=1e-12)
    assert d.cost_argmin == d_full.cost_argmin and d.n_finite == d_full.n_finite
    assert d.cost_min == d_full.cost_min


def test_full_size_determinism_and_finiteness():
    """BASELINE C3 shape end to end (philox mode): reruns are bit-identical,
    costs finite, the plan stays inside the bounds."""
    cfg, cost, model, track, noise = _c3_like(K=16384, M=256, T=50)
    x0 = md.VehicleState.rolling(5.0, model, s=20.0).as_array()
    outs = []
    for _ in range(2):
        ctrl = mc.Controller(cfg, cost, model, track, noise=noise, seed=3, run_path=(5, 3))
        u0, plan = ctrl.control_step(x0)
        u1, plan = ctrl.control_step(x0)
        outs.append((u0, u1, ctrl.last_diagnostics))
    assert np.array_equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1])
    d = outs[0][2]
    assert d["n_finite"] > 0.99 * cfg.samples
    assert np.all(np.abs(plan.controls[:, 0]) <= 0.35) and np.all(np.abs(plan.controls[:, 1]) <= 1.0)


def test_sharded_controller_world1_nccl():
    """The ShardedController code path (partials -> NCCL all-reduce ->
    combine) on a 1-rank NCCL group equals the plain controller."""
    import os
    import torch
    import torch.distributed as dist
    from paper_2408_00494_b200.distributed import ShardedController
    if not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29533")
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda:0"))
    cfg, cost, model, track, noise = _c3_like(K=512, M=64, T=20)
    x0 = md.VehicleState.rolling(5.0, model, s=20.0).as_array()
    a = ShardedController(cfg, cost, model, track, noise=noise, seed=4)
    b = mc.Controller(cfg, cost, model, track, noise=noise, seed=4)
    for _ in range(3):
        ua, _ = a.control_step(x0)
        ub, _ = b.control_step(x0)
        np.testing.assert_allclose(ua, ub, atol=1e-12)
    dist.destroy_process_group()


def test_update_golden_batch_shapes():
    for j in range(4):
        costs, controls, lam = update_batch(j)
        v = mc.mppi_update(mc.RolloutBatch(controls, np.zeros_like(controls), costs), lam, mc.ControlBounds())
        np.testing.assert_allclose(v.controls, c_oracle.update(costs, controls, lam, [-0.35, -1], [0.35, 1]),
                                   atol=1e-12)


def test_step_device_matches_control_step(oval, model):
    """The device-buffer entry point (torch CUDA tensors in and out, no host
    round trip) reproduces control_step bit for bit for the same seed,
    run_path and iteration."""
    import torch
    cfg = mc.MppiConfig(kind="bss", samples=300, horizon=12, inner_samples=24,
                        sigma_eps=np.diag([0.2 ** 2, 0.5 ** 2]))
    noise = md.NoiseModel(np.diag([0.03 ** 2] * 3))
    x0 = md.VehicleState.rolling(4.0, model, s=7.0).as_array()
    host = mc.Controller(cfg, mc.CostSpec(), model, oval, noise=noise, seed=5, run_path=(5, 1))
    dev = mc.Controller(cfg, mc.CostSpec(), model, oval, noise=noise, seed=5, run_path=(5, 1))
    plan = np.zeros((cfg.horizon, 2))
    for _ in range(3):
        host.control_step(x0)
        state = torch.tensor(np.concatenate([x0, np.zeros(16), plan.ravel()]), dtype=torch.float32, device="cuda")
        out = dev.step_device(state)
        torch.cuda.synchronize()
        o = out.cpu().numpy()
        np.testing.assert_array_equal(o[:2 * cfg.horizon].reshape(-1, 2), host.last_diagnostics["vplus"])
        assert o[2 * cfg.horizon + 3] == host.last_diagnostics["n_finite"]
        plan = np.concatenate([o[2:2 * cfg.horizon].reshape(-1, 2), o[2 * cfg.horizon - 2:2 * cfg.horizon][None]])
    assert dev.iteration == host.iteration == 3
    with pytest.raises(ValueError):
        dev.step_device(torch.zeros(5, device="cuda"))
