"""Host-side logic of the B200 path (no GPU): config validation mirroring the
reference, problem packing, track tables, keyed device streams, the
reduce-scatter schedule of the rollout kernel, K-shard partitioning."""

import math

import numpy as np
import pytest

from paper_2408_00494_b200 import controllers as mc
from paper_2408_00494_b200 import dynamics as md
from paper_2408_00494_b200 import streams
from paper_2408_00494_b200.belief import DEFAULT_SUBSET, CovSubset
from paper_2408_00494_b200.constraints import SafetyParams, allocate_budget, backoff_gaussian
from paper_2408_00494_b200.distributed import partial_len, shard_range
from paper_2408_00494_b200.tracks import ellipse_track, named_track, spline_track


class TestConfigValidation:
    """Same ValueErrors as reference controllers.py:85-105, 119-133."""

    def test_bad_kind(self):
        with pytest.raises(ValueError):
            mc.MppiConfig(kind="nope")

    def test_bss_needs_two_inner_samples(self):
        with pytest.raises(ValueError):
            mc.MppiConfig(kind="bss", inner_samples=1)

    def test_temperature(self):
        with pytest.raises(ValueError):
            mc.MppiConfig(temperature=0.0)

    def test_sigma_pair_and_precision(self):
        cfg = mc.MppiConfig(sigma_eps=np.array([0.04, 0.25]))
        assert np.allclose(cfg.sigma_eps, np.diag([0.04, 0.25]))
        assert np.allclose(cfg.precision, np.diag([25.0, 4.0]))

    def test_cost_defaults(self):
        c = mc.CostSpec()
        assert c.backoff == pytest.approx(1.9599639845400538, abs=1e-12)
        assert c.q_diag.tolist() == [6.0, 0.0, 0.02, 0.0, 0.0, 0.2, 0.1, 0.0]
        with pytest.raises(ValueError):
            mc.CostSpec(q_diag=-np.ones(8))

    def test_safety_params(self):
        with pytest.raises(ValueError):
            SafetyParams(cbf_rate=1.0)
        assert allocate_budget(0.05, 2) == [0.025, 0.025]
        assert backoff_gaussian(0.01) == pytest.approx(2.3263478740408408, abs=1e-9)

    def test_bounds(self):
        with pytest.raises(ValueError):
            mc.ControlBounds(delta_max=0.0)

    def test_plan_shift(self):
        p = mc.ControlPlan(np.arange(6.0).reshape(3, 2)).shifted()
        assert p.controls.tolist() == [[2, 3], [4, 5], [4, 5]]

    def test_unsupported_subset_and_hook(self):
        cfg = mc.MppiConfig()
        track = named_track("oval")
        with pytest.raises(NotImplementedError):
            mc.Controller(cfg, mc.CostSpec(), md.VehicleParams(), track, subset=CovSubset((0, 1)))
        cost = mc.CostSpec()
        cost.belief_stage_cost = lambda m, s: 0 * s
        with pytest.raises(NotImplementedError):
            mc.Controller(cfg, cost, md.VehicleParams(), track)


class TestProblemPacking:
    def test_fields(self):
        track = named_track("ellipse")
        ctx = mc.RolloutContext(md.with_timestep(md.VehicleParams(), 0.04, "euler"), track,
                                mc.CostSpec(), noise=md.NoiseModel(np.diag([0.01, 0.02, 0.03])))
        cfg = mc.MppiConfig(samples=100, horizon=7, inner_samples=9)
        p, keep = mc.build_problem("bss", 100, 7, 9, 1.0, 0.1, cfg.sigma_eps, cfg.precision,
                                   cfg.bounds, False, ctx, 10, 40)
        assert (p.kind, p.samples, p.horizon, p.inner_samples, p.k_begin, p.k_count) == (2, 100, 7, 9, 10, 40)
        assert p.dt == 0.04 and p.track_n == 256 and p.track_closed == 1
        assert list(p.phys) == md.phys_vector(ctx.model).tolist()
        F = np.array(list(p.noise_factor)).reshape(3, 3)
        assert np.allclose(F @ F.T, np.diag([0.01, 0.02, 0.03]))
        assert list(p.bounds_lo) == [-0.35, -1.0] and list(p.bounds_hi) == [0.35, 1.0]

    def test_permuted_sigma_factor(self):
        # eigh ordering permutes the factor's columns
        f = md.psd_factor(np.diag([0.5 ** 2, 0.2 ** 2]))
        assert np.allclose(np.abs(f), [[0, 0.5], [0.2, 0]])


class TestTracks:
    def test_ellipse(self):
        t = ellipse_track()
        assert t.s.size == 256 and t.length == pytest.approx(102.108, abs=1e-3)
        assert abs(t.turn_integral() - 2 * math.pi) < 1e-9

    @pytest.mark.parametrize("seed", range(4))
    def test_spline_feasible(self, seed):
        t = spline_track(seed)
        assert np.abs(t.kappa).max() * (t.half_width + 0.5) < 1.0
        assert abs(t.turn_integral() - 2 * math.pi) < 1e-9
        assert 120 < t.length < 160

    def test_round_trip(self, tmp_path):
        t = named_track("spline1")
        md.save_track(t, tmp_path / "t.track")
        u = md.load_track(tmp_path / "t.track")
        assert np.array_equal(u.s, t.s) and np.array_equal(u.kappa, t.kappa)
        assert u.length == t.length

    def test_open_loop_rejected(self):
        with pytest.raises(md.OpenLoop):
            md.make_test_track([(10.0, 0.0), (5.0, 0.1)], half_width=2.0)


class TestStreams:
    def test_device_key_deterministic_and_distinct(self):
        a = streams.device_key(0, 5, 0, 2, 7)
        assert a == streams.device_key(0, 5, 0, 2, 7)
        assert a != streams.device_key(0, 5, 0, 3, 7)
        assert a != streams.device_key(0, 5, 0, 2, 8)
        assert all(0 <= v < 2 ** 32 for v in a)

    def test_reference_substream(self):
        x = streams.substream(3, 1, 2).standard_normal(4)
        y = np.random.Generator(np.random.Philox(
            np.random.SeedSequence(3, spawn_key=(1, 2)))).standard_normal(4)
        assert np.array_equal(x, y)


def _simulate_reduce_scatter(G, vals):
    levels = {32: [(18, 16), (9, 8), (5, 4), (3, 2), (2, 1)], 16: [(18, 8), (9, 4), (5, 2), (3, 1)],
              8: [(18, 4), (9, 2), (5, 1)], 4: [(18, 2), (9, 1)], 2: [(18, 1)]}[G]
    a = [list(v) for v in vals]
    base, cnt = [0] * G, [18] * G
    for N, OFF in levels:
        H = (N + 1) // 2
        new = []
        for lane in range(G):
            up, p = bool(lane & OFF), lane ^ OFF
            out = []
            for i in range(H):
                mine = a[lane][i + H] if (up and i + H < N) else (0.0 if up else a[lane][i])
                theirs = a[p][i + H] if (up and i + H < N) else (0.0 if up else a[p][i])
                out.append(mine + theirs)
            new.append(out)
        for lane in range(G):
            up = bool(lane & OFF)
            base[lane] += H if up else 0
            cnt[lane] = max(cnt[lane] - H, 0) if up else min(cnt[lane], H)
        a = new
    slot = [None] * 18
    for lane in range(G):
        for i in range(len(a[lane])):
            if i < cnt[lane]:
                assert slot[base[lane] + i] is None
                slot[base[lane] + i] = a[lane][i]
    return slot


@pytest.mark.parametrize("G", [2, 4, 8, 16, 32])
def test_reduce_scatter_schedule_covers_every_sum_once(G):
    """Host model of group_allreduce18 (csrc/rollout.cuh): every one of the
    18 moment sums is written by exactly one lane and equals the group sum."""
    vals = np.random.default_rng(G).normal(size=(G, 18))
    slot = _simulate_reduce_scatter(G, vals)
    assert np.allclose(slot, vals.sum(0))


def _simulate_reduce_scatter16(G, vals):
    # group_allreduce16: exact halvings, G = 32 ends with a pairwise add
    levels = {32: [(16, 16), (8, 8), (4, 4), (2, 2)], 16: [(16, 8), (8, 4), (4, 2), (2, 1)],
              8: [(16, 4), (8, 2), (4, 1)], 4: [(16, 2), (8, 1)], 2: [(16, 1)]}[G]
    a = [list(v) for v in vals]
    base = [0] * G
    for N, OFF in levels:
        H = N // 2
        new = []
        for lane in range(G):
            up, p = bool(lane & OFF), lane ^ OFF
            keep = a[lane][H:N] if up else a[lane][:H]
            recv = a[p][H:N] if up else a[p][:H]       # what the partner sends
            new.append([k + r for k, r in zip(keep, recv)])
        for lane in range(G):
            base[lane] += H if lane & OFF else 0
        a = new
    if G == 32:
        a = [[a[lane][0] + a[lane ^ 1][0]] for lane in range(G)]
    slot = [None] * 16
    for lane in range(G):
        if G == 32 and lane & 1:
            continue
        for i, v in enumerate(a[lane]):
            assert slot[base[lane] + i] is None
            slot[base[lane] + i] = v
    return slot


@pytest.mark.parametrize("G", [2, 4, 8, 16, 32])
def test_reduce_scatter16_schedule_covers_every_sum_once(G):
    """Host model of group_allreduce16 (csrc/rollout.cuh, the re-projection
    path's 16 nonzero sums): every sum is written by exactly one lane and
    equals the group sum."""
    vals = np.random.default_rng(100 + G).normal(size=(G, 16))
    slot = _simulate_reduce_scatter16(G, vals)
    assert np.allclose(slot, vals.sum(0))


class TestSharding:
    def test_partition(self):
        for K, W in [(16384, 8), (100, 3), (7, 7), (16384, 1)]:
            ranges = [shard_range(K, r, W) for r in range(W)]
            assert ranges[0][0] == 0
            assert sum(c for _, c in ranges) == K
            for (b0, c0), (b1, _) in zip(ranges, ranges[1:]):
                assert b0 + c0 == b1
            assert max(c for _, c in ranges) - min(c for _, c in ranges) <= 1

    def test_errors(self):
        with pytest.raises(ValueError):
            shard_range(4, 0, 8)
        with pytest.raises(ValueError):
            shard_range(4, 2, 2)

    def test_record_length(self):
        assert partial_len(50) == 105


def test_default_subset():
    assert DEFAULT_SUBSET.indices == (1, 2, 5, 6)
    assert DEFAULT_SUBSET.position(6) == 3


def test_group_width_policy():
    """Lanes per rollout (csrc/bssmppi.cu group_width): one warp for small
    problems; >= 8 particles per lane while >= 1024 warps remain, >= 16 while
    >= 1400 remain, then up to 64 per lane while >= 4096 warps remain -- the measured best G on every
    swept shape (profiles/r1_group_width_sweep.txt)."""
    from paper_2408_00494_b200 import _lib
    gw = _lib.load().bssmppi_group_width
    assert gw(32, 256) == 32 and gw(5, 40) == 8 and gw(2, 16) == 2
    assert gw(256, 16384) == 8          # C3 on one GPU
    assert gw(256, 8192) == 16          # C3 shard at 2 GPUs
    assert gw(256, 2048) == 32          # C3 shard at 8 GPUs
    assert gw(256, 4096) == 16          # C3 shard at 4 GPUs: 16 particles per lane, 2048 warps
    assert gw(256, 3000) == 16 and gw(128, 8192) == 8 and gw(64, 16384) == 4 and gw(64, 12000) == 4
    assert gw(64, 8192) == 8            # C4 shard at 8 GPUs: 1024 warps at G = 4 are too few
    assert gw(256, 32768) == 4          # 64 particles per lane
    assert gw(64, 32768) == 4           # C5 32768 x 64
    assert gw(64, 4096) == 8            # C5 4096 x 64: 8 particles per lane
    assert gw(128, 4096) == 16          # C2
    assert gw(512, 4096) == 32 and gw(512, 32768) == 8
    assert gw(64, 65536) == 2           # C4, C5 65536+ x 64: 32 particles per lane
    assert gw(64, 131072) == 2 and gw(256, 131072) == 4 and gw(512, 131072) == 8
