"""Config-4 extension host logic (beyond the reference): the centerline table
reproduces the reference's TrackFrame, obstacles are placed by seed, and the
extended C oracle's Laplace/slip noise degenerates exactly."""

import math

import numpy as np
import pytest

from helpers import GOLDEN, Inputs

from oracle import c_oracle
from paper_2408_00494_b200 import controllers as mc
from paper_2408_00494_b200.obstacles import (LaplaceSlipNoise, Obstacles, centerline_table,
                                             place_obstacles)
from paper_2408_00494_b200.tracks import named_track


@pytest.mark.parametrize("name", ["ellipse", "spline0", "oval"])
def test_centerline_table_matches_reference_trackframe(name):
    d = np.load(GOLDEN / "trackframe.npz")
    tr = named_track(name)
    tab, ds = centerline_table(tr)
    q = d[name + "_s"]
    i = np.floor(q / ds).astype(int)
    f = q / ds - i
    lerp = tab[i] * (1 - f)[:, None] + tab[i + 1] * f[:, None]
    assert np.abs(lerp - d[name + "_pose"]).max() < 2e-4
    # global point at e_y = 0.7 (TrackFrame.to_global): centerline + e_y n(theta)
    g = d[name + "_global_ey0.7"]
    p = lerp[::10]
    xy = np.stack([p[:, 0] - 0.7 * np.sin(p[:, 2]), p[:, 1] + 0.7 * np.cos(p[:, 2])], 1)
    assert np.abs(xy - g[:, :2]).max() < 3e-4


def test_place_obstacles_seeded_and_on_track():
    tr = named_track("spline0")
    a, b = place_obstacles(tr, 16, seed=3), place_obstacles(tr, 16, seed=3)
    assert np.array_equal(a.xy, b.xy) and len(a.radius) == 16
    assert np.all((a.radius >= 0.5) & (a.radius <= 1.5))
    assert a.backoff == pytest.approx(2.0537489106318225, abs=1e-12)
    tab, _ = centerline_table(tr)
    dist = np.min(np.hypot(tab[:, None, 0] - a.xy[None, :, 0], tab[:, None, 1] - a.xy[None, :, 1]), axis=0)
    assert np.all(dist <= tr.half_width + 1e-9)                        # centres inside the lane
    with pytest.raises(ValueError):
        Obstacles(np.zeros((2, 2)), np.array([1.0, -1.0]))


def _problem(inp, noise=None, obstacles=None):
    ctx = mc.RolloutContext(inp.model, inp.track, inp.cost, noise=noise or inp.noise, obstacles=obstacles)
    cfg = inp.cfg
    return mc.build_problem("bss", inp.K, inp.T, inp.M, cfg.temperature, cfg.control_cost_weight,
                            cfg.sigma_eps, cfg.precision, cfg.bounds, False, ctx)


def test_laplace_zero_scale_equals_noise_free():
    """Laplace/slip with zero scale adds exactly 0 and uses the same
    re-projection normals: the costs equal the noise-free Gaussian ones."""
    from paper_2408_00494_b200 import dynamics as md
    inp = Inputs("c1_s0")
    zero = md.NoiseModel(np.zeros((3, 3)))
    p0, k0 = _problem(inp, noise=zero)
    p1, k1 = _problem(inp, noise=LaplaceSlipNoise(0.0, 0.0))
    a, _ = c_oracle.rollout(p0, inp.x0, inp.cov0, inp.plan, u=inp.u, eps=inp.eps, key_belief=(3, 4))
    b, _ = c_oracle.rollout(p1, inp.x0, inp.cov0, inp.plan, u=inp.u, eps=inp.eps, key_belief=(3, 4))
    np.testing.assert_array_equal(a, b)


def test_far_obstacles_change_nothing_and_near_ones_cost():
    inp = Inputs("c1_s0")
    base, kb = _problem(inp)
    far, kf = _problem(inp, obstacles=Obstacles(np.array([[1e4, 1e4]]), np.array([1.0])))
    a, _ = c_oracle.rollout(base, inp.x0, inp.cov0, inp.plan, u=inp.u, eps=inp.eps, key_belief=(3, 4))
    b, _ = c_oracle.rollout(far, inp.x0, inp.cov0, inp.plan, u=inp.u, eps=inp.eps, key_belief=(3, 4))
    np.testing.assert_array_equal(a, b)
    # an obstacle on the centerline just ahead of x0 raises every finite cost
    tab, ds = centerline_table(inp.track)
    s_ahead = (inp.x0[7] + 4.0) % inp.track.length
    row = tab[int(s_ahead / ds)]
    near, kn = _problem(inp, obstacles=Obstacles(row[None, :2], np.array([0.8])))
    c, _ = c_oracle.rollout(near, inp.x0, inp.cov0, inp.plan, u=inp.u, eps=inp.eps, key_belief=(3, 4))
    fin = np.isfinite(a) & np.isfinite(c)
    assert np.all(c[fin] >= a[fin]) and np.mean(c[fin] > a[fin]) > 0.5
