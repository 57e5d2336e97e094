"""BASELINE config 4 extensions -- BEYOND the reference package.

The reference implements neither non-Gaussian process noise (its
``NoiseModel`` rejects any kind but "gaussian", dynamics.py:289-290) nor
obstacle constraints in the rollouts (they hard-code the track DCBF,
controllers.py:293, 315-317).  BASELINE config 4 asks for both; they are
built here on the reference's own machinery and pinned to the extended C
oracle (oracle/bss_oracle.c), not to the reference (parity unpinned with
respect to the reference):

* ``LaplaceSlipNoise``: process noise Laplace(0, b) on (vx, vy, yaw rate)
  plus a uniform lateral-slip term U(-a, a) on vy, added after integration
  like the reference's Gaussian noise (dynamics.py:571-572);
* ``Obstacles``: circular obstacles (x, y, radius) in the global frame, each
  a chance constraint c_i(x) = radius_i - ||p(s, e_y) - o_i|| < 0 with the
  reference's tightened margin (``heuristic_h_i``, constraints.py:112-120)
  h_i = -c_i(mean) - nu sqrt(eta^T Sigma eta), eta = grad c_i on the tracked
  subset (only e_y of (vy, r, e_psi, e_y) moves p, so
  sqrt(eta^T Sigma eta) = |dc_i/de_y| sigma_y); the rollout charges the
  discrete safety condition on h_obs = min_i h_i with the same Shield-MPPI
  penalty as the track DCBF, and C_obs for a belief mean inside an obstacle;
* ``centerline_table``: global centerline poses at uniform arc length,
  integrated like the reference's ``TrackFrame`` (dynamics.py:592-646:
  exact heading integral of the piecewise-linear curvature, 12-point
  Gauss-Legendre quadrature of (cos, sin)).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .constraints import backoff_gaussian

_GL_NODES, _GL_WEIGHTS = np.polynomial.legendre.leggauss(12)


@dataclass(frozen=True)
class LaplaceSlipNoise:
    """Laplace(0, scale) on (vx, vy, r) + U(-slip_bias, slip_bias) on vy."""

    scale: float = 0.03
    slip_bias: float = 0.05
    channels: tuple = (0, 1, 2)
    kind: str = "laplace_slip"

    def __post_init__(self):
        if self.scale < 0.0 or self.slip_bias < 0.0:
            raise ValueError("scale and slip_bias must be >= 0")

    @property
    def factor(self):          # Gaussian factor of the reference interface: unused
        return np.zeros((3, 3))

    @property
    def cov(self):             # equivalent per-channel variance (2 b^2, + a^2/3 on vy)
        v = 2.0 * self.scale ** 2
        return np.diag([v, v + self.slip_bias ** 2 / 3.0, v])


@dataclass(frozen=True)
class Obstacles:
    """Circular obstacles; ``delta`` is each one's failure probability."""

    xy: np.ndarray        # (n, 2)
    radius: np.ndarray    # (n,)
    delta: float = 0.02

    def __post_init__(self):
        xy = np.asarray(self.xy, dtype=float).reshape(-1, 2)
        r = np.asarray(self.radius, dtype=float).reshape(-1)
        if xy.shape[0] != r.shape[0] or np.any(r <= 0.0):
            raise ValueError("need one positive radius per obstacle centre")
        if not 0.0 < self.delta <= 0.5:
            raise ValueError("delta must lie in (0, 0.5]")
        if xy.shape[0] > 64:
            raise ValueError("at most 64 obstacles on the device path")
        object.__setattr__(self, "xy", xy)
        object.__setattr__(self, "radius", r)

    @property
    def backoff(self):
        return backoff_gaussian(self.delta)

    def as_array(self):
        return np.concatenate([self.xy, self.radius[:, None]], axis=1)


def node_poses(track, extend=False):
    """Centerline (x, y, theta) at the track nodes (+ the closing node),
    TrackFrame's construction (reference dynamics.py:603-646).  ``extend``
    continues a closed track one segment past s = L (for uniform tables)."""
    s, kap = np.asarray(track.s, float), np.asarray(track.kappa, float)
    if track.closed:
        s = np.append(s, track.length)
        kap = np.append(kap, track.kappa[0])
        if extend:
            s = np.append(s, track.length + track.s[1])
            kap = np.append(kap, track.kappa[1])
    theta = np.concatenate([[0.0], np.cumsum(np.diff(s) * 0.5 * (kap[:-1] + kap[1:]))])
    xs, ys = [0.0], [0.0]
    for j in range(len(s) - 1):
        dx, dy = _segment_quad(s, kap, theta, j, s[j + 1])
        xs.append(xs[-1] + dx)
        ys.append(ys[-1] + dy)
    return s, kap, theta, np.array(xs), np.array(ys)


def _segment_quad(s, kap, theta, j, s_to):
    s0 = s[j]
    h = s[j + 1] - s0
    half = 0.5 * (s_to - s0)
    d = half * (_GL_NODES + 1.0)
    slope = (kap[j + 1] - kap[j]) / h
    th = theta[j] + kap[j] * d + 0.5 * slope * d * d
    w = _GL_WEIGHTS * half
    return float(np.dot(w, np.cos(th))), float(np.dot(w, np.sin(th)))


def centerline_table(track, ds: float = 0.05):
    """Poses (x, y, theta) at s = i * ds, i = 0..n-1 (n = ceil(L/ds) + 1),
    evaluated exactly within each curvature segment; the device
    interpolates linearly between rows (error ~ kappa ds^2 / 8 < 1e-4 m)."""
    s, kap, theta, xs, ys = node_poses(track, extend=True)
    n = int(math.ceil(track.length / ds)) + 1
    out = np.empty((n, 3))
    for i in range(n):
        q = i * ds if track.closed else min(i * ds, track.length)
        j = int(np.searchsorted(s, q, side="right") - 1)
        j = min(max(j, 0), len(s) - 2)
        dx, dy = _segment_quad(s, kap, theta, j, q)
        d = q - s[j]
        slope = (kap[j + 1] - kap[j]) / (s[j + 1] - s[j])
        out[i] = (xs[j] + dx, ys[j] + dy, theta[j] + kap[j] * d + 0.5 * slope * d * d)
    return out, ds


def place_obstacles(track, n: int = 16, seed: int = 0, r_range=(0.5, 1.5), delta: float = 0.02,
                    keep_clear: float = 15.0):
    """``n`` circular obstacles placed by seed along the track: evenly spaced
    arc-length slots (jittered) beyond ``keep_clear`` m from s = 0, radius
    ~ U(r_range), centre offset laterally so at least 0.6 m of the lane stays
    free on one side (BASELINE config 4)."""
    rng = np.random.default_rng(seed)
    s_nodes, kap, theta, xs, ys = node_poses(track)
    usable = track.length - keep_clear
    slots = keep_clear + (np.arange(n) + rng.uniform(0.2, 0.8, n)) * usable / n
    radius = rng.uniform(r_range[0], r_range[1], n)
    side = rng.choice([-1.0, 1.0], n)
    w = track.half_width
    xy = np.empty((n, 2))
    table, ds = centerline_table(track)
    for i in range(n):
        ey = side[i] * max(w - 0.6 - radius[i], 0.0) * rng.uniform(0.3, 1.0) + side[i] * radius[i] * 0.5
        ey = float(np.clip(ey, -w, w))
        row = table[min(int(round(slots[i] / ds)), len(table) - 1)]
        xy[i] = (row[0] - ey * math.sin(row[2]), row[1] + ey * math.cos(row[2]))
    return Obstacles(xy, radius, delta)
