"""Benchmark track tables.

The reference only knows tracks as (s, kappa) tables built from
constant-curvature segments (``make_test_track``, reference
dynamics.py:209-246).  The BASELINE configs name an ellipse and a seeded
random closed spline; both are expressed here as segment lists and pushed
through ``make_test_track`` so that the oracle and the device read the
identical table (``save_track`` writes the shared bytes).
"""

from __future__ import annotations

import math

import numpy as np

from .dynamics import make_test_track


def stadium_track(straight: float = 20.0, radius: float = 6.0, half_width: float = 2.0):
    """The reference's default circuit (sim.py:52-60)."""
    return make_test_track(oval_segments(straight, radius), half_width=half_width)


def _closing_segments(arc_len, kappa):
    """Equal-arc segments with curvature renormalised to wind exactly 2*pi."""
    lengths = np.full(kappa.shape, arc_len)
    kappa = kappa * (2.0 * math.pi / float(np.sum(kappa * lengths)))
    return list(zip(lengths.tolist(), kappa.tolist()))


def ellipse_segments(a: float = 20.0, b: float = 12.0, segments: int = 256):
    """20 m x 12 m ellipse (config C1/C2): equal-arc segments with the
    curvature ab / ((a sin th)^2 + (b cos th)^2)^1.5 taken at mid-arc."""
    th = np.linspace(0.0, 2.0 * math.pi, 200001)
    speed = np.hypot(a * np.sin(th), b * np.cos(th))
    arc = np.concatenate([[0.0], np.cumsum(0.5 * (speed[1:] + speed[:-1]) * np.diff(th))])
    total = arc[-1]
    seg = total / segments
    mid_s = (np.arange(segments) + 0.5) * seg
    th_mid = np.interp(mid_s, arc, th)
    kappa = a * b / ((a * np.sin(th_mid)) ** 2 + (b * np.cos(th_mid)) ** 2) ** 1.5
    return _closing_segments(seg, kappa)


def ellipse_track(a: float = 20.0, b: float = 12.0, half_width: float = 1.5,
                  segments: int = 256, build=make_test_track):
    return build(ellipse_segments(a, b, segments), half_width=half_width)


def _spline_attempt(rng, box=(60.0, 40.0), points=12):
    from scipy.interpolate import CubicSpline

    ang = 2.0 * math.pi * np.arange(points) / points + rng.uniform(-0.15, 0.15, points)
    rx = 0.5 * box[0] * rng.uniform(0.6, 1.0, points)
    ry = 0.5 * box[1] * rng.uniform(0.6, 1.0, points)
    px = 0.5 * box[0] + rx * np.cos(ang)
    py = 0.5 * box[1] + ry * np.sin(ang)
    px = np.append(px, px[0])
    py = np.append(py, py[0])
    chord = np.concatenate([[0.0], np.cumsum(np.hypot(np.diff(px), np.diff(py)))])
    cs = CubicSpline(chord, np.stack([px, py], axis=1), bc_type="periodic")
    u = np.linspace(0.0, chord[-1], 20001)
    d1 = cs(u, 1)
    d2 = cs(u, 2)
    speed = np.hypot(d1[:, 0], d1[:, 1])
    kap = (d1[:, 0] * d2[:, 1] - d1[:, 1] * d2[:, 0]) / speed ** 3
    arc = np.concatenate([[0.0], np.cumsum(0.5 * (speed[1:] + speed[:-1]) * np.diff(u))])
    return arc, kap


def spline_segments(seed: int = 0, half_width: float = 2.0, spacing: float = 0.5,
                    max_attempts: int = 64):
    """Seeded random closed spline through 12 star-ordered points in a
    60 m x 40 m box (configs C3/C5).  Star ordering keeps it simple; seeds
    whose tightest corner violates max|kappa| (w + 0.5) < 1 are redrawn
    with seed + 1000 * attempt."""
    for attempt in range(max_attempts):
        rng = np.random.default_rng(seed + 1000 * attempt)
        arc, kap = _spline_attempt(rng)
        if np.max(np.abs(kap)) * (half_width + 0.5) >= 1.0:
            continue
        total = arc[-1]
        n = int(math.ceil(total / spacing))
        seg = total / n
        mid = (np.arange(n) + 0.5) * seg
        k_mid = np.interp(mid, arc, kap)
        return _closing_segments(seg, k_mid)
    raise RuntimeError(f"no feasible spline track for seed {seed}")


def spline_track(seed: int = 0, half_width: float = 2.0, spacing: float = 0.5,
                 build=make_test_track):
    return build(spline_segments(seed, half_width, spacing), half_width=half_width,
                 spacing=spacing)


def oval_segments(straight: float = 20.0, radius: float = 6.0):
    arc = math.pi * radius
    return [(straight, 0.0), (arc, 1.0 / radius), (straight, 0.0), (arc, 1.0 / radius)]


def named_track(name: str, build=make_test_track):
    """'ellipse' (C1/C2), 'oval' (reference test fixture, w=2),
    'stadium' (reference default experiment), 'splineN' (C3/C5, seed N)."""
    if name == "ellipse":
        return ellipse_track(build=build)
    if name in ("oval", "stadium"):
        return build(oval_segments(), half_width=2.0)
    if name.startswith("spline"):
        return spline_track(int(name[6:] or 0), build=build)
    raise ValueError(f"unknown track {name!r}")
