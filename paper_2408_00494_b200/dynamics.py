"""Host-side vehicle / track / noise types for the B200 BSS-MPPI path.

These mirror the reference's public data types so that a caller can pass
either our instances or the reference's own (duck-typed: only attribute
names are read):

* ``VehicleParams``  -> reference ``dynamics.py:55-103``
* ``VehicleState``   -> ``dynamics.py:106-136``
* ``Track``          -> ``dynamics.py:152-196``
* ``make_test_track``/``save_track``/``load_track`` -> ``dynamics.py:209-273``
* ``NoiseModel``/``psd_factor`` -> ``dynamics.py:276-314``
* ``phys_vector``    -> ``_phys_vector`` ``dynamics.py:325-337`` (the 23
  scalars the device kernels consume, same order)

No numerics of the hot path live here: the per-particle dynamics run in the
sm_100a kernels of ``csrc/``.  ``step_array`` is the batched device step
(reference ``dynamics.py:550-573``) exposed through the C ABI.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field, replace

import numpy as np

G = 9.81

IDX_VX, IDX_VY, IDX_YAW_RATE, IDX_OMEGA_F, IDX_OMEGA_R, IDX_EPSI, IDX_EY, IDX_S = range(8)
STATE_DIM = 8
IDX_STEER, IDX_THROTTLE = 0, 1
CONTROL_DIM = 2
DEFAULT_NOISE_CHANNELS = (IDX_VX, IDX_VY, IDX_YAW_RATE)

# mu * m * g / 2 at mu = 0.7 for the 22 kg platform (reference dynamics.py:37-40).
_DEFAULT_PEAK = 0.7 * 22.0 * G / 2.0


class OpenLoop(ValueError):
    """Track segment list does not close the loop."""


class FactorizationFailure(ValueError):
    """Covariance is not positive semidefinite within tolerance."""


@dataclass(frozen=True)
class VehicleParams:
    """Single-track model parameters (reference dynamics.py:55-99)."""

    mass: float = 22.0
    inertia_z: float = 1.2
    lf: float = 0.25
    lr: float = 0.25
    wheel_radius: float = 0.095
    wheel_inertia: float = 0.25
    b_lat_front: float = 4.0
    c_lat_front: float = 1.3
    b_lat_rear: float = 4.0
    c_lat_rear: float = 1.3
    b_long_front: float = 2.0
    c_long_front: float = 1.3
    b_long_rear: float = 2.0
    c_long_rear: float = 1.3
    peak_fx_front: float = _DEFAULT_PEAK
    peak_fy_front: float = _DEFAULT_PEAK
    peak_fx_rear: float = _DEFAULT_PEAK
    peak_fy_rear: float = _DEFAULT_PEAK
    drive_gain: float = 8.0
    roll_resist: float = 0.015
    dt: float = 0.05
    integrator: str = "euler"
    v_floor: float = 0.3

    def __post_init__(self):
        for name in ("mass", "inertia_z", "lf", "lr", "wheel_radius", "wheel_inertia",
                     "peak_fx_front", "peak_fy_front", "peak_fx_rear", "peak_fy_rear",
                     "dt", "v_floor"):
            if getattr(self, name) <= 0.0:
                raise ValueError(f"VehicleParams.{name} must be > 0")
        if self.roll_resist < 0.0:
            raise ValueError("VehicleParams.roll_resist must be >= 0")
        if self.integrator not in ("euler", "rk4"):
            raise ValueError(f"unknown integrator {self.integrator!r}")

    @property
    def wheelbase(self):
        return self.lf + self.lr


def with_timestep(params, dt: float, integrator: str):
    return replace(params, dt=dt, integrator=integrator)


def phys_vector(p) -> np.ndarray:
    """The 23 packed parameter scalars, in the reference's order
    (``_phys_vector``, dynamics.py:325-337)."""
    wb = p.lf + p.lr
    return np.array([
        p.mass, p.inertia_z, p.lf, p.lr, p.wheel_radius, p.wheel_inertia,
        p.b_lat_front, p.c_lat_front, p.b_lat_rear, p.c_lat_rear,
        p.b_long_front, p.c_long_front, p.b_long_rear, p.c_long_rear,
        p.peak_fx_front, p.peak_fy_front, p.peak_fx_rear, p.peak_fy_rear,
        p.drive_gain, p.roll_resist, p.v_floor,
        p.mass * G * p.lr / wb,
        p.mass * G * p.lf / wb,
    ], dtype=np.float64)


@dataclass
class VehicleState:
    vx: float = 0.0
    vy: float = 0.0
    yaw_rate: float = 0.0
    omega_f: float = 0.0
    omega_r: float = 0.0
    e_psi: float = 0.0
    e_y: float = 0.0
    s: float = 0.0

    def as_array(self) -> np.ndarray:
        return np.array([self.vx, self.vy, self.yaw_rate, self.omega_f, self.omega_r,
                         self.e_psi, self.e_y, self.s], dtype=float)

    @classmethod
    def from_array(cls, x):
        return cls(*(float(v) for v in np.asarray(x, dtype=float)))

    @classmethod
    def rolling(cls, vx: float, params, **kwargs):
        """Moving at ``vx`` with wheel speeds matched to ground speed
        (reference dynamics.py:131-135)."""
        omega = vx / params.wheel_radius
        return cls(vx=vx, omega_f=omega, omega_r=omega, **kwargs)


def _loop_turn(s, kappa, length, closed):
    total = float(np.trapezoid(kappa, s))
    if closed:
        total += (length - s[-1]) * 0.5 * (kappa[-1] + kappa[0])
    return total


@dataclass(eq=False)
class Track:
    """Centerline as an (arc length, curvature) table; linear interpolation,
    closing segment [s_{n-1}, length) back to kappa_0 (reference
    dynamics.py:152-196, validation identical)."""

    s: np.ndarray
    kappa: np.ndarray
    half_width: float
    closed: bool = True
    length: float = 0.0

    def __post_init__(self):
        self.s = np.asarray(self.s, dtype=float)
        self.kappa = np.asarray(self.kappa, dtype=float)
        if self.s.ndim != 1 or self.s.shape != self.kappa.shape or self.s.size < 2:
            raise ValueError("track needs matching 1-d s/kappa arrays with >= 2 samples")
        if self.s[0] != 0.0 or np.any(np.diff(self.s) <= 0.0):
            raise ValueError("track s samples must start at 0 and be strictly increasing")
        if self.half_width <= 0.0:
            raise ValueError("track half_width must be > 0")
        if self.closed and self.length <= self.s[-1]:
            raise ValueError("closed track length must exceed the last sample position")
        if not self.closed and self.length < self.s[-1]:
            raise ValueError("track length shorter than sampled range")
        if self.closed:
            total = self.turn_integral()
            if abs(abs(total) - 2.0 * math.pi) > 1e-6:
                raise ValueError(f"closed track curvature integral {total:.9f} is not +-2*pi")

    def turn_integral(self) -> float:
        return _loop_turn(self.s, self.kappa, self.length, self.closed)

    def wrap(self, s):
        if self.closed:
            return np.mod(s, self.length)
        return np.clip(s, 0.0, self.length)


def curvature(track, s):
    """Host-side kappa(s) (reference dynamics.py:199-206); used only by host
    logic such as track generation checks, never by the rollout path."""
    sw = track.wrap(np.asarray(s, dtype=float))
    if track.closed:
        out = np.interp(sw, track.s, track.kappa, period=track.length)
    else:
        out = np.interp(sw, track.s, track.kappa)
    return out if np.ndim(s) else float(out)


def make_test_track(segments, half_width: float, spacing: float = 0.5) -> Track:
    """Closed track from (length, curvature) segments, densified at
    ``spacing`` and rescaled so the interpolant winds exactly +-2*pi
    (reference dynamics.py:209-246)."""
    segs = [(float(a), float(b)) for a, b in segments]
    if not segs:
        raise OpenLoop("empty segment list")
    if any(a <= 0.0 for a, _ in segs):
        raise OpenLoop("segment lengths must be > 0")
    turn = math.fsum(a * b for a, b in segs)
    if abs(abs(turn) - 2.0 * math.pi) > 1e-6:
        raise OpenLoop(f"segments do not close the loop: integral kappa ds = {turn:.9f}")
    s_list, k_list = [], []
    start = 0.0
    for seg_len, seg_k in segs:
        pieces = max(1, math.ceil(seg_len / spacing))
        s_list.extend(start + j * seg_len / pieces for j in range(pieces))
        k_list.extend([seg_k] * pieces)
        start += seg_len
    s_arr = np.array(s_list)
    k_arr = np.array(k_list, dtype=float)
    k_arr *= math.copysign(2.0 * math.pi, turn) / _loop_turn(s_arr, k_arr, start, True)
    return Track(s=s_arr, kappa=k_arr, half_width=float(half_width), closed=True,
                 length=start)


def save_track(track, path):
    """Text table, same format as the reference (dynamics.py:249-256)."""
    with open(path, "w") as fh:
        fh.write(f"# length={track.length!r} half_width={track.half_width!r} "
                 f"closed={1 if track.closed else 0}\n")
        for a, b in zip(track.s, track.kappa):
            fh.write(f"{float(a)!r} {float(b)!r}\n")


def load_track(path) -> Track:
    with open(path) as fh:
        header = fh.readline().strip()
        if not header.startswith("#"):
            raise ValueError(f"{path}: missing track header line")
        meta = dict(item.split("=", 1) for item in header[1:].split())
        rows = [line.split() for line in fh if line.strip()]
    data = np.array([[float(a), float(b)] for a, b in rows])
    return Track(s=data[:, 0], kappa=data[:, 1], half_width=float(meta["half_width"]),
                 closed=bool(int(meta["closed"])), length=float(meta["length"]))


def psd_factor(cov, tol: float = 1e-10) -> np.ndarray:
    """F with F F^T = cov via eigh, eigenvalues in [-tol, 0) clamped
    (reference dynamics.py:303-314).  The column order follows eigh, so the
    factor of a non-ascending diagonal is column-permuted; oracle-mode
    parity depends on using exactly this factor."""
    cov = np.asarray(cov, dtype=float)
    sym = 0.5 * (cov + cov.T)
    if not np.allclose(cov, cov.T, atol=tol, rtol=0.0):
        raise FactorizationFailure("covariance is not symmetric")
    if not np.any(sym):
        return np.zeros_like(sym)
    w, v = np.linalg.eigh(sym)
    if w.min() < -tol:
        raise FactorizationFailure(f"covariance has eigenvalue {w.min():.3e} < -{tol:g}")
    return v * np.sqrt(np.clip(w, 0.0, None))


@dataclass(eq=False)
class NoiseModel:
    """Additive Gaussian process noise on (vx, vy, yaw rate)
    (reference dynamics.py:276-300)."""

    cov: np.ndarray
    channels: tuple = DEFAULT_NOISE_CHANNELS
    kind: str = "gaussian"
    _factor: np.ndarray = field(default=None, repr=False, compare=False)

    def __post_init__(self):
        self.cov = np.atleast_2d(np.asarray(self.cov, dtype=float))
        if self.cov.shape != (len(self.channels), len(self.channels)):
            raise ValueError("noise covariance shape does not match channel count")
        if self.kind != "gaussian":
            raise ValueError(f"unsupported noise distribution {self.kind!r}")

    @property
    def factor(self):
        if self._factor is None:
            self._factor = psd_factor(self.cov)
        return self._factor

    @property
    def is_zero(self):
        return not np.any(self.cov)
