"""Closed-loop driver around the device controller (BASELINE
config 2).

Mirrors the reference harness ``belief_mppi.sim.run_closed_loop``
(sim.py:232-309): the controller replans every ``dt_control`` on the device
(``Controller.control_step``), the plant integrates the FULL model with RK4 at
``dt_plant`` on the host in FP64 -- deliberately finer than the controller's
Euler model, exactly like the reference -- and process noise enters once per
control period on the last substep.  Initial-state jitter and plant noise
are drawn from the reference's own keyed streams, so a run with
``noise_source="reference"`` follows the reference trajectory step for step
until FP32-vs-FP64 differences grow (tests/test_gpu_closed_loop.py).

The plant is the simulator, not the optimisation step: it stays on the host
as in the reference (``dynamics.py:447-478`` RK4 branch of ``_step_kernel``).
The realised-safety bookkeeping (``SafetyMonitor``, reference sim.py:157-220)
re-propagates the window's belief through the device rollout kernel.
"""

from __future__ import annotations

import math
import time
from collections import deque
from dataclasses import dataclass, field, replace

import numpy as np

from . import _lib, streams
from .belief import DEFAULT_SUBSET
from .controllers import Controller, ControlBounds, CostSpec, DeviceContext, MppiConfig, RolloutContext, \
    build_problem
from .dynamics import IDX_EY, IDX_S, NoiseModel, VehicleParams, VehicleState, phys_vector
from .tracks import stadium_track


# ------------------------------------------------------------------ plant (FP64, host)

def _curvature(track, s):
    sw = np.mod(s, track.length) if track.closed else np.clip(s, 0.0, track.length)
    if track.closed:
        return np.interp(sw, track.s, track.kappa, period=track.length)
    return np.interp(sw, track.s, track.kappa)


def _derivs(x, u, p, track):
    """Single-track Pacejka derivatives (reference dynamics.py:372-437), FP64."""
    vx, vy, r, wf, wr, e_psi, e_y, s = x
    vx_eff = max(vx, p[20]) if vx >= 0.0 else min(vx, -p[20])
    den = abs(vx_eff)
    a_f = u[0] - math.atan2(vy + p[2] * r, vx_eff)
    a_r = -math.atan2(vy - p[3] * r, vx_eff)
    sf = (wf * p[4] - vx) / den
    sr = (wr * p[4] - vx) / den
    fyf0 = p[15] * math.sin(p[7] * math.atan(p[6] * a_f))
    fyr0 = p[17] * math.sin(p[9] * math.atan(p[8] * a_r))
    fxf = p[14] * math.sin(p[11] * math.atan(p[10] * sf))
    fxr = p[16] * math.sin(p[13] * math.atan(p[12] * sr))
    fyf = fyf0 * math.sqrt(max(1.0 - (fxf / p[14]) ** 2, 0.0))
    fyr = fyr0 * math.sqrt(max(1.0 - (fxr / p[16]) ** 2, 0.0))
    cd, sd = math.cos(u[0]), math.sin(u[0])
    fxb, fyb = fxf * cd - fyf * sd, fxf * sd + fyf * cd
    kap = float(_curvature(track, s))
    frame = 1.0 - kap * e_y
    ok = frame > 0.0
    frame = max(frame, 1e-3)
    ce, se = math.cos(e_psi), math.sin(e_psi)
    ds = (vx * ce - vy * se) / frame
    return np.array([
        (fxb + fxr) / p[0] + vy * r,
        (fyb + fyr) / p[0] - vx * r,
        (p[2] * fyb - p[3] * fyr) / p[1],
        (-p[4] * fxf - p[19] * p[21] * p[4] * math.tanh(wf * p[4] / 0.1)) / p[5],
        (p[18] * u[1] - p[4] * fxr - p[19] * p[22] * p[4] * math.tanh(wr * p[4] / 0.1)) / p[5],
        r - kap * ds,
        vx * se + vy * ce,
        ds,
    ]), ok


def plant_step(x, u, w, params, track, channels=(0, 1, 2)):
    """One RK4 plant step over params.dt; noise added after integration
    (reference step_array, dynamics.py:550-573).  Returns (x', frame_ok)."""
    p = phys_vector(params)
    dt = params.dt
    x = np.asarray(x, dtype=float)
    k1, g1 = _derivs(x, u, p, track)
    k2, g2 = _derivs(x + 0.5 * dt * k1, u, p, track)
    k3, g3 = _derivs(x + 0.5 * dt * k2, u, p, track)
    k4, g4 = _derivs(x + dt * k3, u, p, track)
    out = x + (dt / 6.0) * (k1 + 2.0 * k2 + 2.0 * k3 + k4)
    out[5] = math.pi - (math.pi - out[5]) % (2.0 * math.pi)
    out[7] = out[7] % track.length if track.closed else min(max(out[7], 0.0), track.length)
    ok = g1 and g2 and g3 and g4
    bad = ~np.isfinite(out)
    if bad.any():
        ok = False
        out[bad] = 0.0
    if w is not None and np.any(w):
        out[list(channels)] += w
    return out, bool(ok)


# ------------------------------------------------------------------ experiment

@dataclass(eq=False)
class ExperimentConfig:
    """Subset of the reference ExperimentConfig (sim.py:63-123) that the
    closed loop needs."""

    controller: MppiConfig = field(default_factory=MppiConfig)
    cost: CostSpec = field(default_factory=CostSpec)
    vehicle: VehicleParams = field(default_factory=VehicleParams)
    track: object = field(default_factory=stadium_track)
    noise: NoiseModel = None
    dt_control: float = 0.05
    dt_plant: float = 0.01
    master_seed: int = 0
    laps: int = 1
    collision_threshold: float = 1.8
    max_steps: int = 1200
    init_speed: float = 2.0
    init_jitter: float = 0.1
    monitor_window: int = 0   # 0 -> half the controller horizon (reference sim.py:86)

    def __post_init__(self):
        if self.noise is None:
            self.noise = NoiseModel(np.diag([0.15 ** 2, 0.15 ** 2, 0.3 ** 2]))
        sub = self.dt_control / self.dt_plant
        if abs(sub - round(sub)) > 1e-9 or round(sub) < 1:
            raise ValueError("dt_control must be an integer multiple of dt_plant")
        if not self.collision_threshold < self.track.half_width:
            raise ValueError("collision threshold must be below the track half width")

    @property
    def plant_substeps(self):
        return round(self.dt_control / self.dt_plant)

    def plant_params(self):
        return replace(self.vehicle, dt=self.dt_plant, integrator="rk4")

    def model_params(self):
        return replace(self.vehicle, dt=self.dt_control, integrator="euler")


@dataclass
class RunRecord:
    run_index: int
    crashed: bool
    collisions: int
    violation_rate: float       # fraction of steps with |e_y| > collision threshold
    lap_time: float = None
    mean_speed: float = 0.0
    satisfaction_rate: float = None   # SafetyMonitor.rate (None for plain MPPI)
    steps: int = 0
    latency_ms: np.ndarray = None       # wall time of each control_step
    device_ms: np.ndarray = None        # device time of each iteration
    trajectory: np.ndarray = None       # (steps, 10): x (8) after the step, u0 (2)


# ------------------------------------------------------------------ safety monitor

class SafetyMonitor:
    """Realised safety-condition bookkeeping along the executed trajectory
    (reference sim.py:157-220): the fraction of executed steps whose
    (h_k, h_{k-1}) pair satisfies the discrete safety condition
    h_k - (1 - beta) h_{k-1} >= 0, with h = max(w - nu sigma_y, 0)^2 - e_y^2
    (constraints.py:130-137, 172-181).

    For the belief-space controller sigma_y is the e_y spread of the belief
    re-propagated Monte-Carlo style over a sliding window of executed
    controls from the measured state at the window start -- the reference's
    ``propagate_mc_batch`` loop (sim.py:189-201) -- run here as ONE device
    rollout (K = 1, the window's controls given, the reference's own keyed
    MONITOR stream supplying the normals, per-step moments returned);
    deterministic shielded controllers use sigma_y = 0."""

    def __init__(self, cfg, run_index, device=0):
        c = cfg.controller
        self.kind = c.kind
        self.nu = float(cfg.cost.backoff)
        self.beta = float(cfg.cost.safety.cbf_rate)
        self.half_width = float(cfg.track.half_width)
        self.track = cfg.track
        self.w = int(getattr(cfg, "monitor_window", 0) or max(1, c.horizon // 2))
        self.window = deque(maxlen=self.w)
        self.inner = max(2, int(c.inner_samples))
        self.master_seed = cfg.master_seed
        self.run_index = run_index
        self.h_prev = None
        self.satisfied = 0
        self.total = 0
        self.last = (np.nan, np.nan, 0.0)   # (h, residual, sigma_y) of the latest step
        self._dev = None
        self._cfg = cfg
        self._device = device

    def _context(self):
        if self._dev is None:
            cfg = self._cfg
            ctx = RolloutContext(cfg.model_params(), cfg.track, cfg.cost, noise=cfg.noise)
            prob, keep = build_problem("bss", 1, self.w, self.inner, 1.0, 0.0, np.eye(2), None,
                                       ControlBounds(), False, ctx)
            self._dev = DeviceContext(prob, self._device)
            del keep
        return self._dev

    def _kappa(self, s):
        tr = self.track
        sw = np.mod(s, tr.length) if tr.closed else np.clip(s, 0.0, tr.length)
        return float(np.interp(sw, tr.s, tr.kappa, period=tr.length) if tr.closed
                     else np.interp(sw, tr.s, tr.kappa))

    def _window_sigma(self, step_index):
        rng = streams.substream(self.master_seed, streams.DOMAIN_RUN, self.run_index,
                                streams.DOMAIN_MONITOR, step_index)
        n = len(self.window)
        x0 = np.ascontiguousarray(self.window[0][0], dtype=np.float64)
        u = np.zeros((1, self.w, 2))
        u[0, :n] = np.array([uu for _, uu in self.window])
        z = np.zeros((self.w, 1, self.inner, 7), dtype=np.float32)
        # the reference draws (1, N, 7) per propagated step from one stream:
        # the same numbers as one (n, 1, N, 7) draw
        z[:n] = rng.standard_normal((n, 1, self.inner, 7))
        dev = self._context()
        eps = np.zeros_like(u)
        nom = np.zeros((self.w, 2))
        cost = np.empty(1)
        mom = np.empty((self.w, 1, 18), dtype=np.float32)
        _lib.check(dev.lib.bssmppi_rollout(dev.h, _lib.dptr(x0), None, _lib.dptr(u), _lib.dptr(eps),
                                           _lib.dptr(nom), _lib.fptr(z), None, _lib.dptr(cost),
                                           _lib.fptr(mom)))
        # stop at the first step whose mean leaves the frame or turns
        # non-finite (belief.py:376-379; sim.py:198-200), else the window end
        m = mom[:n, 0].astype(np.float64)
        t_end = n - 1
        for t in range(n):
            fin = np.all(np.isfinite(m[t]))
            if not fin or not (1.0 - self._kappa(m[t, IDX_S]) * m[t, IDX_EY] > 0.0):
                t_end = t
                break
        var_ey = m[t_end, 17]   # covariance upper triangle, entry (e_y, e_y)
        return float(np.sqrt(max(var_ey, 0.0))) if np.isfinite(var_ey) else float("nan")

    def update(self, state_before, control, state_after, step_index):
        self.window.append((np.asarray(state_before, dtype=float).copy(),
                            np.asarray(control, dtype=float).copy()))
        sigma_y = self._window_sigma(step_index) if self.kind == "bss" else 0.0
        margin = max(self.half_width - self.nu * sigma_y, 0.0)
        h = float(margin * margin - state_after[IDX_EY] ** 2)
        if self.h_prev is None:
            self.h_prev = h   # k = 0: the previous belief equals the current one
        residual = h - (1.0 - self.beta) * self.h_prev
        self.satisfied += residual >= 0.0
        self.total += 1
        self.h_prev = h
        self.last = (h, residual, sigma_y)

    @property
    def rate(self):
        if self.kind == "mppi" or self.total == 0:
            return None
        return self.satisfied / self.total

    def close(self):
        if self._dev is not None:
            self._dev.close()
            self._dev = None


def initial_state(cfg, run_index):
    """reference sim.py:223-229 (same keyed stream)."""
    rng = streams.substream(cfg.master_seed, streams.DOMAIN_RUN, run_index, streams.DOMAIN_INIT)
    jitter = cfg.init_jitter * rng.standard_normal(2)
    return VehicleState.rolling(cfg.init_speed + jitter[0], cfg.vehicle, e_y=jitter[1]).as_array()


def run_closed_loop(cfg: ExperimentConfig, run_index: int = 0, *, noise_source="philox",
                    device=0, max_steps=None, record=True, controller_factory=None,
                    monitor=True) -> RunRecord:
    """Alternate device controller and host plant until lap completion, crash
    (|e_y| beyond the lane or a frame break) or the step budget.
    ``controller_factory(cfg, run_path)`` swaps in another controller with
    the same interface (e.g. a CPU reference arm)."""
    track = cfg.track
    plant = cfg.plant_params()
    if controller_factory is not None:
        ctrl = controller_factory(cfg, (streams.DOMAIN_RUN, run_index))
    else:
        ctrl = Controller(cfg.controller, cfg.cost, cfg.model_params(), track, noise=cfg.noise,
                          subset=DEFAULT_SUBSET, seed=cfg.master_seed,
                          run_path=(streams.DOMAIN_RUN, run_index), noise_source=noise_source,
                          device=device)
    plant_rng = streams.substream(cfg.master_seed, streams.DOMAIN_RUN, run_index, streams.DOMAIN_PLANT)
    monitor = SafetyMonitor(cfg, run_index, device) if monitor else None
    if hasattr(ctrl, "prepare"):
        ctrl.prepare()      # CUDA context + kernel modules before the first timed step
    F = cfg.noise.factor
    x = initial_state(cfg, run_index)
    target = cfg.laps * track.length
    progress, prev_s = 0.0, x[IDX_S]
    crashed, lap_time, steps = False, None, 0
    active = abs(x[IDX_EY]) > cfg.collision_threshold
    collisions = 0
    violating = 0
    lat, dev, rows = [], [], []
    n_steps = cfg.max_steps if max_steps is None else max_steps
    try:
        for step_index in range(n_steps):
            tic = time.perf_counter()
            u0, _ = ctrl.control_step(x)
            lat.append(1e3 * (time.perf_counter() - tic))
            dev.append(ctrl.last_diagnostics["device_ms"])
            w = plant_rng.standard_normal(len(cfg.noise.channels)) @ F.T   # sample_noise, dynamics.py:317-322
            x_before = x
            frame_ok = True
            for j in range(cfg.plant_substeps):
                x, ok = plant_step(x, u0, w if j == cfg.plant_substeps - 1 else None, plant, track,
                                   cfg.noise.channels)
                if not ok:
                    frame_ok = False
                    break
            steps = step_index + 1
            ds = x[IDX_S] - prev_s
            if track.closed:
                ds = (ds + 0.5 * track.length) % track.length - 0.5 * track.length
            progress += ds
            prev_s = x[IDX_S]
            if monitor is not None:
                monitor.update(x_before, u0, x, step_index)
            if record:
                rows.append(np.concatenate([x, u0]))
            v = abs(x[IDX_EY]) > cfg.collision_threshold
            violating += v
            if v and not active:
                collisions += 1
            active = v
            if not frame_ok or abs(x[IDX_EY]) > track.half_width:
                crashed = True
                break
            if progress >= target:
                lap_time = steps * cfg.dt_control
                break
    finally:
        ctrl.close()
        if monitor is not None:
            monitor.close()
    elapsed = steps * cfg.dt_control
    return RunRecord(run_index=run_index, crashed=crashed, collisions=collisions,
                     violation_rate=violating / max(steps, 1), lap_time=lap_time,
                     mean_speed=progress / elapsed if elapsed > 0 else 0.0,
                     satisfaction_rate=None if monitor is None else monitor.rate, steps=steps,
                     latency_ms=np.array(lat), device_ms=np.array(dev),
                     trajectory=np.array(rows) if rows else None)
