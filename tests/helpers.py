"""Shared test helpers: load golden fixtures, rebuild their inputs with this
repo's host mirror, and run the CPU oracle on them."""

import json
import math
import types
from pathlib import Path

import numpy as np

from cases import build, case_by_name

from paper_2408_00494_b200 import controllers as mc
from paper_2408_00494_b200 import dynamics as md

GOLDEN = Path(__file__).resolve().parent / "golden"

from paper_2408_00494_b200.constraints import SafetyParams  # noqa: E402

MINE = types.SimpleNamespace(
    VehicleParams=md.VehicleParams, VehicleState=md.VehicleState, NoiseModel=md.NoiseModel,
    CostSpec=mc.CostSpec, MppiConfig=mc.MppiConfig, make_test_track=md.make_test_track,
    with_timestep=md.with_timestep, SafetyParams=SafetyParams, Track=md.Track)


def load_golden(name):
    d = np.load(GOLDEN / f"{name}.npz")
    meta = json.loads(str(d["meta"]))
    return meta, {k: d[k] for k in d.files if k != "meta"}


class Inputs:
    """Everything the captured iteration of a golden case consumed."""

    def __init__(self, name):
        from oracle import bss_oracle as orc

        self.name = name
        self.meta, self.gold = load_golden(name)
        case = self.case = case_by_name(name)
        (self.cfg, self.cost, self.model, self.track, self.noise, self.x0, self.cov0,
         _) = build(case, MINE)
        self.K, self.T, self.M = case["K"], case["T"], case["M"]
        self.kind = case["kind"]
        self.plan = self.gold["plan_before"]
        self.iteration = self.meta["iteration"]
        lo = np.array([-self.cfg.bounds.delta_max, self.cfg.bounds.throttle_min])
        hi = np.array([self.cfg.bounds.delta_max, self.cfg.bounds.throttle_max])
        self.lo, self.hi = lo, hi
        factor = md.psd_factor(self.cfg.sigma_eps)
        self.u, self.eps, self.z = orc.control_step_inputs(
            case["seed"], case["run_path"], self.iteration, self.K, self.T, max(self.M, 2),
            self.plan, factor, lo, hi, kind=self.kind)
        self.ctx = mc.RolloutContext(self.model, self.track, self.cost, noise=self.noise)
        self.prob = orc.Problem.from_reference(self.ctx)

    def oracle(self, record=None):
        from oracle import bss_oracle as orc

        if self.kind == "bss":
            costs = orc.rollout_bss(self.prob, self.x0, self.cov0, self.u, self.eps, self.plan,
                                    self.z, self.cfg.precision, self.cfg.control_cost_weight,
                                    persist=self.case["persist"], record=record)
        else:
            costs = orc.rollout_det(self.prob, self.kind, self.x0, self.u, self.eps, self.plan,
                                    self.cfg.precision, self.cfg.control_cost_weight)
        vplus = None
        if np.isfinite(costs).any():
            vplus = orc.mppi_update(costs, self.u, self.cfg.temperature, self.lo, self.hi)
        return costs, vplus


COV_FLOOR = 1e-24   # sigma^2 of 1e-12: below it a variance is rounding noise


def unpack_moments(mom):
    """(..., 18) device/C-oracle layout -> mean (..., 8), cov (..., 4, 4)."""
    mean = np.asarray(mom[..., :8], dtype=np.float64)
    up = np.asarray(mom[..., 8:], dtype=np.float64)
    cov = np.empty(mean.shape[:-1] + (4, 4))
    q = 0
    for a in range(4):
        for b in range(a, 4):
            cov[..., a, b] = cov[..., b, a] = up[..., q]
            q += 1
    return mean, cov


def channel_spread(noise_factor):
    """(8,) particle spread of the components outside the tracked
    covariance: vx carries the process noise added after every step
    (dynamics.py:571-572), std sqrt((F F^T)_00); the wheel speeds and s are
    shared by a rollout's particles after re-projection (spread 0)."""
    F = np.asarray(noise_factor, dtype=float).reshape(3, 3)
    out = np.zeros(8)
    out[0] = math.sqrt((F @ F.T)[0, 0])
    return out


def moments_err_arrays(mean_a, cov_a, mean_b, cov_b, spread=None):
    """Elementwise SURVEY 8c moment errors: (em (..., 8), ec (..., 4, 4)).
    Mean scale: max(|mu_i|, sigma_i) with sigma_i from b's covariance for
    the tracked subset (vy, r, e_psi, e_y) and from ``spread``
    (channel_spread) for the others -- a component crossing zero (vx at a
    standstill) is measured against its belief spread, not against 0."""
    sub = [1, 2, 5, 6]
    sig = np.sqrt(np.clip(np.diagonal(cov_b, axis1=-2, axis2=-1), 0, None))
    scale_m = np.abs(mean_b).copy()
    scale_m[..., sub] = np.maximum(scale_m[..., sub], sig)
    if spread is not None:
        scale_m = np.maximum(scale_m, np.asarray(spread, dtype=float))
    with np.errstate(divide="ignore", invalid="ignore"):
        em = np.abs(mean_a - mean_b) / scale_m
        em = np.where(scale_m == 0, np.where(mean_a == mean_b, 0.0, np.inf), em)
        var = np.maximum(sig ** 2, COV_FLOOR)
        denom = np.sqrt(np.einsum("...i,...j->...ij", var, var))
        ec = np.abs(cov_a - cov_b) / denom
        ec = np.where(denom == 0, np.where(cov_a == cov_b, 0.0, np.inf), ec)
    return em, ec


def moments_rel_err(mean_a, cov_a, mean_b, cov_b, spread=None):
    """SURVEY.md 8c moment metric (max over all entries): |dmu_i| /
    max(|mu_i|, sigma_i) and |dSigma_ab| / sqrt(S_aa S_bb), sigma from b.
    The covariance scale is floored at COV_FLOOR: the FP64 reference's
    two-pass variance of M identical particles is ~ulp^2 (e.g. 3e-33 for
    e_y at M = 24) where the device's shifted sums give exactly 0."""
    if mean_a.size == 0:
        return 0.0, 0.0
    em, ec = moments_err_arrays(mean_a, cov_a, mean_b, cov_b, spread)
    return float(np.max(em)), float(np.max(ec))


def fp32_jitter_floor(name):
    """Largest belief-mean error of 8 careful FP32 ports of the reference
    that differ only in +-1 ulp roundings of the mean (committed fixture,
    tests/golden/make_fp32_floor.py); 0 for cases without an entry."""
    import json
    d = json.loads((GOLDEN / "fp32_floor.json").read_text())
    return d["cases"].get(name, {}).get("mean_max", 0.0)


def fp32_state_floor(inp, ks=None):
    """Per-step (mean, cov) of the reference algorithm (FP64 oracle) with
    every particle state rounded to FP32 after each re-projection and step:
    the error any FP32-register implementation carries irreducibly
    (oracle/bss_oracle.py rollout_bss(round_state=float32))."""
    from oracle import bss_oracle as orc

    rec = []
    orc.rollout_bss(inp.prob, inp.x0, inp.cov0, inp.u, inp.eps, inp.plan, inp.z, inp.cfg.precision,
                    inp.cfg.control_cost_weight, persist=inp.case["persist"], record=rec,
                    round_state=np.float32)
    mean, cov = np.stack([r[0] for r in rec]), np.stack([r[1] for r in rec])
    return (mean, cov) if ks is None else (mean[:, ks], cov[:, ks])


def death_mismatches_weightless(gpu, ref, lam=1.0, span=100.0):
    """Rollouts dead (+inf) in exactly one of two FP32 / FP64 runs of the same
    batch: (count, all weightless).  A rollout that leaves the curvilinear
    frame near the end of the horizon can die one step apart in FP32 and
    FP64 (the frame check is a sharp threshold on a chaotic off-track
    trajectory); such a rollout must carry no weight, i.e. its finite cost
    sits more than span * lambda above the best one."""
    import numpy as np
    gf, rf = np.isfinite(gpu), np.isfinite(ref)
    mism = gf != rf
    best = min(np.min(gpu[gf]) if gf.any() else np.inf, np.min(ref[rf]) if rf.any() else np.inf)
    alive_cost = np.where(rf, ref, gpu)
    return int(mism.sum()), bool(np.all(alive_cost[mism] - best > span * lam))
