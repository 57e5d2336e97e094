"""CPU FP64 oracle for the BSS-MPPI step -- TEST INFRASTRUCTURE ONLY.

A numpy restatement of the reference algorithm (arxiv 2408.00494 package
``belief_mppi``, read-only at /root/reference/pkg/src/belief_mppi).  Only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` leg may import this module; the product path
(``paper_2408_00494_b200``) never does.

Parity pin: ``tests/golden/make_golden.py`` runs the real reference in the
build container and stores its outputs; ``tests/test_oracle.py`` checks this
restatement against them (costs/moments/v+ to ~1e-10).

Every function cites the reference lines it restates.  Inputs are the
*captured* noise arrays (eps after the factor, z_all), exactly as the
reference consumes them, so the restatement is independent of the RNG.
"""

from __future__ import annotations

import math

import numpy as np

IDX_VX, IDX_VY, IDX_R, IDX_WF, IDX_WR, IDX_EPSI, IDX_EY, IDX_S = range(8)
SUBSET = np.array([1, 2, 5, 6])   # DEFAULT_SUBSET, belief.py:69
P_EY = 3                          # DEFAULT_SUBSET.position(IDX_EY)
G = 9.81


def phys(p) -> np.ndarray:
    """``_phys_vector`` (dynamics.py:325-337)."""
    wb = p.lf + p.lr
    return np.array([
        p.mass, p.inertia_z, p.lf, p.lr, p.wheel_radius, p.wheel_inertia,
        p.b_lat_front, p.c_lat_front, p.b_lat_rear, p.c_lat_rear,
        p.b_long_front, p.c_long_front, p.b_long_rear, p.c_long_rear,
        p.peak_fx_front, p.peak_fy_front, p.peak_fx_rear, p.peak_fy_rear,
        p.drive_gain, p.roll_resist, p.v_floor,
        p.mass * G * p.lr / wb, p.mass * G * p.lf / wb])


def curv(s, s_nodes, k_nodes, length, closed):
    """``_curv_scalar`` (dynamics.py:340-369), vectorised.  Python ``%`` is a
    floor-mod like numba's, so (-tiny) % L == L and hits the wrap segment."""
    s = np.asarray(s, dtype=float)
    sw = np.mod(s, length) if closed else np.clip(s, 0.0, length)
    n = s_nodes.shape[0]
    lo = np.searchsorted(s_nodes, sw, side="right") - 1     # binary search, :354-361
    lo = np.clip(lo, 0, n - 1)
    wrap = closed & (sw >= s_nodes[n - 1])
    x0 = np.where(wrap, s_nodes[n - 1], s_nodes[lo])
    x1 = np.where(wrap, length, s_nodes[np.minimum(lo + 1, n - 1)])
    y0 = np.where(wrap, k_nodes[n - 1], k_nodes[lo])
    y1 = np.where(wrap, k_nodes[0], k_nodes[np.minimum(lo + 1, n - 1)])
    with np.errstate(invalid="ignore", divide="ignore"):
        val = y0 + (y1 - y0) * (sw - x0) / (x1 - x0)
    val = np.where(x1 == x0, y0, val)
    if not closed:
        val = np.where(lo >= n - 1, k_nodes[n - 1], val)     # :362-363
    return val


def tire(vx, vy, r, wf, wr, delta, p):
    """``_tire_row`` (dynamics.py:372-395)."""
    vx_eff = np.where(vx >= 0.0, np.maximum(vx, p[20]), np.minimum(vx, -p[20]))
    denom = np.abs(vx_eff)
    alpha_f = delta - np.arctan2(vy + p[2] * r, vx_eff)
    alpha_r = -np.arctan2(vy - p[3] * r, vx_eff)
    sigma_f = (wf * p[4] - vx) / denom
    sigma_r = (wr * p[4] - vx) / denom
    fyf0 = p[15] * np.sin(p[7] * np.arctan(p[6] * alpha_f))
    fyr0 = p[17] * np.sin(p[9] * np.arctan(p[8] * alpha_r))
    fxf = p[14] * np.sin(p[11] * np.arctan(p[10] * sigma_f))
    fxr = p[16] * np.sin(p[13] * np.arctan(p[12] * sigma_r))
    fyf = fyf0 * np.sqrt(np.maximum(1.0 - (fxf / p[14]) ** 2, 0.0))
    fyr = fyr0 * np.sqrt(np.maximum(1.0 - (fxr / p[16]) ** 2, 0.0))
    return fxf, fyf, fxr, fyr


def derivs(x, u0, u1, p, track):
    """``_derivs_row`` (dynamics.py:398-437); x (..., 8) -> (dx, frame_ok)."""
    vx, vy, r, wf, wr, e_psi, e_y, s = (x[..., i] for i in range(8))
    fxf, fyf, fxr, fyr = tire(vx, vy, r, wf, wr, u0, p)
    cos_d, sin_d = np.cos(u0), np.sin(u0)
    fxf_b = fxf * cos_d - fyf * sin_d
    fyf_b = fxf * sin_d + fyf * cos_d
    dx = np.empty(x.shape, x.dtype)
    dx[..., 0] = (fxf_b + fxr) / p[0] + vy * r
    dx[..., 1] = (fyf_b + fyr) / p[0] - vx * r
    dx[..., 2] = (p[2] * fyf_b - p[3] * fyr) / p[1]
    spin_f = np.tanh(wf * p[4] / 0.1)
    spin_r = np.tanh(wr * p[4] / 0.1)
    dx[..., 3] = (-p[4] * fxf - p[19] * p[21] * p[4] * spin_f) / p[5]
    dx[..., 4] = (p[18] * u1 - p[4] * fxr - p[19] * p[22] * p[4] * spin_r) / p[5]
    kappa = curv(s, track.s, track.kappa, track.length, track.closed)
    frame = 1.0 - kappa * e_y
    ok = frame > 0.0
    frame = np.where(frame < 1e-3, 1e-3, frame)
    cos_e, sin_e = np.cos(e_psi), np.sin(e_psi)
    ds = (vx * cos_e - vy * sin_e) / frame
    dx[..., 7] = ds
    dx[..., 6] = vx * sin_e + vy * cos_e
    dx[..., 5] = r - kappa * ds
    return dx, ok


def step_euler(x, u, p, track, dt, wrap_when_needed=False):
    """Euler branch of ``_step_kernel`` (dynamics.py:447-497): x + dt f(x),
    e_psi wrapped to (-pi, pi], s floor-mod L, non-finite -> 0 and ok=False.
    ``wrap_when_needed`` applies the heading formula only outside (-pi, pi]
    (where it is the identity in exact arithmetic): the FP32 emulations use
    it, since the literal formula quantises e_psi to ulp(pi) in FP32."""
    u = np.asarray(u, dtype=x.dtype)
    with np.errstate(all="ignore"):
        dx, ok = derivs(x, u[..., 0], u[..., 1], p, track)
        out = x + dt * dx
        pi = out.dtype.type(math.pi)
        wrapped = pi - np.mod(pi - out[..., 5], 2 * pi)
        if wrap_when_needed:
            inside = (out[..., 5] > -pi) & (out[..., 5] <= pi)
            out[..., 5] = np.where(inside, out[..., 5], wrapped)
        else:
            out[..., 5] = wrapped
        if track.closed:
            out[..., 7] = np.mod(out[..., 7], track.length)
        else:
            out[..., 7] = np.clip(out[..., 7], 0.0, track.length)
    bad = ~np.isfinite(out)
    ok = ok & ~bad.any(axis=-1)
    out[bad] = 0.0
    return out, ok


def chol_psd(covs):
    """``_psd_chol_kernel`` (belief.py:235-256): zero-pivot columns stay zero."""
    k, t, _ = covs.shape
    out = np.zeros_like(covs)
    for c in range(t):
        acc = covs[:, c, c].copy()
        for q in range(c):
            acc = acc - out[:, c, q] * out[:, c, q]
        live = acc > 1e-300
        piv = np.sqrt(np.where(live, acc, 1.0))
        out[:, c, c] = np.where(live, piv, 0.0)
        for r in range(c + 1, t):
            a = covs[:, r, c].copy()
            for q in range(c):
                a = a - out[:, r, q] * out[:, c, q]
            out[:, r, c] = np.where(live, a / piv, 0.0)
    return out


def tree_mean(x):
    """Pairwise tree mean over axis 1 (``_moments_kernel`` belief.py:282-296)."""
    n = x.shape[1]
    buf = x.copy()
    width = n
    while width > 1:
        half = width // 2
        nxt = buf[:, 0:2 * half:2] + buf[:, 1:2 * half:2]
        if width % 2 == 1:
            nxt = np.concatenate([nxt, buf[:, width - 1:width]], axis=1)
            width = half + 1
        else:
            width = half
        buf = nxt
    return buf[:, 0] / n


def moments(x1):
    """Tree mean of all 8 components + unbiased two-pass 4x4 covariance over
    the tracked subset (belief.py:275-308)."""
    mean = tree_mean(x1)
    n = x1.shape[1]
    dev = x1[:, :, SUBSET] - mean[:, None, SUBSET]
    cov = np.empty((x1.shape[0], 4, 4))
    for a in range(4):
        for b in range(a, 4):
            acc = np.zeros(x1.shape[0])
            for j in range(n):                      # fixed sequential order, :302-305
                acc = acc + dev[:, j, a] * dev[:, j, b]
            cov[:, a, b] = cov[:, b, a] = acc / (n - 1)
    return mean, cov


def stage_cost(x, q, v_goal, c_obs, half_width):
    """``stage_cost_values`` (controllers.py:215-220)."""
    g = np.zeros(8)
    g[IDX_VX] = v_goal
    quad = np.square(x - g) @ q
    return quad + c_obs * (np.abs(x[..., IDX_EY]) > half_width)


def dcbf(e_y, sigma_y, half_width, nu):
    """``track_dcbf_values`` (constraints.py:130-137)."""
    margin = np.clip(half_width - nu * sigma_y, 0.0, None)
    return margin * margin - e_y * e_y


def penalty(h_cur, h_prev, beta, c_pen):
    """``penalty_values`` (constraints.py:172-186)."""
    return c_pen * np.clip(-(h_cur - (1.0 - beta) * h_prev), 0.0, None)


def control_cost(nominal, eps, precision, gamma):
    """``control_cost_values`` (controllers.py:223-228); unclamped v+eps."""
    if gamma == 0.0:
        return np.zeros(eps.shape[0])
    return gamma * np.einsum("kc,cd,mkd->m", nominal, precision, nominal[None] + eps)


def _finite_or_zero(x):
    return np.where(np.isfinite(x), x, 0.0)


class Problem:
    """Bundle of the per-controller constants (RolloutContext +
    MppiConfig + CostSpec, controllers.py:71-138, 197-212)."""

    def __init__(self, params, track, q_diag, v_goal=6.0, obstacle_penalty=1e4,
                 terminal_scale=1.0, cbf_rate=0.35, penalty=2000.0,
                 backoff=1.959963984540054, noise_factor=None):
        self.p = phys(params)
        self.dt = float(params.dt)
        self.track = track
        self.q = np.asarray(q_diag, dtype=float)
        self.v_goal = float(v_goal)
        self.c_obs = float(obstacle_penalty)
        self.term = float(terminal_scale)
        self.beta = float(cbf_rate)
        self.c_pen = float(penalty)
        self.nu = float(backoff)
        self.F = np.zeros((3, 3)) if noise_factor is None else np.asarray(noise_factor, float)

    @classmethod
    def from_reference(cls, ctx):
        """Build from a (reference or mirror) RolloutContext-like object."""
        c = ctx.cost
        F = ctx.noise.factor if ctx.noise is not None else np.zeros((3, 3))
        return cls(ctx.model, ctx.track, c.q_diag, c.v_goal, c.obstacle_penalty,
                   c.terminal_scale, c.safety.cbf_rate, c.safety.penalty, c.backoff, F)

    def astype(self, dtype):
        """Copy whose constants and track tables are ``dtype`` (FP32
        emulation of the reference, tests/test_fp32_conditioning.py): numpy
        then evaluates the reference's formulas in that precision."""
        import copy
        import types
        out = copy.copy(self)
        out.p = self.p.astype(dtype)
        out.dt = dtype(self.dt)
        out.q = self.q.astype(dtype)
        out.F = self.F.astype(dtype)
        tr = self.track
        out.track = types.SimpleNamespace(s=np.asarray(tr.s, dtype), kappa=np.asarray(tr.kappa, dtype),
                                          length=dtype(tr.length), closed=tr.closed,
                                          half_width=dtype(tr.half_width))
        return out

    def stage(self, x):
        return stage_cost(x, self.q, self.v_goal, self.c_obs, self.track.half_width)

    def h(self, e_y, sigma_y):
        return dcbf(e_y, sigma_y, self.track.half_width, self.nu)


def rollout_bss(prob: Problem, x0, cov0, u, eps, nominal, z_all, precision=None,
                gamma=0.0, persist=False, record=None, dtype=np.float64, round_state=None,
                step_dtype=None, careful=False):
    """Belief rollout costs (``_rollout`` bss branch, controllers.py:261-319, 340).

    u: (K, T, 2) clamped controls, eps: (K, T, 2) raw perturbations,
    z_all: (T, K, M, 7) standard normals.  ``record`` (list) receives
    (mean, cov, ok) per step like the reference's propagate_mc_batch.
    ``dtype=np.float32`` evaluates the same algorithm (dynamics, tree mean,
    two-pass covariance, Cholesky) in FP32 -- the SURVEY A4 emulation that
    separates FP32's own conditioning from device deviations.
    ``round_state=np.float32`` keeps FP64 arithmetic but rounds every
    particle state to FP32 after the re-projection and after the step: the
    irreducible error of holding particles in FP32 registers.
    ``step_dtype=np.float32`` (with ``round_state``) additionally evaluates
    the Euler step -- tire model, derivatives, update -- in FP32 arithmetic
    (numpy float32 libm, heading wrap only when needed), everything else in
    FP64: the floor of a careful FP32 implementation of the step.
    ``careful=True`` with ``dtype=np.float32``: the whole algorithm in FP32
    except the literal heading-wrap formula (applied only outside (-pi, pi],
    where it is not the identity) -- a careful FP32 port."""
    rnd = (lambda a: a) if round_state is None else (lambda a: a.astype(round_state).astype(a.dtype))
    K, T, _ = u.shape
    M = z_all.shape[2]
    if dtype is not np.float64:
        prob = prob.astype(dtype)
        u = np.asarray(u, dtype)
        z_all = np.asarray(z_all, dtype)
    x0 = np.asarray(x0, dtype)
    cov0 = np.asarray(cov0, dtype)
    precision = np.zeros((2, 2)) if precision is None else precision
    total = control_cost(np.asarray(nominal, float), eps, precision, gamma)
    dead = np.zeros(K, dtype=bool)
    means = np.repeat(x0[None], K, axis=0)
    covs = np.repeat(cov0[None], K, axis=0)
    noise_on = bool(np.any(prob.F))
    cloud = None
    if persist:                                           # gaussian_cloud, belief.py:338-348
        cloud = means[:, None, :].repeat(M, axis=1)
        cloud[:, :, SUBSET] += np.einsum("kab,kmb->kma", chol_psd(covs), z_all[0][:, :, :4])
    sig = np.sqrt(np.clip(covs[:, P_EY, P_EY], 0.0, None))
    h_cur = prob.h(means[:, IDX_EY], sig)
    h_prev = h_cur
    for t in range(T):
        total = total + prob.stage(means)
        if t > 0:
            total = total + penalty(h_cur, h_prev, prob.beta, prob.c_pen)
        if persist:
            x = cloud
        else:                                             # propagate_mc_batch, belief.py:311-335
            L = chol_psd(covs)
            x = np.repeat(means[:, None, :], M, axis=1)
            x[:, :, SUBSET] += np.einsum("kab,kmb->kma", L, z_all[t][:, :, :4])
        x = rnd(x)
        ub = np.repeat(u[:, t][:, None, :], M, axis=1)
        if dtype is not np.float64:                      # FP32 port: heading wrap only when needed
            x1, _ = step_euler(x, ub, prob.p, prob.track, prob.dt, wrap_when_needed=careful)
        elif step_dtype is not None:
            p32 = prob.astype(step_dtype)
            x1, _ = step_euler(x.astype(step_dtype), ub.astype(step_dtype), p32.p, p32.track, p32.dt,
                               wrap_when_needed=True)
            x1 = x1.astype(x.dtype)
        else:
            x1, _ = step_euler(x, ub, prob.p, prob.track, prob.dt)   # per-particle ok discarded
        if noise_on:                                      # dynamics.py:571-572
            x1[..., 0:3] += z_all[t][:, :, 4:7] @ prob.F.T
        x1 = rnd(x1)
        if persist:
            cloud = x1
        mean1, cov1 = moments(x1)
        ok = np.isfinite(mean1).all(-1) & np.isfinite(cov1).all((-1, -2))
        kap = curv(mean1[:, IDX_S], prob.track.s, prob.track.kappa, prob.track.length,
                   prob.track.closed)
        with np.errstate(invalid="ignore"):
            ok &= (1.0 - kap * mean1[:, IDX_EY]) > 0.0       # belief.py:376-379
        if record is not None:
            record.append((mean1.copy(), cov1.copy(), ok.copy()))
        means = _finite_or_zero(mean1)
        covs = _finite_or_zero(cov1)
        dead |= ~ok
        sig = np.sqrt(np.clip(covs[:, P_EY, P_EY], 0.0, None))
        h_prev, h_cur = h_cur, prob.h(means[:, IDX_EY], sig)
    total = total + prob.term * prob.stage(means)
    total = total + penalty(h_cur, h_prev, prob.beta, prob.c_pen)
    total[dead] = np.inf
    return total


def rollout_det(prob: Problem, kind, x0, u, eps, nominal, precision=None, gamma=0.0):
    """mppi / smppi rollouts (controllers.py:320-338)."""
    K, T, _ = u.shape
    precision = np.zeros((2, 2)) if precision is None else precision
    total = control_cost(np.asarray(nominal, float), eps, precision, gamma)
    dead = np.zeros(K, dtype=bool)
    x = np.repeat(np.asarray(x0, float)[None], K, axis=0)
    shielded = kind == "smppi"
    if shielded:
        h_cur = prob.h(x[:, IDX_EY], 0.0)
        h_prev = h_cur
    for t in range(T):
        total = total + prob.stage(x)
        if shielded and t > 0:
            total = total + penalty(h_cur, h_prev, prob.beta, prob.c_pen)
        x, ok = step_euler(x, u[:, t], prob.p, prob.track, prob.dt)
        dead |= ~ok
        if shielded:
            h_prev, h_cur = h_cur, prob.h(x[:, IDX_EY], 0.0)
    total = total + prob.term * prob.stage(x)
    if shielded:
        total = total + penalty(h_cur, h_prev, prob.beta, prob.c_pen)
    total[dead] = np.inf
    return total


def mppi_update(costs, u, lam, lo, hi):
    """``mppi_weights`` + ``mppi_update`` (controllers.py:180-194)."""
    costs = np.asarray(costs, float)
    fin = np.isfinite(costs)
    if not fin.any():
        raise RuntimeError("AllRolloutsInvalid")
    w = np.exp(-(costs - costs[fin].min()) / lam)
    v = np.einsum("m,mkc->kc", w, u) / w.sum()
    return np.clip(v, lo, hi)


def sample_controls(nominal, factor, z_ctrl, lo, hi):
    """``sample_controls`` (controllers.py:166-177) from captured normals."""
    eps = z_ctrl @ np.asarray(factor).T
    return np.clip(np.asarray(nominal)[None] + eps, lo, hi), eps


def control_step_inputs(seed, run_path, iteration, K, T, M, nominal, sigma_factor, lo, hi,
                        kind="bss"):
    """Draw eps and z_all from the reference's own keyed substreams
    (controllers.py:371-372, 384-393, 285-287; streams.py:21-28)."""
    def sub(*path):
        ss = np.random.SeedSequence(int(seed), spawn_key=tuple(int(p) for p in path))
        return np.random.Generator(np.random.Philox(ss))
    rp = tuple(run_path)
    z_ctrl = sub(*rp, 2, iteration).standard_normal((K, T, 2))
    u, eps = sample_controls(nominal, sigma_factor, z_ctrl, lo, hi)
    z_all = sub(*rp, 3, iteration).standard_normal((T, K, M, 7)) if kind == "bss" else None
    return u, eps, z_all


def shard_record(costs, u, lam, k_begin=0):
    """Partial update record of one K-shard, restating csrc/update.cuh on the
    host (test infrastructure): {beta, Z, Z2, n_finite, argmin, N[2T]} with
    weights relative to the shard's own minimum."""
    costs = np.asarray(costs, float)
    T2 = u.shape[1] * 2
    rec = np.zeros(5 + T2)
    fin = np.isfinite(costs)
    rec[0] = costs[fin].min() if fin.any() else np.inf
    rec[3] = fin.sum()
    rec[4] = (k_begin + int(np.argmin(np.where(fin, costs, np.inf)))) if fin.any() else -1
    if fin.any():
        w = np.where(fin, np.exp(-(costs - rec[0]) / lam), 0.0)
        rec[1] = w.sum()
        rec[2] = (w * w).sum()
        rec[5:] = np.einsum("k,ki->i", w, u.reshape(len(costs), T2))
    return rec


def combine_records(recs, lam, lo, hi):
    """Rank-order combine of shard records -> clamp(v+) (csrc/update.cuh
    combine_kernel); equals mppi_update on the concatenated batch."""
    recs = np.asarray(recs, float)
    live = recs[:, 3] > 0
    if not live.any():
        raise RuntimeError("AllRolloutsInvalid")
    beta = recs[live, 0].min()
    sc = np.where(live, np.exp(-(recs[:, 0] - beta) / lam), 0.0)
    Z = (sc * recs[:, 1]).sum()
    N = (sc[:, None] * recs[:, 5:]).sum(0)
    v = (N / Z).reshape(-1, 2)
    return np.clip(v, lo, hi)
