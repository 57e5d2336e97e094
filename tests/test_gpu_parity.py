"""GPU parity: the sm_100a path (through the C ABI) vs the CPU oracle on the
same inputs and the reference's own noise (oracle-noise mode).

Tolerances (north_star):
  * rollout costs: 1e-3 relative for every rollout with non-negligible
    weight (S - min S <= 100 lambda); the fraction of ALL rollouts within
    1e-3 is asserted separately (off-track rollouts diverge chaotically);
  * belief moments: |dmu_i| <= 1e-4 max(|mu_i|, sigma_i) and
    |dSigma_ab| <= 1e-4 sqrt(S_aa S_bb), exact zeros stay zero;
  * v+: 1e-4 absolute unless the oracle's best two costs are a near-tie.
"""

import numpy as np
import pytest

from cases import CASES, UPDATE_BATCHES, update_batch
from helpers import (GOLDEN, Inputs, channel_spread, fp32_jitter_floor, fp32_state_floor, moments_rel_err,
                     unpack_moments)

from paper_2408_00494_b200 import controllers as mc

pytestmark = pytest.mark.gpu

BSS = [c["name"] for c in CASES if c["kind"] == "bss"]
ALL = [c["name"] for c in CASES]
COST_RTOL = 1e-3
MOM_TOL = 1e-4
VPLUS_ATOL = 1e-4


def _weighted(costs, lam):
    fin = np.isfinite(costs)
    out = np.zeros_like(fin)
    if fin.any():
        out = fin & (costs - costs[fin].min() <= 100.0 * lam)
    return out


def _near_tie(costs, lam, cost_err=1e-5):
    fin = np.sort(costs[np.isfinite(costs)])
    return fin.size > 1 and (fin[1] - fin[0]) < 10 * cost_err * abs(fin[0]) + 1e-9


def _gpu_rollout(inp, moments=False, group_width=0):
    batch = mc.RolloutBatch(inp.u, inp.eps)
    if inp.kind == "bss":
        class _Z:
            def standard_normal(self, shape):
                assert shape == inp.z.shape
                return inp.z
        return mc.rollout_bss(inp.x0, inp.cov0, batch, inp.plan, inp.ctx, _Z(), inp.M,
                              precision=inp.cfg.precision, cost_weight=inp.cfg.control_cost_weight,
                              persist_particles=inp.case["persist"], moments=moments,
                              group_width=group_width)
    fn = mc.rollout_smppi if inp.kind == "smppi" else mc.rollout_mppi
    return fn(inp.x0, batch, inp.plan, inp.ctx, precision=inp.cfg.precision,
              cost_weight=inp.cfg.control_cost_weight)


@pytest.mark.parametrize("name", ALL)
def test_rollout_costs(name):
    inp = Inputs(name)
    ref = inp.gold["costs"]
    got = _gpu_rollout(inp)
    fin = np.isfinite(ref)
    assert np.array_equal(np.isfinite(got), fin), "dead-rollout pattern differs"
    rel = np.abs(got[fin] - ref[fin]) / np.abs(ref[fin])
    w = _weighted(ref, inp.cfg.temperature)
    print(f"{name}: max rel err weighted {rel[w[fin]].max() if w.any() else 0:.2e}, "
          f"all {rel.max() if rel.size else 0:.2e}, frac<1e-3 {np.mean(rel < COST_RTOL) if rel.size else 1:.4f}")
    if w.any():
        assert rel[w[fin]].max() <= COST_RTOL
    if rel.size:
        assert np.mean(rel < COST_RTOL) >= 0.99


# Lane-group widths: 0 = the launch policy (G = 32 for every golden case),
# 2 / 4 / 8 / 16 = the widths the BASELINE shapes run at (C3: G = 8, 32
# particles per lane; C5 32768 x 64: G = 4; C4 and C5 65536+ x 64: G = 2;
# C2: G = 16), pinned through bssmppi_problem.group_width so each lane
# pre-sums up to 64 particles of the golden cases (M = 256 at G = 4; G = 2
# is run where M <= 128, as the policy's 64-per-lane cap implies).
WIDTHS = (0, 2, 4, 8, 16)
MAX_PER_LANE = 64   # the policy never pre-sums more particles per lane


def moment_tolerance(inp, ks, alive, spread):
    """1e-4 (north_star), unless FP32 itself cannot resolve the case to that:

    * the reference's own algorithm with its particle states held in FP32
      (helpers.fp32_state_floor: FP64 arithmetic, one FP32 rounding per
      state component per step) already errs by more than half of 1e-4
      -> 2x that floor (computed here, on the same inputs: it applies where
      particles straddle s = L -- s_wrap, the belief mean of wrapped arc
      lengths -- and to the 4x4 sample covariance of M = 5 particles);
    * for the mean, the largest error of 8 careful FP32 ports of the
      reference that differ only in a +-1 ulp rounding of the belief mean
      per step (tests/golden/fp32_floor.json, tests/golden/make_fp32_floor.py)
      -> that error.  Above 1e-4 only on s_wrap and on low_speed, where
      explicit Euler at the v_floor regularisation is unstable and FP32
      rounding grows ~2.5x per step (an IEEE libdevice build of the kernel
      errs like the fast one there: tools/diag_case.py)."""
    fm, fc = fp32_state_floor(inp, ks)
    gold = inp.gold
    fem, fec = moments_rel_err(fm[alive], fc[alive], gold["means"][alive], gold["covs"][alive], spread)
    jit = fp32_jitter_floor(inp.name)
    return max(MOM_TOL, 2.0 * fem, jit), max(MOM_TOL, 2.0 * fec), (fem, fec, jit)


@pytest.mark.parametrize("G", WIDTHS, ids=lambda g: f"G{g}")
@pytest.mark.parametrize("name", BSS)
def test_belief_moments(name, G):
    """Per-step belief moments (belief.py:275-308) vs the reference's, at the
    policy width and pinned production widths; metric of SURVEY 8c with the
    mean of vx measured against its process-noise spread
    (helpers.channel_spread), no other floor."""
    inp = Inputs(name)
    if G and -(-inp.M // G) > MAX_PER_LANE:
        pytest.skip(f"G = {G} would pre-sum {-(-inp.M // G)} particles per lane (policy cap {MAX_PER_LANE})")
    costs, mom = _gpu_rollout(inp, moments=True, group_width=G)
    gold = inp.gold
    ks = gold["ks"]
    mean, cov = unpack_moments(mom[:, ks])
    # compare rollouts that survive the horizon (a dead rollout is +inf and
    # weightless; its moments after leaving the curvilinear frame are
    # frame-singular in both implementations)
    alive = np.broadcast_to(np.isfinite(gold["costs"][ks])[None, :], mean.shape[:2])
    spread = channel_spread(inp.noise.factor)
    em, ec = moments_rel_err(mean[alive], cov[alive], gold["means"][alive], gold["covs"][alive], spread)
    tol_m, tol_c, floor = moment_tolerance(inp, ks, alive, spread)
    zero = gold["covs"][alive] == 0.0
    print(f"{name} G={G}: moments mean {em:.2e} cov {ec:.2e} (tol {tol_m:.1e}/{tol_c:.1e}; "
          f"fp32-state floor {floor[0]:.1e}/{floor[1]:.1e}; fp32-port rounding spread {floor[2]:.1e})")
    assert em <= tol_m and ec <= tol_c
    assert np.all(cov[alive][zero] == 0.0), "exact zero covariances must stay zero"


@pytest.mark.parametrize("name", ALL)
def test_control_step_oracle_noise(name):
    """Controller.control_step in oracle-noise mode reproduces v+ / u0 /
    next plan of the reference iteration."""
    inp = Inputs(name)
    ctrl = mc.Controller(inp.cfg, inp.cost, inp.model, inp.track, noise=inp.noise,
                         seed=inp.case["seed"], run_path=inp.case["run_path"],
                         noise_source="reference")
    ctrl.plan = mc.ControlPlan(inp.plan.copy())
    ctrl.iteration = inp.iteration
    if inp.meta["invalid"]:
        with pytest.raises(mc.AllRolloutsInvalid):
            ctrl.control_step(inp.x0, inp.cov0)
        assert ctrl.iteration == inp.iteration
        return
    u0, nxt = ctrl.control_step(inp.x0, inp.cov0)
    gold = inp.gold
    d = ctrl.last_diagnostics
    err = np.abs(d["vplus"] - gold["vplus"]).max()
    print(f"{name}: |dv+| {err:.2e} ess {d['ess']:.3f} argmin {d['cost_argmin']} "
          f"ref argmin {int(np.argmin(gold['costs']))}")
    if not _near_tie(gold["costs"], inp.cfg.temperature):
        assert err <= VPLUS_ATOL
        assert d["cost_argmin"] == int(np.argmin(gold["costs"]))
    np.testing.assert_allclose(u0, gold["u0"], atol=VPLUS_ATOL)
    np.testing.assert_allclose(nxt.controls, gold["plan_after"], atol=VPLUS_ATOL)
    assert ctrl.iteration == inp.iteration + 1


@pytest.mark.parametrize("j", range(len(UPDATE_BATCHES)))
def test_update_law_golden(j):
    d = np.load(GOLDEN / "update_law.npz")
    costs, controls, lam = update_batch(j)
    plan = mc.mppi_update(mc.RolloutBatch(controls, np.zeros_like(controls), costs), lam,
                          mc.ControlBounds())
    np.testing.assert_allclose(plan.controls, d[f"u{j}_vplus"], rtol=0, atol=1e-12)
