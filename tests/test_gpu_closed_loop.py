"""Closed loop (BASELINE config 2 setting at parity size): the device
controller in oracle-noise mode inside the host harness follows the
reference's own closed-loop trajectory (sim.run_closed_loop, golden
fixture) step for step until FP32/FP64 differences are amplified by the
closed-loop dynamics."""

import json

import numpy as np
import pytest

from cases import CLOSED_LOOP, build_closed_loop
from helpers import GOLDEN, MINE

from paper_2408_00494_b200 import sim

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("case", CLOSED_LOOP, ids=[c["name"] for c in CLOSED_LOOP])
def test_closed_loop_tracks_reference(case):
    gold = np.load(GOLDEN / f"{case['name']}.npz")
    ref = gold["trajectory"]            # t, s, e_Y, e_psi, vX, vY, psi_dot, delta, T, h, residual, sigma_y
    cfg = build_closed_loop(case, MINE, sim)
    rec = sim.run_closed_loop(cfg, case["run"], noise_source="reference")
    assert rec.steps == int(gold["steps"][0]) and rec.crashed == bool(gold["crashed"][0])
    tr = rec.trajectory
    mine = np.stack([tr[:, 7], tr[:, 6], tr[:, 5], tr[:, 0], tr[:, 1], tr[:, 2], tr[:, 8], tr[:, 9]], 1)
    theirs = ref[:, 1:9]
    err_u = np.abs(mine[:, 6:] - theirs[:, 6:]).max(axis=1)
    scale = np.maximum(np.abs(theirs[:, :6]).max(axis=0), 1.0)     # s ~ tens of metres
    err_x = (np.abs(mine[:, :6] - theirs[:, :6]) / scale).max(axis=1)
    first_div = int(np.argmax(err_u > 1e-3)) if np.any(err_u > 1e-3) else len(err_u)
    print(f"{case['name']}: first step with |du0|>1e-3: {first_div}; |dx| at 10/20/60: "
          f"{err_x[9]:.2e} {err_x[19]:.2e} {err_x[-1]:.2e}")
    # MPPI at lambda = 1 is near-argmin (ESS ~ 1): once an FP32/FP64 cost
    # difference flips a near-tie the two loops separate, so step-for-step
    # agreement is asserted over the first steps only ...
    assert first_div >= 5
    assert err_x[:5].max() < 5e-4   # v+ agrees to ~1e-5 (tolerance 1e-4); the plant propagates it
    # ... and the run statistics afterwards
    assert abs(tr[:, 0].mean() - theirs[:, 3].mean()) < 0.02 * abs(theirs[:, 3].mean())
    assert np.abs(tr[:, 6]).max() < 1.2 and np.abs(theirs[:, 2]).max() < 1.2
