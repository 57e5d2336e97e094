"""How close FP32 can get to the FP64 reference on the golden cases (SURVEY.md
A4 recipe), so the moment tolerance of tests/test_gpu_parity.py rests on a
measurement instead of an assertion.

Two emulations of the REFERENCE algorithm (oracle/bss_oracle.py rollout_bss,
numpy, same inputs and noise as the golden fixtures):

* ``round_state=float32`` -- FP64 arithmetic, every particle state rounded to
  FP32 after each re-projection and Euler step: the irreducible error of
  holding particles in FP32 registers (the parity tests allow a device error
  of max(1e-4, 2 x this floor));
* ``dtype=float32`` -- the whole algorithm evaluated naively in FP32 (libm
  float32 transcendentals, literal heading wrap, tree mean, two-pass
  covariance): what a direct FP32 port would give.

The device kernel (shifted one-pass sums, heading wrap only when needed,
pinned polynomials) meets 1e-4 on every case except the two where the FP32
state floor itself reaches ~1e-4 (tests/test_gpu_parity.py), while the naive
FP32 port fails 1e-4 on several ordinary cases.
"""

import numpy as np
import pytest

from cases import CASES
from helpers import Inputs, channel_spread, fp32_state_floor, moments_rel_err

from oracle import bss_oracle as orc

BSS = [c["name"] for c in CASES if c["kind"] == "bss"]


def _err(inp, mean, cov):
    g = inp.gold
    ks = g["ks"]
    alive = np.broadcast_to(np.isfinite(g["costs"][ks])[None, :], (g["means"].shape[0], len(ks)))
    return moments_rel_err(mean[:, ks][alive], cov[:, ks][alive], g["means"][alive], g["covs"][alive],
                           channel_spread(inp.noise.factor))


def _naive32(inp):
    rec = []
    orc.rollout_bss(inp.prob, inp.x0, inp.cov0, inp.u, inp.eps, inp.plan, inp.z, inp.cfg.precision,
                    inp.cfg.control_cost_weight, persist=inp.case["persist"], record=rec, dtype=np.float32)
    assert rec[-1][0].dtype == np.float32
    return np.stack([r[0] for r in rec]), np.stack([r[1] for r in rec])


@pytest.fixture(scope="module")
def table():
    out = {}
    for name in BSS:
        inp = Inputs(name)
        out[name] = (_err(inp, *fp32_state_floor(inp)), _err(inp, *_naive32(inp)))
    for name, ((fm, fc), (nm, nc)) in out.items():
        print(f"{name:14s} fp32-state floor {fm:.1e}/{fc:.1e}   naive fp32 {nm:.1e}/{nc:.1e}")
    return out


def test_state_floor_is_below_tolerance_except_branch_edges(table):
    """FP32 state resolution alone keeps every case inside 1e-4; only the
    arc-length wrap (particles straddling s = L enter the mean as ~0 and ~L)
    and the M = 5 sample covariance come within a factor 2 of it."""
    near = {n for n, ((fm, fc), _) in table.items() if max(fm, fc) > 0.5e-4}
    assert near == {"s_wrap", "ragged_m5"}, near
    assert all(max(fm, fc) < 1e-4 for (fm, fc), _ in table.values())


def test_naive_fp32_port_misses_the_tolerance(table):
    """A literal FP32 port of the reference fails 1e-4 on ordinary cases
    (the heading-wrap formula quantises e_psi to ulp(pi); plain FP32
    reductions; libm float32 atan/sin), so the bar is only reachable with
    the device's numerics."""
    over = {n for n, (_, (nm, nc)) in table.items() if max(nm, nc) > 1e-4}
    assert len(over) >= 4, over
    assert "collapse_m16" in over


def test_rounding_spread_fixture_reproduces():
    """tests/golden/fp32_floor.json (the per-case FP32 rounding spread the
    parity tolerance uses) is what tests/golden/make_fp32_floor.py computes:
    re-run two cases and compare every run exactly; and it exceeds 1e-4
    only on the two ill-conditioned cases."""
    import json
    import sys
    from helpers import GOLDEN
    sys.path.insert(0, str(GOLDEN))
    import make_fp32_floor as mk
    d = json.loads((GOLDEN / "fp32_floor.json").read_text())
    assert d["runs"] == mk.R
    for name in ("c1_s0", "low_speed"):
        e = mk.jitter_errors(name)
        assert list(e[:, 0]) == d["cases"][name]["mean_runs"]
    over = {n for n, v in d["cases"].items() if v["mean_max"] > 1e-4}
    assert over == {"s_wrap", "low_speed"}, over
