"""Measured FP32 resolution of each BSS golden case (test infrastructure for
tests/test_gpu_parity.py moment_tolerance; run in the build container):

    python tests/golden/make_fp32_floor.py  ->  tests/golden/fp32_floor.json

For every case, R = 8 runs of a careful FP32 port of the reference
algorithm (oracle/bss_oracle.py rollout_bss(dtype=float32, careful=True):
everything in FP32 except the literal heading-wrap formula), each with a
different but equally valid rounding of the belief mean -- +-1 FP32 ulp on
every nonzero mean component after each step, at random -- and the SURVEY
8c moment errors of each run against the reference fixture.  The spread of
these errors is what FP32 itself allows on the case: on well-conditioned
cases it stays far below 1e-4; on the chaotic low-speed case (explicit Euler
at the v_floor regularisation, errors grow ~2.5x per step) it reaches it.
"""

import json
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
sys.path[:0] = [str(HERE.parent), str(HERE.parent.parent)]

import numpy as np

from cases import CASES
from helpers import Inputs, channel_spread, moments_rel_err
from oracle import bss_oracle as orc

R = 8


def jitter_errors(name):
    inp = Inputs(name)
    g = inp.gold
    ks = g["ks"]
    alive = np.broadcast_to(np.isfinite(g["costs"][ks])[None, :], (g["means"].shape[0], len(ks)))
    orig = orc.moments
    out = []
    for r in range(R):
        rng = np.random.default_rng(1000 + r)

        def jittered(x1):
            m, c = orig(x1)
            ulp = np.spacing(np.abs(m).astype(np.float32)).astype(m.dtype)
            step = rng.integers(-1, 2, m.shape) * (m != 0)
            return m + ulp * step, c

        orc.moments = jittered
        try:
            rec = []
            orc.rollout_bss(inp.prob, inp.x0, inp.cov0, inp.u, inp.eps, inp.plan, inp.z, inp.cfg.precision,
                            inp.cfg.control_cost_weight, persist=inp.case["persist"], record=rec,
                            dtype=np.float32, careful=True)
        finally:
            orc.moments = orig
        m, c = np.stack([q[0] for q in rec]), np.stack([q[1] for q in rec])
        # rollouts alive in the reference and in this run (a rounding choice
        # can move a frame-edge rollout's death by a step)
        ok = alive & np.isfinite(m[:, ks]).all(-1) & np.all(np.stack([q[2] for q in rec])[:, ks], axis=0)[None]
        out.append(moments_rel_err(m[:, ks][ok], c[:, ks][ok], g["means"][ok], g["covs"][ok],
                                   channel_spread(inp.noise.factor)))
    return np.array(out)


def main():
    res = {}
    for case in CASES:
        if case["kind"] != "bss":
            continue
        e = jitter_errors(case["name"])
        res[case["name"]] = {"mean_max": float(e[:, 0].max()), "cov_max": float(e[:, 1].max()),
                             "mean_runs": [float(v) for v in e[:, 0]], "cov_runs": [float(v) for v in e[:, 1]]}
        print(f"{case['name']:14s} mean {e[:, 0].max():.2e} cov {e[:, 1].max():.2e}", flush=True)
    (HERE / "fp32_floor.json").write_text(json.dumps({"runs": R, "cases": res}, indent=1))


if __name__ == "__main__":
    main()
