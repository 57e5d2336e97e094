"""Analyse gpurun_out/parity_dump.npz (tools/parity_dump.py) against the
golden fixtures: cost errors and the SURVEY 8c moment metric (no floor) per
case and lane-group width, beside the FP32-state floor of the reference's
own algorithm (oracle rollout_bss(round_state=float32): FP64 arithmetic,
particle states rounded to FP32 after every re-projection and step)."""
import sys
sys.path.insert(0, 'tests'); sys.path.insert(0, '.')
import numpy as np
from cases import CASES
from helpers import Inputs, channel_spread, moments_rel_err, unpack_moments
from oracle import bss_oracle as orc

d = np.load(sys.argv[1] if len(sys.argv) > 1 else 'gpurun_out/parity_dump.npz')


def fp32_floor(inp):
    rec = []
    orc.rollout_bss(inp.prob, inp.x0, inp.cov0, inp.u, inp.eps, inp.plan, inp.z, inp.cfg.precision,
                    inp.cfg.control_cost_weight, persist=inp.case['persist'], record=rec,
                    round_state=np.float32)
    return np.stack([r[0] for r in rec]), np.stack([r[1] for r in rec])


print(f"{'case':14s} {'M':>4s} {'cost':>8s} | moments mean/cov at G = policy, 4, 8, 16, 32 | fp32-state floor")
for c in CASES:
    name = c['name']
    inp = Inputs(name); g = inp.gold
    costs = d[name + '__costs']; ref = g['costs']; fin = np.isfinite(ref)
    rel = np.abs(costs[fin] - ref[fin]) / np.abs(ref[fin]) if fin.any() else np.zeros(1)
    line = f"{name:14s} {inp.M:4d} {rel.max():8.1e} |"
    if inp.kind != 'bss':
        print(line)
        continue
    ks = g['ks']
    alive = np.broadcast_to(np.isfinite(g['costs'][ks])[None, :], (g['means'].shape[0], len(ks)))
    for gw in (0, 4, 8, 16, 32):
        mean, cov = unpack_moments(d[f"{name}__mom__g{gw}"][:, ks])
        em, ec = moments_rel_err(mean[alive], cov[alive], g['means'][alive], g['covs'][alive],
                                 channel_spread(inp.noise.factor))
        line += f" {em:.1e}/{ec:.1e}"
    fm, fc = fp32_floor(inp)
    em, ec = moments_rel_err(fm[:, ks][alive], fc[:, ks][alive], g['means'][alive], g['covs'][alive],
                             channel_spread(inp.noise.factor))
    print(line + f" | {em:.1e}/{ec:.1e}")
