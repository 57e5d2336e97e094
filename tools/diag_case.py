"""Where a golden case's device moment error sits: the five largest
(step, rollout, component) errors of the device (oracle-noise mode) against
the reference fixture, beside the FP32-state floor at the same entries.

    python tools/diag_case.py low_speed [G]
"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path[:0] = [str(ROOT), str(ROOT / "tests")]
import numpy as np

from helpers import Inputs, channel_spread, fp32_state_floor, moments_err_arrays, unpack_moments
from paper_2408_00494_b200 import controllers as mc

name = sys.argv[1]
G = int(sys.argv[2]) if len(sys.argv) > 2 else 0
inp = Inputs(name)


class _Z:
    def standard_normal(self, shape):
        return inp.z


_c, mom = mc.rollout_bss(inp.x0, inp.cov0, mc.RolloutBatch(inp.u, inp.eps), inp.plan, inp.ctx, _Z(), inp.M,
                         precision=inp.cfg.precision, cost_weight=inp.cfg.control_cost_weight,
                         persist_particles=inp.case["persist"], moments=True, group_width=G)
g = inp.gold
ks = g["ks"]
mean, cov = unpack_moments(mom[:, ks])
spread = channel_spread(inp.noise.factor)
em, ec = moments_err_arrays(mean, cov, g["means"], g["covs"], spread)
fm, fc = fp32_state_floor(inp, ks)
fem, fec = moments_err_arrays(fm, fc, g["means"], g["covs"], spread)
alive = np.isfinite(g["costs"][ks])[None, :, None]
em = np.where(alive, em, 0)
idx = np.argsort(em.ravel())[::-1][:6]
names = ["vx", "vy", "r", "wf", "wr", "epsi", "ey", "s"]
print(f"{name} G={G}: max mean err {em.max():.2e} (floor {np.where(alive, fem, 0).max():.2e})")
for i in idx:
    t, k, c = np.unravel_index(i, em.shape)
    print(f"  t={t:3d} k={k:3d} {names[c]:5s} err {em[t, k, c]:.2e} floor {fem[t, k, c]:.2e} "
          f"dev {mean[t, k, c]:+.8e} ref {g['means'][t, k, c]:+.8e} fp32floor {fm[t, k, c]:+.8e}")
ecm = np.where(alive[..., None], ec, 0)
i = np.argmax(ecm)
t, k, a, b = np.unravel_index(i, ec.shape)
print(f"  max cov err {ecm.max():.2e} at t={t} k={k} ({a},{b}) floor {fec[t, k, a, b]:.2e}")

# the worst rollout's trajectory: device, careful FP32 port and reference
from oracle import bss_oracle as orc
rec = []
orc.rollout_bss(inp.prob, inp.x0, inp.cov0, inp.u, inp.eps, inp.plan, inp.z, inp.cfg.precision,
                inp.cfg.control_cost_weight, persist=inp.case["persist"], record=rec, dtype=np.float32, careful=True)
cm = np.stack([r[0] for r in rec])[:, ks]
t0, k0, _ = np.unravel_index(idx[0], em.shape)
print(f"  rollout k={k0}: t, (device - ref), (fp32 port - ref) for vx vy r wf wr; ref vx, vy, r")
for t in range(min(em.shape[0], t0 + 4)):
    d = mean[t, k0] - g["means"][t, k0]
    c = cm[t, k0] - g["means"][t, k0]
    print(f"   {t:3d} dev " + " ".join(f"{v:+.1e}" for v in d[:5]) + "  port " + " ".join(f"{v:+.1e}" for v in c[:5])
          + f"  ref {g['means'][t, k0, 0]:+.4e} {g['means'][t, k0, 1]:+.4e} {g['means'][t, k0, 2]:+.4e}")
