"""Small end-to-end exercise of every kernel for compute-sanitizer."""
import sys
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np
from helpers import Inputs
from test_gpu_parity import _gpu_rollout
from paper_2408_00494_b200 import controllers as mc, dynamics as md
from paper_2408_00494_b200.tracks import named_track
for name in ["c1_s0", "persist", "ragged_m5", "smppi", "dead", "collapse_m2"]:
    inp = Inputs(name)
    out = _gpu_rollout(inp, moments=inp.kind == "bss")
    ctrl = mc.Controller(inp.cfg, inp.cost, inp.model, inp.track, noise=inp.noise, seed=1, run_path=(2,))
    try:
        ctrl.control_step(inp.x0, inp.cov0)
    except mc.AllRolloutsInvalid:
        pass
    ctrl.close()
model = md.with_timestep(md.VehicleParams(), 0.04, "euler")
cfg = mc.MppiConfig(kind="bss", samples=16384, horizon=10, inner_samples=256, sigma_eps=np.diag([0.04, 0.25]))
c = mc.Controller(cfg, mc.CostSpec(), model, named_track("spline0"), noise=md.NoiseModel(np.diag([0.0025] * 3)))
c.control_step(md.VehicleState.rolling(5.0, model, s=3.0).as_array())
print("sanitize run ok")
