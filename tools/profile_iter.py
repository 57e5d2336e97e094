"""Run N philox-mode iterations of one shape (for ncu capture)."""
import argparse, sys
sys.path.insert(0, ".")
import numpy as np
from paper_2408_00494_b200 import controllers as mc, dynamics as md
from paper_2408_00494_b200.tracks import named_track

ap = argparse.ArgumentParser()
ap.add_argument("--K", type=int, default=16384)
ap.add_argument("--M", type=int, default=256)
ap.add_argument("--T", type=int, default=50)
ap.add_argument("--dt", type=float, default=0.04)
ap.add_argument("--track", default="spline0")
ap.add_argument("--iters", type=int, default=2)
a = ap.parse_args()
model = md.with_timestep(md.VehicleParams(), a.dt, "euler")
cfg = mc.MppiConfig(kind="bss", samples=a.K, horizon=a.T, inner_samples=a.M,
                    sigma_eps=np.diag([0.2**2, 0.5**2]))
ctrl = mc.Controller(cfg, mc.CostSpec(), model, named_track(a.track),
                     noise=md.NoiseModel(np.diag([0.05**2]*3)), seed=0, run_path=(5, 0))
x0 = md.VehicleState.rolling(5.0, model, s=10.0).as_array()
for _ in range(a.iters):
    ctrl.control_step(x0)
print("ok", ctrl.last_diagnostics["device_ms"])
