"""Device time per iteration vs forced group width G for one (K, M, T)
shape:  python tools/g_sweep.py K M T [G]   (G = 0 or absent: the policy)."""
import os, sys
sys.path.insert(0, ".")
import numpy as np
from paper_2408_00494_b200 import controllers as mc, dynamics as md, _lib
from paper_2408_00494_b200.tracks import named_track

K, M, T = (int(v) for v in sys.argv[1:4])
G_FORCE = int(sys.argv[4]) if len(sys.argv) > 4 else 0
model = md.with_timestep(md.VehicleParams(), 0.04, "euler")
cfg = mc.MppiConfig(kind="bss", samples=K, horizon=T, inner_samples=M, sigma_eps=np.diag([0.04, 0.25]))
ctrl = mc.Controller(cfg, mc.CostSpec(), model, named_track("spline0"),
                     noise=md.NoiseModel(np.diag([0.05 ** 2] * 3)), seed=0, run_path=(5, 0),
                     group_width=G_FORCE)
x0 = md.VehicleState.rolling(5.0, model, s=10.0).as_array()
ctrl.upload_state(x0)
keys = [((1, i), (2, i)) for i in range(40)]
for i in range(5):
    ctrl.enqueue_iteration(*keys[i])
ctrl.download()
ms = []
for i in range(5, 40):
    ctrl.enqueue_iteration(*keys[i])
    _, d = ctrl.download()
    ms.append(d["device_ms"])
g, _ = ctrl.launch_shape()
print(f"K={K} M={M} T={T} G={g} device {np.median(ms):.3f} ms  {K * M * T / np.median(ms) / 1e6:.1f} G/s")
