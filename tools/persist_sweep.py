import sys
sys.path.insert(0, ".")
import numpy as np
from paper_2408_00494_b200 import controllers as mc, dynamics as md, _lib
from paper_2408_00494_b200.tracks import named_track
def run(K, M, T, G):
    model = md.with_timestep(md.VehicleParams(), 0.04, "euler")
    cfg = mc.MppiConfig(kind="bss", samples=K, horizon=T, inner_samples=M, sigma_eps=np.diag([0.04, 0.25]), persist_particles=True)
    ctrl = mc.Controller(cfg, mc.CostSpec(), model, named_track("spline0"), noise=md.NoiseModel(np.diag([0.05 ** 2] * 3)), seed=0, run_path=(5, 0), group_width=G)
    x0 = md.VehicleState.rolling(5.0, model, s=10.0).as_array()
    ctrl.upload_state(x0)
    keys = [((1, i), (2, i)) for i in range(20)]
    for i in range(3): ctrl.enqueue_iteration(*keys[i])
    ctrl.download()
    ms = []
    for i in range(3, 20):
        ctrl.enqueue_iteration(*keys[i]); _, d = ctrl.download(); ms.append(d["device_ms"])
    g, b = ctrl.launch_shape()
    print(f"persist K={K} M={M} T={T} G={g} block={b} device {np.median(ms):.3f} ms {K*M*T/np.median(ms)/1e6:.1f} G/s", flush=True)
for K, M, T in [(16384, 256, 50), (4096, 128, 40), (256, 32, 20), (4096, 64, 60)]:
    for G in (0, 4, 8, 16, 32):
        try: run(K, M, T, G)
        except Exception as e: print("fail", K, M, G, e)
