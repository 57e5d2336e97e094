"""Where the e2e time of Controller.control_step goes at small K (C1)."""
import sys, time
sys.path.insert(0, ".")
import numpy as np
from paper_2408_00494_b200 import controllers as mc, dynamics as md, streams, _lib
from paper_2408_00494_b200.tracks import named_track
model = md.with_timestep(md.VehicleParams(), 0.05, "euler")
cfg = mc.MppiConfig(kind="bss", samples=256, horizon=20, inner_samples=32, sigma_eps=np.diag([0.04, 0.25]))
ctrl = mc.Controller(cfg, mc.CostSpec(), model, named_track("ellipse"), noise=md.NoiseModel(np.diag([0.03**2]*3)))
x0 = md.VehicleState.rolling(5.0, model, s=10.0).as_array()
for _ in range(20): ctrl.control_step(x0)
N = 300
def t(f):
    t0 = time.perf_counter()
    for _ in range(N): f()
    return (time.perf_counter() - t0) / N * 1e6
print("control_step total  %.1f us" % t(lambda: ctrl.control_step(x0)))
print("device_key x2       %.1f us" % t(lambda: (streams.device_key(0, 5, 0, 2, 7), streams.device_key(0, 5, 0, 3, 7))))
print("_inputs              %.1f us" % t(lambda: ctrl._inputs(x0, None)))
dev = ctrl._device_ctx(); x, c, p, kc, kb, e, z = ctrl._inputs(x0, None)
v = np.empty((20, 2)); d = _lib.Diag()
print("C ABI call only      %.1f us" % t(lambda: dev.lib.bssmppi_control_step(dev.h, _lib.dptr(x), None, _lib.dptr(p), kc, kb, None, None, _lib.dptr(v), _lib.C.byref(d))))
print("device_ms            %.1f us" % (1e3 * d.device_ms))
