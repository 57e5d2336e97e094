"""Quick device timing of one BSS-MPPI iteration at several shapes."""
import sys, time
sys.path.insert(0, ".")
import numpy as np
from paper_2408_00494_b200 import controllers as mc, dynamics as md, _lib, streams
from paper_2408_00494_b200.tracks import named_track

def run(name, K, M, T, dt, track, iters=20):
    model = md.with_timestep(md.VehicleParams(), dt, "euler")
    tr = named_track(track)
    cfg = mc.MppiConfig(kind="bss", samples=K, horizon=T, inner_samples=M,
                        sigma_eps=np.diag([0.2**2, 0.5**2]))
    noise = md.NoiseModel(np.diag([0.05**2]*3))
    ctrl = mc.Controller(cfg, mc.CostSpec(), model, tr, noise=noise, seed=0, run_path=(5, 0))
    x0 = md.VehicleState.rolling(5.0, model, s=10.0).as_array()
    for _ in range(3):
        ctrl.control_step(x0)
    dev = ctrl._device_ctx()
    lib = dev.lib
    plan = np.ascontiguousarray(ctrl.plan.controls)
    _lib.check(lib.bssmppi_upload_state(dev.h, _lib.dptr(x0), None, _lib.dptr(plan)))
    ms = []
    d = _lib.Diag()
    for i in range(iters):
        kc = _lib.key_arr(streams.device_key(0, 5, 0, 2, 100 + i))
        kb = _lib.key_arr(streams.device_key(0, 5, 0, 3, 100 + i))
        _lib.check(lib.bssmppi_enqueue_iteration(dev.h, kc, kb))
        _lib.check(lib.bssmppi_download(dev.h, None, _lib.C.byref(d)))
        ms.append(d.device_ms)
    t0 = time.perf_counter()
    for _ in range(iters):
        ctrl.control_step(x0)
    wall = (time.perf_counter() - t0) / iters * 1e3
    med = float(np.median(ms))
    ps = K * M * T
    print(f"{name}: K={K} M={M} T={T} device {med:.3f} ms  e2e {wall:.3f} ms  "
          f"{ps/med/1e6:.3f} G particle-steps/s  ess {d.ess:.2f} nfin {d.n_finite}", flush=True)

run("C1", 256, 32, 20, 0.05, "ellipse")
run("C2", 4096, 128, 40, 0.05, "ellipse")
run("C3", 16384, 256, 50, 0.04, "spline0")
run("C5a", 4096, 512, 60, 0.04, "spline0")
run("C5b", 32768, 64, 60, 0.04, "spline0")
run("S8", 2048, 256, 50, 0.04, "spline0")
