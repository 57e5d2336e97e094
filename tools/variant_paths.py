"""Device time of the secondary paths at BASELINE shapes (Philox mode): the
deterministic kinds (mppi, smppi), persist-particles BSS, BSS with a general
(non-diagonal) process-noise factor and BSS without process noise, beside the
hot path (re-projection, diagonal noise).  One line per path."""
import sys
sys.path.insert(0, ".")
import numpy as np
from paper_2408_00494_b200 import controllers as mc, dynamics as md, _lib, streams
from paper_2408_00494_b200.tracks import named_track


def run(name, K, M, T, dt, track, kind="bss", persist=False, noise=None, iters=20):
    model = md.with_timestep(md.VehicleParams(), dt, "euler")
    cfg = mc.MppiConfig(kind=kind, samples=K, horizon=T, inner_samples=M,
                        sigma_eps=np.diag([0.2 ** 2, 0.5 ** 2]), persist_particles=persist)
    if noise is None:
        noise = md.NoiseModel(np.diag([0.05 ** 2] * 3))
    ctrl = mc.Controller(cfg, mc.CostSpec(), model, named_track(track), noise=noise, seed=0, run_path=(5, 0))
    x0 = md.VehicleState.rolling(5.0, model, s=10.0).as_array()
    for _ in range(3):
        ctrl.control_step(x0)
    dev = ctrl._device_ctx()
    lib = dev.lib
    plan = np.ascontiguousarray(ctrl.plan.controls)
    _lib.check(lib.bssmppi_upload_state(dev.h, _lib.dptr(x0), None, _lib.dptr(plan)))
    ms, d = [], _lib.Diag()
    for i in range(iters):
        kc = _lib.key_arr(streams.device_key(0, 5, 0, 2, 100 + i))
        kb = _lib.key_arr(streams.device_key(0, 5, 0, 3, 100 + i))
        _lib.check(lib.bssmppi_enqueue_iteration(dev.h, kc, kb))
        _lib.check(lib.bssmppi_download(dev.h, None, _lib.C.byref(d)))
        ms.append(d.device_ms)
    med = float(np.median(ms))
    units = K * T * (M if kind == "bss" else 1)
    g, b = ctrl.launch_shape()
    print(f"{name}: K={K} M={M if kind == 'bss' else 1} T={T} G={g} block={b} device {med:.3f} ms  "
          f"{units / med / 1e6:.2f} G dynamics steps/s  nfin {d.n_finite}", flush=True)


full = np.array([[0.05, 0.0, 0.0], [0.01, 0.05, 0.0], [0.0, 0.02, 0.05]])
run("C3 bss (hot path)", 16384, 256, 50, 0.04, "spline0")
run("C3 bss, general 3x3 noise factor", 16384, 256, 50, 0.04, "spline0", noise=md.NoiseModel(full @ full.T))
run("C3 bss, no process noise", 16384, 256, 50, 0.04, "spline0", noise=md.NoiseModel(np.zeros((3, 3))))
run("C3 bss, persist particles", 16384, 256, 50, 0.04, "spline0", persist=True)
run("C2 bss, persist particles", 4096, 128, 40, 0.05, "ellipse", persist=True)
run("C3-shape smppi", 16384, 1, 50, 0.04, "spline0", kind="smppi")
run("C3-shape mppi", 16384, 1, 50, 0.04, "spline0", kind="mppi")
run("131072 smppi", 131072, 1, 60, 0.04, "spline0", kind="smppi")
