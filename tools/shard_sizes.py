"""Device time of one C3 iteration for the K-shard a rank owns at N GPUs
(K/N rollouts, same M, T, track): projects strong scaling without the
~10-20 us NCCL all-reduce of the 3.3 KB record buffer."""
import json, sys
sys.path.insert(0, ".")
import numpy as np
from paper_2408_00494_b200 import controllers as mc, dynamics as md, streams
from paper_2408_00494_b200.distributed import shard_range
from paper_2408_00494_b200.tracks import named_track

model = md.with_timestep(md.VehicleParams(), 0.04, "euler")
track = named_track("spline0")
noise = md.NoiseModel(np.diag([0.05 ** 2] * 3))
x0 = md.VehicleState.rolling(5.0, model, s=10.0).as_array()
rows = []
base = None
for n in (1, 2, 4, 8):
    b, kn = shard_range(16384, n - 1, n)
    ctx = mc.RolloutContext(model, track, mc.CostSpec(), noise=noise)
    cfg = mc.MppiConfig(kind="bss", samples=16384, horizon=50, inner_samples=256, sigma_eps=np.diag([0.04, 0.25]))
    prob, keep = mc.build_problem("bss", 16384, 50, 256, 1.0, 0.1, cfg.sigma_eps, cfg.precision, cfg.bounds,
                                  False, ctx, b, kn)
    dc = mc.DeviceContext(prob)
    import torch
    R = dc.lib.bssmppi_partial_len(50)
    buf = torch.zeros((n, R), dtype=torch.float64, device="cuda")
    from paper_2408_00494_b200 import _lib
    plan = np.zeros((50, 2))
    ms = []
    for i in range(25):
        kc = _lib.key_arr(streams.device_key(0, 2, i)); kb = _lib.key_arr(streams.device_key(0, 3, i))
        _lib.check(dc.lib.bssmppi_step_partials(dc.h, _lib.dptr(x0), None, _lib.dptr(plan), kc, kb, None, None,
                                                _lib.C.c_void_p(buf.data_ptr()), n - 1))
        d = _lib.Diag()
        v = np.empty((50, 2))
        _lib.check(dc.lib.bssmppi_update_combine(dc.h, _lib.C.c_void_p(buf.data_ptr()), n, _lib.dptr(v),
                                                 _lib.C.byref(d)))
        if i >= 5:
            ms.append(d.device_ms)
    t = float(np.median(ms))
    base = base or t
    rows.append(dict(n_gpus=n, k_local=kn, device_ms=t, projected_speedup=base / t, efficiency=base / t / n))
    print(json.dumps(rows[-1]), flush=True)
    dc.close()
json.dump(rows, open("gpurun_out/shard_sizes.json", "w"), indent=1)
