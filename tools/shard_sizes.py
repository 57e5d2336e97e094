"""Device time of one iteration for the K-shard a rank owns at N GPUs (K/N
rollouts of a bench workload: C3, C4, C5:K:M), measured on one B200 through
bssmppi_step_partials + bssmppi_update_combine (N records combined).
Projects strong scaling without the ~10-20 us NCCL all-reduce of the
[N, 5 + 2T] record buffer.

    python tools/shard_sizes.py [workload ...]   ->  gpurun_out/shard_sizes.json
"""
import json
import sys

sys.path.insert(0, ".")
import numpy as np
import torch

import bench
from paper_2408_00494_b200 import _lib
from paper_2408_00494_b200 import controllers as mc
from paper_2408_00494_b200 import streams
from paper_2408_00494_b200.distributed import shard_range


def workload(name):
    if name.startswith("C5:"):
        _, k, m = name.split(":")
        return dict(K=int(k), M=int(m), T=60, dt=0.04, track="spline0", noise_std=0.05)   # as bench.py
    return bench.WORKLOADS[name]


def project(name):
    wl = workload(name)
    cfg, cost, model, track, noise, x0, obstacles = bench.build_problem_objects(wl)
    K, M, T = wl["K"], wl["M"], wl["T"]
    rows, base = [], None
    for n in (1, 2, 4, 8):
        b, kn = shard_range(K, n - 1, n)       # the last (smallest) shard
        ctx = mc.RolloutContext(model, track, cost, noise=noise, obstacles=obstacles)
        prob, keep = mc.build_problem("bss", K, T, M, cfg.temperature, cfg.control_cost_weight, cfg.sigma_eps,
                                      cfg.precision, cfg.bounds, False, ctx, b, kn)
        dc = mc.DeviceContext(prob)
        buf = torch.zeros((n, dc.lib.bssmppi_partial_len(T)), dtype=torch.float64, device="cuda")
        plan = np.zeros((T, 2))
        ms = []
        for i in range(25):
            kc = _lib.key_arr(streams.device_key(0, 2, i))
            kb = _lib.key_arr(streams.device_key(0, 3, i))
            _lib.check(dc.lib.bssmppi_step_partials(dc.h, _lib.dptr(x0), None, _lib.dptr(plan), kc, kb, None, None,
                                                    _lib.C.c_void_p(buf.data_ptr()), n - 1))
            d = _lib.Diag()
            v = np.empty((T, 2))
            _lib.check(dc.lib.bssmppi_update_combine(dc.h, _lib.C.c_void_p(buf.data_ptr()), n, _lib.dptr(v),
                                                     _lib.C.byref(d)))
            if i >= 5:
                ms.append(d.device_ms)
        t = float(np.median(ms))
        base = base or t
        rows.append(dict(workload=name, n_gpus=n, k_local=kn, device_ms=t, projected_speedup=base / t,
                         efficiency=base / t / n))
        print(json.dumps(rows[-1]), flush=True)
        dc.close()
    return rows


if __name__ == "__main__":
    names = sys.argv[1:] or ["C3"]
    out = [r for name in names for r in project(name)]
    json.dump(out, open("gpurun_out/shard_sizes.json", "w"), indent=1)
