"""Experiment: C3 as TWO concurrent K-shards with different lane-group widths
(G = 8 for most rollouts, G = 16 for the rest) so that the warps of both
launches fill whole waves of 148 SMs x 16 warps, against the single G = 8
launch (1.73 waves).  Times the rollout part only (enqueue_partials on two
streams), CUDA events around both."""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
import bench
from paper_2408_00494_b200 import _lib, controllers as mc, streams


def make(K, T, M, b, kn, G, cfg, cost, model, track, noise, stream):
    ctx = mc.RolloutContext(model, track, cost, noise=noise)
    prob, keep = mc.build_problem("bss", K, T, M, cfg.temperature, cfg.control_cost_weight, cfg.sigma_eps,
                                  cfg.precision, cfg.bounds, False, ctx, b, kn, group_width=G)
    dc = mc.DeviceContext(prob)
    _lib.check(dc.lib.bssmppi_set_stream(dc.h, _lib.C.c_void_p(stream.cuda_stream)))
    return dc, keep


def main():
    wl = bench.WORKLOADS["C3"]
    cfg, cost, model, track, noise, x0, _ = bench.build_problem_objects(wl)
    K, M, T = wl["K"], wl["M"], wl["T"]
    plan = np.zeros((T, 2))
    s0, s1 = torch.cuda.Stream(), torch.cuda.Stream()
    for ka, ga, gb in [(K, 8, 8), (13824, 8, 16), (12288, 8, 16), (14848, 8, 32), (9472, 8, 16), (9472, 8, 8)]:
        parts = [(0, ka, ga, s0)] + ([(ka, K - ka, gb, s1)] if ka < K else [])
        dcs = [make(K, T, M, b, kn, G, cfg, cost, model, track, noise, st) for b, kn, G, st in parts]
        bufs = [torch.zeros((2, dc.lib.bssmppi_partial_len(T)), dtype=torch.float64, device="cuda") for dc, _ in dcs]
        for dc, _ in dcs:
            _lib.check(dc.lib.bssmppi_upload_state(dc.h, _lib.dptr(x0), None, _lib.dptr(plan)))
        torch.cuda.synchronize()
        ms = []
        for i in range(25):
            kc = _lib.key_arr(streams.device_key(0, 2, i))
            kb = _lib.key_arr(streams.device_key(0, 3, i))
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s0)
            s1.wait_event(e0)
            for j, ((dc, _), buf) in enumerate(zip(dcs, bufs)):
                _lib.check(dc.lib.bssmppi_enqueue_partials(dc.h, kc, kb, _lib.C.c_void_p(buf.data_ptr()), j))
            done = torch.cuda.Event()
            done.record(s1)
            s0.wait_event(done)
            e1.record(s0)
            torch.cuda.synchronize()
            if i >= 5:
                ms.append(e0.elapsed_time(e1))
        print(f"K_a={ka} (G={ga}) + K_b={K - ka} (G={gb}): {np.median(ms):.3f} ms", flush=True)
        for dc, _ in dcs:
            dc.close()


main()
