"""The world-size-2 K-sharded controller end to end on one GPU: two
processes, gloo backend (the all-reduce of the CUDA partial-record buffer
is staged through the host, so no kernel of one rank waits on the other),
each rank owning half of K.  Every rank returns the same (u0, plan) as the
single-process controller, step after step: to 1e-12 when the shard picks
the same group width G as the whole problem (M = 256: one warp per rollout
at K = 2048 and 1024), and within the v+ parity bound when the local group
width differs (M = 64: G = 16 unsharded, 32 per shard), which changes only
the FP32 summation order of the belief moments."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _setup(M=256):
    from paper_2408_00494_b200 import controllers as mc, dynamics as md
    from paper_2408_00494_b200.tracks import named_track
    model = md.with_timestep(md.VehicleParams(), 0.05, "euler")
    cfg = mc.MppiConfig(kind="bss", samples=2048, horizon=20, inner_samples=M,
                        sigma_eps=np.diag([0.2 ** 2, 0.5 ** 2]))
    x0 = md.VehicleState.rolling(5.0, model, s=12.0).as_array()
    return cfg, mc.CostSpec(), model, named_track("ellipse"), md.NoiseModel(np.diag([0.03 ** 2] * 3)), x0


def _rank(rank, world, port, noise_source, M, out):
    import torch
    import torch.distributed as dist
    from paper_2408_00494_b200.distributed import ShardedController
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    cfg, cost, model, track, noise, x0 = _setup(M)
    ctrl = ShardedController(cfg, cost, model, track, noise=noise, seed=9, run_path=(5, 9), device=0,
                             noise_source=noise_source)
    us = []
    for _ in range(4):
        u0, plan = ctrl.control_step(x0)
        us.append(np.concatenate([u0, plan.controls.ravel()]))
    out[rank] = (np.array(us), ctrl._k_range())
    dist.destroy_process_group()


@pytest.mark.parametrize("noise_source,M,atol", [("philox", 256, 1e-12), ("reference", 256, 1e-12),
                                                  ("philox", 64, 1e-4)])
def test_two_rank_sharded_equals_single(noise_source, M, atol):
    from paper_2408_00494_b200 import _lib
    from paper_2408_00494_b200 import controllers as mc
    gw = _lib.load().bssmppi_group_width
    assert (gw(M, 2048) == gw(M, 1024)) == (atol < 1e-6)
    cfg, cost, model, track, noise, x0 = _setup(M)
    single = mc.Controller(cfg, cost, model, track, noise=noise, seed=9, run_path=(5, 9),
                           noise_source=noise_source)
    ref = []
    for _ in range(4):
        u0, plan = single.control_step(x0)
        ref.append(np.concatenate([u0, plan.controls.ravel()]))
    ref = np.array(ref)
    single.close()
    mgr = mp.get_context("spawn").Manager()
    out = mgr.dict()
    mp.start_processes(_rank, args=(2, _port(), noise_source, M, out), nprocs=2, join=True, start_method="spawn")
    assert out[0][1] == (0, 1024) and out[1][1] == (1024, 1024)
    np.testing.assert_array_equal(out[0][0], out[1][0])       # identical v+ on every rank
    np.testing.assert_allclose(out[0][0], ref, rtol=0, atol=atol)
