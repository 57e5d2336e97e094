"""World-size-2 gloo test of the K-sharded update on CPU:
each rank builds the partial record of its shard, ONE all-reduce(SUM) of the
zero-initialised rank-slotted buffer gathers them, and the rank-order
combine reproduces the unsharded reference update on every rank."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from cases import update_batch

from oracle import bss_oracle as orc
from paper_2408_00494_b200.distributed import partial_len, shard_range

LO, HI = np.array([-0.35, -1.0]), np.array([0.35, 1.0])


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, j, out):
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    costs, controls, lam = update_batch(j)
    K, T, _ = controls.shape
    b, n = shard_range(K, rank, world)
    buf = torch.zeros((world, partial_len(T)), dtype=torch.float64)
    buf[rank] = torch.from_numpy(orc.shard_record(costs[b:b + n], controls[b:b + n], lam, b))
    dist.all_reduce(buf)
    v = orc.combine_records(buf.numpy(), lam, LO, HI)
    out[rank] = v
    dist.destroy_process_group()


@pytest.mark.parametrize("j", [0, 1, 2])
def test_two_rank_sharded_update_matches_unsharded(j):
    world = 2
    mgr = mp.get_context("spawn").Manager()
    out = mgr.dict()
    mp.start_processes(_worker, args=(world, _free_port(), j, out), nprocs=world, join=True,
                       start_method="spawn")
    costs, controls, lam = update_batch(j)
    ref = orc.mppi_update(costs, controls, lam, LO, HI)
    for r in range(world):
        np.testing.assert_allclose(out[r], ref, rtol=0, atol=1e-12)
    np.testing.assert_array_equal(out[0], out[1])


def test_single_record_is_plain_update():
    costs, controls, lam = update_batch(1)
    rec = orc.shard_record(costs, controls, lam)
    np.testing.assert_allclose(orc.combine_records(rec[None], lam, LO, HI),
                               orc.mppi_update(costs, controls, lam, LO, HI), atol=1e-13)
    assert rec[4] == int(np.argmin(costs))
