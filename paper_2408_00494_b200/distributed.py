"""K-sharded BSS-MPPI across GPUs.

Rollouts k are independent until the weighted update, so rank r of N owns a
contiguous k-range and computes, on its own GPU, the rollouts plus a partial
record {beta_r = min finite cost, Z_r, Z2_r, n_r, argmin_r, N_r[T,2]} with
weights relative to its own beta_r.  ONE collective per iteration -- an
all-reduce(SUM) of a zero-initialised [N, 5 + 2T] FP64 buffer in which each
rank fills only its slot (an all-gather in one all-reduce, 3.3 KB at T=50,
N=8) -- then every rank combines the records in rank order on its device
(rescaling by exp(-(beta_r - beta)/lambda)) and holds the identical v+.

Philox counters use the GLOBAL k, so every rollout draws the same noise at
any N; v+ differs from the single-GPU result by FP64 summation order, and by
FP32 summation order of the belief moments when a shard's lane-group width
(chosen from its local rollout count) differs from the whole problem's.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .controllers import CONTROL_DIM, Controller, _status


def shard_range(K: int, rank: int, world: int):
    """Contiguous k-range [begin, begin + count) of ``rank``; the first
    K % world ranks take one extra rollout."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    if K < world:
        raise ValueError(f"cannot shard K={K} rollouts over {world} ranks")
    base, rem = divmod(K, world)
    begin = rank * base + min(rank, rem)
    return begin, base + (1 if rank < rem else 0)


def partial_len(T: int) -> int:
    return 5 + 2 * T


class ShardedController(Controller):
    """``Controller`` whose K rollouts are split over the ranks of a
    ``torch.distributed`` process group (backend "nccl", one GPU per rank).
    ``control_step`` is collective: every rank must call it with the same
    state; all ranks return the same (u0, next plan)."""

    def __init__(self, config, cost, model, track, noise=None, subset=None, seed: int = 0,
                 run_path=(), *, group=None, device=None, noise_source: str = "philox", obstacles=None):
        import torch
        import torch.distributed as dist

        self._dist = dist
        self._torch = torch
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        if device is None:
            device = torch.cuda.current_device()
        super().__init__(config, cost, model, track, noise, subset, seed, run_path,
                         noise_source=noise_source, device=device,
                         stream=torch.cuda.current_stream(device).cuda_stream, obstacles=obstacles)
        self.partials = torch.zeros((self.world, partial_len(config.horizon)), dtype=torch.float64,
                                    device=f"cuda:{device}")

    def _k_range(self):
        return shard_range(self.config.samples, self.rank, self.world)

    def control_step(self, state, cov=None):
        dev = self._device_ctx()
        x0, cov0, plan, kc, kb, eps, z = self._inputs(state, cov)
        buf = self.partials
        buf.zero_()
        _status(dev.lib.bssmppi_step_partials(dev.h, _lib.dptr(x0), _lib.dptr(cov0), _lib.dptr(plan), kc, kb,
                                              _lib.dptr(eps), _lib.fptr(z),
                                              _lib.C.c_void_p(buf.data_ptr()), self.rank))
        self._dist.all_reduce(buf, group=self.group)
        vplus = np.empty((self.config.horizon, CONTROL_DIM))
        diag = _lib.Diag()
        _status(dev.lib.bssmppi_update_combine(dev.h, _lib.C.c_void_p(buf.data_ptr()), self.world,
                                               _lib.dptr(vplus), _lib.C.byref(diag)))
        return self._finish(vplus, diag)

    # device-resident loop (bench): partials -> all-reduce -> combine, async
    def enqueue_iteration(self, key_ctrl, key_belief):
        dev = self._device_ctx()
        buf = self.partials
        buf.zero_()
        _lib.check(dev.lib.bssmppi_enqueue_partials(dev.h, _lib.key_arr(key_ctrl), _lib.key_arr(key_belief),
                                                    _lib.C.c_void_p(buf.data_ptr()), self.rank))
        self._dist.all_reduce(buf, group=self.group)
        _lib.check(dev.lib.bssmppi_enqueue_combine(dev.h, _lib.C.c_void_p(buf.data_ptr()), self.world))
