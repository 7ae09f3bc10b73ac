"""Batch sharding of independent Hamiltonians across GPUs.

One process per GPU (torchrun).  The batch is split into contiguous shards, each
rank runs the whole MLSP2 pipeline on its shard with no data-path collective, and
the fixed-size per-matrix result records {Tr D, Tr D^2, status} are gathered to
every rank with one NCCL all-gather (C1 in SURVEY.md 2.2).  D stays on the GPU
that computed it.  The same code runs over gloo on CPU for the host-logic tests,
with a caller-supplied `compute` in place of the device pipeline.
"""
from __future__ import annotations

from typing import Callable, Sequence

import numpy as np

RECORD = 4  # float64 fields per matrix: trace, trace_square, status, global index


def shard_range(total: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous shard [lo, hi) of `total` items for `rank`; sizes differ by at most one."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError(f"bad world/rank {world}/{rank}")
    base, extra = divmod(total, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def max_shard(total: int, world: int) -> int:
    return -(-total // world)


class ResultGather:
    """All-gather of per-matrix result records (padded to the largest shard)."""

    def __init__(self, world: int, rank: int, per_rank: int, device, total: int | None = None):
        import torch

        self.world, self.rank, self.per_rank = world, rank, per_rank
        self.total = total if total is not None else per_rank * world
        self.device = device
        self.local = torch.full((per_rank, RECORD), -1.0, dtype=torch.float64, device=device)
        self.all = torch.empty((world * per_rank, RECORD), dtype=torch.float64, device=device)

    def gather(self, stats, status, count: int | None = None, offset: int | None = None):
        """stats [b,2] f64, status [b] int -> (stats [total,2], status [total]) on every rank."""
        import torch
        import torch.distributed as dist

        b = stats.shape[0] if count is None else count
        lo = shard_range(self.total, self.world, self.rank)[0] if offset is None else offset
        self.local.fill_(-1.0)
        self.local[:b, 0:2] = stats[:b]
        self.local[:b, 2] = status[:b].to(torch.float64)
        self.local[:b, 3] = torch.arange(lo, lo + b, dtype=torch.float64, device=self.device)
        if self.world > 1:
            dist.all_gather_into_tensor(self.all, self.local)
        else:
            self.all.copy_(self.local)
        return self.all

    @staticmethod
    def unpack(all_records, total: int):
        """Records -> (stats [total,2], status [total]) ordered by global index."""
        rec = all_records.detach().cpu().numpy()
        rec = rec[rec[:, 3] >= 0]
        order = np.argsort(rec[:, 3], kind="stable")
        rec = rec[order]
        if rec.shape[0] != total or not np.array_equal(rec[:, 3], np.arange(total)):
            raise RuntimeError("result gather lost or duplicated records")
        return rec[:, 0:2].copy(), rec[:, 2].astype(np.int32)


def sharded_density_matrices(H_global: Sequence[np.ndarray], mu, kT, model=None, mode=None,
                             compute: Callable | None = None, device=None):
    """Run the batch sharded over the current process group; every rank gets all stats.

    compute(H_dev [b,n,n] f64 tensor, mu [b], kT [b]) -> (stats [b,2], status [b]) tensors;
    default: the B200 pipeline (engine.compute_density_matrices_device).
    """
    import torch
    import torch.distributed as dist

    world = dist.get_world_size() if dist.is_initialized() else 1
    rank = dist.get_rank() if dist.is_initialized() else 0
    G = len(H_global)
    mu = np.broadcast_to(np.asarray(mu, dtype=np.float64), (G,))
    kT = np.broadcast_to(np.asarray(kT, dtype=np.float64), (G,))
    lo, hi = shard_range(G, world, rank)
    if compute is None:
        from . import engine as E

        mode = E.PrecisionMode.MIXED_EMULATED if mode is None else mode

        def compute(Hd, m_, k_):
            s, st, _ = E.compute_density_matrices_device(Hd, m_, k_, model, mode)
            return s, st
        device = device or torch.device("cuda", torch.cuda.current_device())
    device = device or torch.device("cpu")
    g = ResultGather(world, rank, max_shard(G, world), device, total=G)
    if hi > lo:
        Hd = torch.from_numpy(np.stack([np.asarray(h, dtype=np.float64) for h in H_global[lo:hi]])).to(device)
        stats, status = compute(Hd, mu[lo:hi], kT[lo:hi])
    else:
        stats = torch.zeros((0, 2), dtype=torch.float64, device=device)
        status = torch.zeros((0,), dtype=torch.int32, device=device)
    recs = g.gather(stats, status, count=hi - lo, offset=lo)
    return ResultGather.unpack(recs, G)
