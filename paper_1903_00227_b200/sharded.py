"""Sharded PSA sampling across the GPUs of one box (one process per GPU).

Design: rank g of G owns the contiguous item shard
[g*ceil(n/G), min(n, (g+1)*ceil(n/G))) -- the reference's TwoLevelTable group
rule (two_level.hpp:33-41) -- and builds an ordinary PSA table over it with
local ids.  The only exchange is an all-gather of the G shard totals (each the
bit-exact pairwise sum of its shard, two_level.hpp:49-51); every rank then
derives the same per-shard sample counts from the seed with the
communication-free binomial descent (wrs_b200_shard_counts) and draws its own
count from its own table, writing global ids (local + shard base).  The
top-level table of the reference (an alias table over the group totals,
two_level.hpp:56-57) is built redundantly on every rank from the gathered
totals when per-sample routing is wanted (`top_table`).

The collective is torch.distributed's (NCCL on GPUs, gloo in the CPU tests);
this module only moves G doubles.
"""
from __future__ import annotations

from typing import Callable

import numpy as np

from . import wrs as _w


def shard_of(n: int, world: int, rank: int) -> tuple[int, int]:
    return _w.shard_range(n, world, rank)


def default_gather(local_total: float) -> np.ndarray:
    """All-gather one float64 per rank with torch.distributed."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size()
    backend = dist.get_backend()
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    mine = torch.tensor([local_total], dtype=torch.float64, device=dev)
    out = torch.empty(world, dtype=torch.float64, device=dev)
    dist.all_gather_into_tensor(out, mine)
    return out.cpu().numpy()


class ShardedSampler:
    """One rank's part of a sharded PSA sampler.

    weights: this rank's shard as a Weights handle (local ids 0..hi-lo).
    """

    def __init__(self, weights: "_w.Weights", n_total: int, rank: int, world: int,
                 gather: Callable[[float], np.ndarray] = default_gather):
        self.weights = weights
        self.n_total, self.rank, self.world = n_total, rank, world
        self.lo, self.hi = shard_of(n_total, world, rank)
        if weights.count() != self.hi - self.lo:
            raise ValueError(f"rank {rank}: shard has {weights.count()} items, expected "
                             f"{self.hi - self.lo}")
        self.sampler = _w.Sampler.build(weights, "psa", 1)
        self.totals = np.asarray(gather(weights.total()), dtype=np.float64)
        if self.totals.size != world:
            raise ValueError("gathered totals do not match the world size")

    def counts(self, seed: int, k: int) -> np.ndarray:
        """Draws per shard for (seed, k): identical on every rank."""
        return _w.shard_counts(self.totals, seed, k)

    def draw_device(self, seed: int, k: int, out, stream=None) -> int:
        """This rank's draws of a k-draw job into `out` (device tensor),
        global ids.  Returns how many were written."""
        mine = int(self.counts(seed, k)[self.rank])
        self.sampler.draw_shard_device(seed, self.rank, mine, self.lo, out, stream)
        return mine

    def top_table(self) -> "_w.Sampler":
        """The reference's top-level table (two_level.hpp:56-57): a PSA alias
        table over the gathered shard totals, built identically on every rank."""
        self._top_w = _w.Weights.from_array(self.totals)
        return _w.Sampler.build(self._top_w, "psa", 1)
