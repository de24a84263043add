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


def default_gather_obj(obj) -> list:
    """All-gather one picklable object per rank with torch.distributed."""
    import torch.distributed as dist
    out = [None] * dist.get_world_size()
    dist.all_gather_object(out, obj)
    return out


def worker_slice(k: int, workers: int, w: int) -> tuple[int, int]:
    """parallel.hpp:37-43."""
    per, rem = divmod(k, workers)
    lo = per * w + min(w, rem)
    return lo, lo + per + (1 if w < rem else 0)


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

    # ---- routed two-level draws ---------------------------
    def open_peers(self, gather_obj: Callable[[object], list] = default_gather_obj) -> None:
        """Exchange every shard table's CUDA IPC handle, size and bucket mean
        and open the peers' tables in this process (their buckets are then
        read over NVLink by the routed draw)."""
        meta = (_w.ipc_handle(self.sampler), self.sampler.size, self.sampler.bucket_mean)
        metas = gather_obj(meta)
        self._peer_ptrs = []
        self._opened = []
        for r, (h, _, _) in enumerate(metas):
            if r == self.rank:
                self._peer_ptrs.append(self.sampler.device_buckets())
            else:
                p = _w.ipc_open(h)
                self._opened.append(p)
                self._peer_ptrs.append(p)
        self._sizes = np.array([m[1] for m in metas], np.uint64)
        self._means = np.array([m[2] for m in metas], np.float64)
        self._bases = np.array([shard_of(self.n_total, self.world, r)[0]
                                for r in range(self.world)], np.uint64)
        self._top = self.top_table()

    def routed_draw_device(self, seed: int, k: int, out, stream=None) -> tuple[int, int]:
        """Worker `rank` of `world` of TwoLevelTable::sample_many(seed, k, world)
        (two_level.hpp:71-81) over the shard tables: rows [q0, q1) of the global
        output into out[0 .. q1 - q0).  Every query picks its shard with the top
        table and gathers from that shard's table, wherever it lives."""
        if not hasattr(self, "_peer_ptrs"):
            raise RuntimeError("open_peers() first")
        q0, q1 = worker_slice(k, self.world, self.rank)
        _w.two_level_draw_device(self._peer_ptrs, self._sizes, self._means, self._bases,
                                 self._top.device_buckets(), self._top.bucket_mean, seed, q0, q1,
                                 k, self.world, out, stream)
        return q0, q1

    def close_peers(self) -> None:
        for p in getattr(self, "_opened", []):
            _w.ipc_close(p)
        self._opened = []


# ---- the C++-owned multi-GPU sampler (wrs_b200_multi_*) ---------------------------
def job_nccl_id(rank: int, world: int) -> bytes:
    """The job's NCCL unique id: made by rank 0 (wrs_b200_nccl_unique_id),
    broadcast to every rank over torch.distributed."""
    import torch.distributed as dist
    nid = [_w.nccl_unique_id() if rank == 0 else None]
    if world > 1:
        dist.broadcast_object_list(nid, src=0)
    return nid[0]


def multi_create(weights: "_w.Weights", n_total: int, rank: int, world: int,
                 use_nccl: bool | None = None) -> "_w.MultiSampler":
    """This rank's wrs_b200_multi handle.  With NCCL (the default when
    libnccl.so.2 loads and torch.distributed runs the nccl backend) rank 0
    makes the job's NCCL unique id, torch.distributed broadcasts those 128
    bytes, and the library creates its own communicator and all-gathers the
    shard totals device to device.  Otherwise (gloo, CPU tests) the totals
    are gathered with torch.distributed and handed to the library."""
    import torch.distributed as dist
    if use_nccl is None:
        use_nccl = _w.nccl_available()[0] and (world == 1 or dist.get_backend() == "nccl")
    if use_nccl:
        m = _w.MultiSampler.create(weights, n_total, rank, world, job_nccl_id(rank, world))
        m.has_comm = True
        return m
    m = _w.MultiSampler.create(weights, n_total, rank, world, None)
    m.has_comm = False
    m.set_totals(default_gather(weights.total()) if world > 1 else [weights.total()])
    return m

