"""CPU, world_size 2 over gloo: the multi-GPU host logic of the sharded path.

Each rank takes its contiguous shard (two_level.hpp:33-41), computes the
shard's pairwise total with the oracle (the device computes the same value,
bit-exact, in K0), all-gathers the totals with torch.distributed (gloo here,
NCCL on the box) and derives the per-shard draw counts.  Every rank must
agree on every count, the counts must sum to k, and they must equal a host
replay of the descent with the reference's own binomial_split.
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, k, seed, out_dir):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    import paper_1903_00227_b200 as wrs
    from paper_1903_00227_b200.sharded import default_gather, shard_of
    P = oracle.port()
    w = P.generate_uniform(n, 42)  # every rank can regenerate the global vector
    lo, hi = shard_of(n, world, rank)
    local_total = P.pairwise_sum(w[lo:hi])
    totals = default_gather(local_total)
    counts = wrs.shard_counts(totals, seed, k)
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), totals=totals, counts=counts,
             lo=lo, hi=hi)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_sharded_counts_agree_across_ranks(tmp_path, world):
    n, k, seed = 100_003, 10**9 + 7, 2024
    port = _free_port()
    mp.spawn(_worker, args=(world, port, n, k, seed, str(tmp_path)), nprocs=world, join=True)
    res = [np.load(tmp_path / f"rank{r}.npz") for r in range(world)]
    for r in range(1, world):
        assert np.array_equal(res[r]["totals"], res[0]["totals"])
        assert np.array_equal(res[r]["counts"], res[0]["counts"])
    assert int(res[0]["counts"].sum()) == k
    # shards tile [0, n)
    bounds = sorted((int(x["lo"]), int(x["hi"])) for x in res)
    assert bounds[0][0] == 0 and bounds[-1][1] == n
    assert all(bounds[i][1] == bounds[i + 1][0] for i in range(world - 1))
    # totals are the reference TwoLevelTable group totals (two_level.hpp:49-51)
    import oracle
    R = oracle.ref()
    if R is not None:
        w = oracle.port().generate_uniform(n, 42)
        assert res[0]["totals"].tobytes() == R.two_level_group_totals(w, world).tobytes()
        from tests.test_capi_host import _replay_counts
        assert list(res[0]["counts"]) == _replay_counts(R, oracle.port(), list(res[0]["totals"]),
                                                        seed, k)


def _id_worker(rank, world, port, out_dir):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1903_00227_b200.sharded import job_nccl_id
    nid = job_nccl_id(rank, world)
    with open(os.path.join(out_dir, f"id{rank}.bin"), "wb") as f:
        f.write(nid)
    dist.barrier()
    dist.destroy_process_group()


def test_multi_gpu_job_shares_one_nccl_id(tmp_path):
    """bench.py's N > 1 path (sharded.multi_create): rank 0 makes the job's
    NCCL unique id through the library, the process group broadcasts it, and
    every rank hands the same 128 bytes to wrs_b200_multi_create."""
    import paper_1903_00227_b200 as wrs
    if not wrs.nccl_available()[0]:
        pytest.skip("libnccl.so.2 not loadable")
    world = 2
    mp.spawn(_id_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    ids = [(tmp_path / f"id{r}.bin").read_bytes() for r in range(world)]
    assert len(ids[0]) == 128 and all(x == ids[0] for x in ids)

