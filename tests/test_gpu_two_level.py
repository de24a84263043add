"""GPU parity of the routed two-level draws:
wrs_b200_two_level_draw_device reproduces TwoLevelTable::sample_many
(two_level.hpp:66-81) bit for bit when fed the same group tables -- pinned to
the reference-generated fixture (tests/golden/two_level.npz) and to the
oracle port on larger cases -- and the sharded path routes queries to shard
tables opened from CUDA IPC handles.
"""
import os

import numpy as np
import pytest

import oracle
import paper_1903_00227_b200 as wrs

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def P():
    return oracle.port()


def upload(b):
    import torch
    return torch.from_numpy(b.view(np.uint8).copy()).cuda()


def routed(tabs, means, bases, top, tm, seed, k, W, q0, q1):
    import torch
    dt = [upload(t) for t in tabs]
    dtop = upload(top)
    out = torch.empty(max(q1 - q0, 1), dtype=torch.int32, device="cuda")
    wrs.wrs.two_level_draw_device(dt, [t.size for t in tabs], means, bases, dtop, tm, seed, q0,
                                  q1, k, W, out)
    torch.cuda.synchronize()
    return out[:q1 - q0].cpu().numpy().view(np.uint32)


def test_two_level_golden(P):
    t = np.load(os.path.join(GOLD, "two_level.npz"))
    w = P.generate_powerlaw(3001, 1.0, 5)
    for G in (4, 7):
        tabs, means, bases, top, tm = P.two_level_build(w, G)
        for W in (1, 3):
            got = routed(tabs, means, bases, top, tm, 7, 5001, W, 0, 5001)
            assert np.array_equal(got, t[f"G{G}/draws_s7_k5001_W{W}"]), (G, W)


def test_two_level_random_vs_oracle(P):
    rng = np.random.default_rng(8)
    for n, G, k, W in ((1, 1, 1000, 1), (10, 3, 10_000, 2), (100_003, 8, 2_000_003, 5),
                       (1_000_000, 64, 3_000_000, 1), (50_000, 256, 500_000, 7)):
        w = rng.random(n) + 1e-3 if n > 1 else np.array([1.0])
        tabs, means, bases, top, tm = P.two_level_build(w, G)
        for q0, q1 in ((0, k), (k // 3, k // 3 + 12345)):
            q1 = min(q1, k)
            ref = P.two_level_sample_range(tabs, means, bases, top, tm, 42, k, W, q0, q1)
            assert np.array_equal(routed(tabs, means, bases, top, tm, 42, k, W, q0, q1), ref), \
                (n, G, k, W, q0)


def _ipc_rank(rank, world, port, n_total, k, seed, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1903_00227_b200.sharded import ShardedSampler
        torch.cuda.set_device(0)
        lo, hi = wrs.shard_range(n_total, world, rank)
        W = wrs.Weights.generate_range("uniform", 0.0, n_total, lo, hi, seed)
        sh = ShardedSampler(W, n_total, rank, world)
        sh.open_peers()
        out = torch.empty(k, dtype=torch.int32, device="cuda")
        q0, q1 = sh.routed_draw_device(seed, k, out)
        torch.cuda.synchronize()
        dist.barrier()  # peers' tables stay alive until every rank has drawn
        q.put((rank, q0, q1, out[:q1 - q0].cpu().numpy().view(np.uint32).copy(),
               sh.sampler.buckets(), sh.sampler.bucket_mean,
               sh._top.buckets(), sh._top.bucket_mean))
        sh.close_peers()
        dist.barrier()
    finally:
        dist.destroy_process_group()


def test_sharded_routed_draws_through_ipc(P):
    """Two processes on this GPU, each owning a shard table; every query is
    routed by the top table and read from whichever process's table it picks
    (opened through CUDA IPC).  Checked against the oracle fed the same
    tables.  (The processes never wait on each other's kernels.)"""
    import socket

    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    n_total, k, seed, world = 300_007, 400_001, 19, 2
    procs = [ctx.Process(target=_ipc_rank, args=(r, world, port, n_total, k, seed, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in range(world)], key=lambda x: x[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    tabs = [r[4] for r in res]
    means = np.array([r[5] for r in res])
    bases = np.array([wrs.shard_range(n_total, world, r)[0] for r in range(world)], np.uint64)
    top, tm = res[0][6], res[0][7]
    assert res[1][6].tobytes() == top.tobytes()  # the top table is identical on every rank
    for rank, q0, q1, got, *_ in res:
        ref = P.two_level_sample_range(tabs, means, bases, top, tm, seed, k, world, q0, q1)
        assert np.array_equal(got, ref), rank
