"""GPU: the C++-owned multi-GPU sampler (wrs_b200_multi_*).

* one rank with a real NCCL communicator (ncclCommInitRank over one rank, the
  shard total all-gathered device to device): totals, counts, top table and
  draws agree with the plain sampler of the whole vector;
* G = 2, 4, 8 ranks on the one GPU a test box has, the totals exchanged by
  the caller (wrs_b200_multi_set_totals): per-rank counts equal the
  reference's binomial descent, per-rank draws equal the oracle's
  AliasTable(shard).sample_many(shard seed) plus the shard base, the top
  table equals the oracle's table over the totals, and the union of the
  ranks' draws passes the chi-square policy against w_i / W.
"""
import numpy as np
import pytest

import oracle
import paper_1903_00227_b200 as wrs
from paper_1903_00227_b200.sharded import multi_create
from tests.stats_util import chi_square

pytestmark = pytest.mark.gpu


def test_multi_single_rank_with_nccl():
    import torch
    if not wrs.nccl_available()[0]:
        pytest.skip("libnccl.so.2 not loadable")
    P = oracle.port()
    n, k, seed = 300_007, 2_000_003, 5
    w = P.generate_uniform(n, 9)
    W = wrs.Weights.from_array(w)
    M = wrs.MultiSampler.create(W, n, 0, 1, wrs.nccl_unique_id())
    assert M.totals(1).tolist() == [W.total()]
    assert M.counts(seed, k, 1).tolist() == [k]
    out = torch.empty(k, dtype=torch.int32, device="cuda")
    assert M.draw_device(seed, k, out) == k
    M.exchange()  # a second all-gather over the live communicator
    M.rebuild_async()
    M.sampler.check()
    torch.cuda.synchronize()
    b = M.sampler.buckets()
    ref = P.sample_many(b, M.sampler.bucket_mean, wrs.shard_seed(seed, 0), k, 1)
    assert np.array_equal(out.cpu().numpy().view(np.uint32), ref)
    top, tm = M.top_buckets(1)
    assert top["alias"][0] == 0 and top["item"][0] == 0
    M.free()


@pytest.mark.parametrize("G", [2, 4, 8])
def test_multi_ranks_on_one_gpu(G):
    import torch
    P = oracle.port()
    n, k, seed = 1_000_003, 20_000_000, 11
    w = P.generate_powerlaw(n, 1.0, 42)
    shards, Ms = [], []
    for g in range(G):
        lo, hi = wrs.shard_range(n, G, g)
        shards.append(wrs.Weights.from_array(w[lo:hi]))
    totals = np.array([s.total() for s in shards])
    for g in range(G):
        M = wrs.MultiSampler.create(shards[g], n, g, G, None)
        M.set_totals(totals)
        Ms.append(M)
    counts = Ms[0].counts(seed, k, G)
    assert int(counts.sum()) == k
    for M in Ms[1:]:
        assert np.array_equal(M.counts(seed, k, G), counts)
    R = oracle.ref()
    if R is not None:
        from tests.test_capi_host import _replay_counts
        assert list(counts) == _replay_counts(R, P, list(totals), seed, k)
    ob, own = P.psa_build(totals, wrs.default_jobs(G))
    top, tm = Ms[0].top_buckets(G)
    assert top.tobytes() == ob.tobytes() and tm == own
    hist = torch.zeros(n, dtype=torch.int64, device="cuda")
    for g, M in enumerate(Ms):
        lo, hi = wrs.shard_range(n, G, g)
        out = torch.empty(max(int(counts[g]), 1), dtype=torch.int32, device="cuda")
        assert M.draw_device(seed, k, out) == counts[g]
        torch.cuda.synchronize()
        got = out[:int(counts[g])].cpu().numpy().view(np.uint32)
        tb = M.sampler.buckets()
        ref = P.sample_many(tb, M.sampler.bucket_mean, wrs.shard_seed(seed, g), int(counts[g]), 1)
        assert np.array_equal(got - np.uint32(lo), ref), g
        hist += torch.bincount(out[:int(counts[g])].long(), minlength=n)
    stat, crit, df, ok = chi_square(hist.cpu().numpy(), w / w.sum())
    assert ok, (stat, crit, df)
    for M in Ms:
        M.free()


def test_multi_create_helper_single_process():
    """sharded.multi_create as bench.py uses it, world = 1 (NCCL when loadable)."""
    import torch
    import torch.distributed as dist
    if not dist.is_initialized():
        import os
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29533")
        dist.init_process_group("gloo", rank=0, world_size=1)
    W = wrs.Weights.generate("uniform", 0.0, 100_000, 3)
    M = multi_create(W, 100_000, 0, 1)
    out = torch.empty(1000, dtype=torch.int32, device="cuda")
    assert M.draw_device(1, 1000, out) == 1000
    M.free()
