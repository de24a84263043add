"""GPU: the sharded (multi-GPU) path, with every shard built on the one GPU a
test box has.  Per-shard tables, shard totals, the top table over the totals,
per-shard draw counts and per-shard draws are each checked bit-for-bit against
the oracle / reference; the combined draws pass the reference's chi-square
policy against w_i / W."""
import numpy as np
import pytest

import oracle
import paper_1903_00227_b200 as wrs
from paper_1903_00227_b200.sharded import ShardedSampler
from tests.stats_util import chi_square

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("G", [2, 4, 8])
def test_sharded_build_and_draw(G):
    import torch
    P = oracle.port()
    n, k, seed = 1_000_003, 20_000_000, 77
    w = P.generate_powerlaw(n, 1.0, 42)
    shards = []
    for g in range(G):
        lo, hi = wrs.shard_range(n, G, g)
        shards.append((lo, hi, wrs.Weights.from_array(w[lo:hi])))
    totals = np.array([s[2].total() for s in shards])
    for g, (lo, hi, _) in enumerate(shards):
        assert totals[g] == P.pairwise_sum(w[lo:hi])  # two_level.hpp:49-51
    R = oracle.ref()
    if R is not None:
        assert totals.tobytes() == R.two_level_group_totals(w, G).tobytes()

    samplers = [ShardedSampler(W, n, g, G, gather=lambda _t: totals)
                for g, (_, _, W) in enumerate(shards)]
    counts = samplers[0].counts(seed, k)
    assert int(counts.sum()) == k
    for s in samplers[1:]:
        assert np.array_equal(s.counts(seed, k), counts)

    # top table over the shard totals (two_level.hpp:56-57)
    top = samplers[0].top_table()
    ob, own = P.psa_build(totals, wrs.default_jobs(G))
    assert top.buckets().tobytes() == ob.tobytes() and top.bucket_mean == own

    hist = torch.zeros(n, dtype=torch.int64, device="cuda")
    for g, s in enumerate(samplers):
        out = torch.empty(int(counts[g]), dtype=torch.int32, device="cuda")
        assert s.draw_device(seed, k, out) == counts[g]
        torch.cuda.synchronize()
        tb = s.sampler.buckets()
        ref = P.sample_many(tb, s.sampler.bucket_mean, wrs.shard_seed(seed, g), int(counts[g]), 1)
        got = out.cpu().numpy().view(np.uint32)
        bad = np.nonzero(got - np.uint32(s.lo) != ref)[0]
        assert bad.size == 0, (g, bad.size, bad[:8], got[bad[:4]], ref[bad[:4]], s.lo)
        hist += torch.bincount(out.long(), minlength=n)
    stat, crit, df, ok = chi_square(hist.cpu().numpy(), w / w.sum())
    assert ok, (stat, crit, df)
