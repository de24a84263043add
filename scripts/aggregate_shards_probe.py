"""BASELINE configs[3] per GPU on one B200: n = 1e8 lognormal(0, 2) weights
sharded contiguously over G GPUs, k = 1e9 with-replacement draws aggregated to
(item, count) pairs.  This process plays rank `--rank` of `--world`: it builds
the PSA table over its shard, derives its draw count from the shard totals with
the seed's binomial descent (wrs_b200_shard_counts; the totals of all shards
are computed here from the one generated array instead of being gathered), and
aggregates its draws (wrs_b200_sampler_draw_counts_device).  The pairs stay
sharded: shard g's items are [lo_g, hi_g) of the global ids.  Prints one JSON
line per G.

    python scripts/aggregate_shards_probe.py [--worlds 1,2,4,8]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=float, default=1e8)
    ap.add_argument("--k", type=float, default=1e9)
    ap.add_argument("--worlds", default="1,2,4,8")
    ap.add_argument("--seed", type=int, default=42)
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    import numpy as np
    import torch

    import paper_1903_00227_b200 as wrs

    n, k = int(args.n), int(args.k)
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(args.seed)
    wt = torch.exp(2.0 * torch.randn(n, dtype=torch.float64, device=dev, generator=g))
    st = torch.cuda.current_stream()
    for world in (int(x) for x in args.worlds.split(",")):
        totals = []
        for r in range(world):
            a, b = wrs.shard_range(n, world, r)
            Wr = wrs.Weights.from_device(wt[a:b].contiguous())
            totals.append(Wr.total())
            if r:
                Wr.free()
            else:
                W0 = Wr
        mine = int(wrs.shard_counts(np.asarray(totals, np.float64), args.seed, k)[0])
        S = wrs.Sampler.build(W0, "psa", 1)
        m_items = W0.count()
        cap = min(m_items, mine)
        items = torch.empty(cap, dtype=torch.int32, device=dev)
        counts = torch.empty(cap, dtype=torch.int64, device=dev)
        m = torch.zeros(1, dtype=torch.int64, device=dev)
        best = None
        for _ in range(args.reps + 1):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record(st)
            S.draw_counts_device(args.seed, mine, 1, items, counts, m, st)
            e1.record(st)
            torch.cuda.synchronize()
            t = e0.elapsed_time(e1)
            best = t if best is None else min(best, t)
        nu = int(m.item())
        assert int(counts[:nu].sum()) == mine
        print(json.dumps({
            "workload": "BASELINE configs[3] shard: n=%d lognormal(0,2) (torch cuda generator, "
                        "seed %d), k=%d aggregated to (item, count), %d shard(s); rank 0"
                        % (n, args.seed, k, world),
            "world": world, "shard_items": m_items, "shard_draws": mine, "ms": best,
            "gsamples_per_s": mine / best / 1e6, "n_unique": nu}), flush=True)
        S.free()
        W0.free()


if __name__ == "__main__":
    main()
