"""BASELINE configs[2] per GPU on one B200: n = 1e9 power-law (i+1)^-1 weights
(reference generator: host pow, Fisher-Yates deal on the device), sharded
contiguously over G GPUs; this process plays rank `--rank` of `--world`: it
builds the PSA table over its shard and draws its share of k = 1e10 (the
per-shard counts of the seed's binomial descent, identical on every rank --
wrs_b200_shard_counts over the shards' pairwise totals, which this script
computes for all shards from the one generated array instead of gathering
them).  Prints one JSON line: build and draw times of that rank (each alone, and a step of both).

    python scripts/config3_probe.py --world 1           # the whole job on one GPU
    python scripts/config3_probe.py --world 8 --rank 0  # one GPU's share at G = 8
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=float, default=1e9)
    ap.add_argument("--k", type=float, default=1e10)
    ap.add_argument("--world", type=int, default=1)
    ap.add_argument("--rank", type=int, default=0)
    ap.add_argument("--seed", type=int, default=42)
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    import numpy as np
    import torch

    import paper_1903_00227_b200 as wrs

    n, k = int(args.n), int(args.k)
    t0 = time.perf_counter()
    Wall = wrs.Weights.generate("powerlaw", 1.0, n, args.seed)
    gen_s = time.perf_counter() - t0
    lo, hi = wrs.shard_range(n, args.world, args.rank)
    if args.world > 1:
        vals = Wall.values()
        totals, Ws = [], None
        for g in range(args.world):  # each shard's pairwise total (two_level.hpp:49-51)
            a, b = wrs.shard_range(n, args.world, g)
            Wg = wrs.Weights.from_array(np.ascontiguousarray(vals[a:b]))
            totals.append(Wg.total())
            if g == args.rank:
                Ws = Wg
            else:
                Wg.free()
        Wall.free()
    else:
        Ws, totals = Wall, [Wall.total()]
    counts = wrs.shard_counts(np.asarray(totals, np.float64), args.seed, k)
    mine = int(counts[args.rank])
    S = wrs.Sampler.build(Ws, "psa", 1)
    out = torch.empty(mine, dtype=torch.int32, device="cuda")
    st = torch.cuda.current_stream()

    def timed(fn):
        best = None
        for _ in range(args.reps + 1):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record(st)
            fn()
            e1.record(st)
            torch.cuda.synchronize()
            t = e0.elapsed_time(e1)
            best = t if best is None else min(best, t)
        return best

    def draw():
        S.draw_shard_device(args.seed, args.rank, mine, lo, out, st)

    def step():  # rebuild + draw; the draw's table-independent scatter overlaps the rebuild
        S.rebuild_async(st)
        draw()

    best_b = timed(lambda: S.rebuild_async(st))
    best_d = timed(draw)
    best_s = timed(step)
    print(json.dumps({
        "workload": "BASELINE configs[2] shard: n=%d power-law s=1 (shuffled, seed %d), k=%d "
                    "split over %d shard(s); this is rank %d" % (n, args.seed, k, args.world, args.rank),
        "shard_items": hi - lo, "shard_draws": mine, "jobs": S.jobs,
        "step_ms": best_s, "step_g_items_plus_samples_per_s": (hi - lo + mine) / best_s / 1e6,
        "build_ms": best_b, "build_gitems_per_s": (hi - lo) / best_b / 1e6,
        "draw_ms": best_d, "draw_gsamples_per_s": mine / best_d / 1e6,
        "generate_s": gen_s, "checksum": int(out[-1].item()) if mine else None}))


if __name__ == "__main__":
    main()
