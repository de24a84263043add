"""BASELINE configs[4] on one B200: size sweep n = 2^10 .. 2^30 (powers of 4)
for Uniform(0,1] (generate_uniform, on the device) and power-law s=0.5
(generate_powerlaw: host pow, Fisher-Yates deal on the device), build time (rebuild alone, median of
reps) and 1e9-draw query throughput per size, each with its HBM roofline
fraction (72 B/item build, 36 B/sample draws) and whether the 16n-B table is
L2-resident.

    python scripts/size_sweep.py [--draws 1000000000] [--max-log2 30] [--out profiles/r01_size_sweep]
"""
import argparse
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))

BUILD_B, DRAW_B = 72, 36


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--draws", type=int, default=10**9)
    ap.add_argument("--max-log2", type=int, default=30)
    ap.add_argument("--powerlaw-max-log2", type=int, default=30,
                    help="cap the power-law sizes (its (i+1)^-s values are computed on the host)")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--out", default="profiles/r01_size_sweep")
    args = ap.parse_args()

    import torch

    import paper_1903_00227_b200 as wrs
    peaks = json.load(open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")))
    hbm = None
    for key in ("hbm_gbs",):
        if key in peaks:
            hbm = float(peaks[key])
    if hbm is None:
        hbm = 6550.4
    l2 = torch.cuda.get_device_properties(0).L2_cache_size
    stream = torch.cuda.Stream()
    rows = []

    def timed(fn, reps):
        ts = []
        for _ in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(stream):
                a.record(stream)
                fn()
                b.record(stream)
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        return statistics.median(ts)

    out = torch.empty(args.draws, dtype=torch.int32, device="cuda")
    for log2 in range(10, args.max_log2 + 1, 2):
        n = 1 << log2
        for dist in ("uniform", "powerlaw"):
            if dist == "powerlaw" and log2 > args.powerlaw_max_log2:
                continue
            t0 = time.time()
            if dist == "uniform":
                W = wrs.Weights.generate_range("uniform", 0.0, n, 0, n, 42)
            else:
                W = wrs.Weights.generate("powerlaw", 0.5, n, 42)
            gen_s = time.time() - t0
            S = wrs.Sampler.build(W, "psa", 1)
            S.rebuild_async(stream)
            build_ms = timed(lambda: S.rebuild_async(stream), args.reps)
            S.draw_device(7, args.draws, 1, out, stream)
            draw_ms = timed(lambda: S.draw_device(7, args.draws, 1, out, stream), args.reps)
            S.check()
            row = {
                "log2_n": log2, "n": n, "dist": dist, "jobs": S.jobs,
                "table_bytes": 16 * n, "l2_resident": 16 * n <= l2,
                "build_ms": build_ms, "build_gitems_per_s": n / build_ms / 1e6,
                "build_hbm_frac": BUILD_B * n / (build_ms * 1e-3) / 1e9 / hbm,
                "draw_ms": draw_ms, "draw_gsamples_per_s": args.draws / draw_ms / 1e6,
                # an L2-resident table's gathers never reach HBM;
                # its HBM bytes are the 4-B index stores
                "draw_bytes_per_sample": 4 if 16 * n <= l2 else DRAW_B,
                "draw_hbm_frac": (4 if 16 * n <= l2 else DRAW_B) * args.draws /
                                 (draw_ms * 1e-3) / 1e9 / hbm,
                "generate_s": gen_s,
            }
            rows.append(row)
            print(json.dumps(row), flush=True)
            del S, W
            torch.cuda.empty_cache()
    res = {"config": "BASELINE configs[4] on 1 B200 (sizes 2^10..2^%d, k=%d draws per size)"
                     % (args.max_log2, args.draws),
           "peak_hbm_GBps": hbm, "l2_bytes": l2, "rows": rows}
    os.makedirs(os.path.dirname(args.out) or ".", exist_ok=True)
    with open(args.out + ".json", "w") as f:
        json.dump(res, f, indent=1)
    with open(args.out + ".md", "w") as f:
        f.write("| n | dist | table | L2-resident | build ms | G items/s | build frac (72 B/item) | "
                "draw ms (1e9) | G samples/s | draw frac (B/sample) |\n"
                "|---|---|---|---|---|---|---|---|---|---|\n")
        for r in rows:
            f.write("| 2^%d | %s | %.1f MB | %s | %.3f | %.2f | %.2f | %.2f | %.1f | %.2f (%d) |\n" % (
                r["log2_n"], r["dist"], r["table_bytes"] / 2**20, "yes" if r["l2_resident"] else "no",
                r["build_ms"], r["build_gitems_per_s"], r["build_hbm_frac"], r["draw_ms"],
                r["draw_gsamples_per_s"], r["draw_hbm_frac"], r["draw_bytes_per_sample"]))


if __name__ == "__main__":
    main()
