"""BASELINE configs[0] (the reference's CPU-runnable case) on one B200 beside
the reference itself on the host: n = 1e6 Uniform(0,1] weights (reference
generator, seed 42), PSA build, 1e7 with-replacement draws -- with the
reference's SplitMix64 stream (bit-exact with sample_many) and with the Philox
mode the config names.  The host side is the unmodified reference
(oracle/_ref: AliasTable(wt, psa, T) + sample_many with T = all host threads),
timed as bench.py's CPU arm times it.  Prints one JSON line.

    python scripts/config0_probe.py
"""
import json
import os
import sys

sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))


def main():
    import torch

    import bench
    import paper_1903_00227_b200 as wrs

    n, k, seed = 10**6, 10**7, 42
    W = wrs.Weights.generate("uniform", 0.0, n, seed)
    S = wrs.Sampler.build(W, "psa", 1)
    st = torch.cuda.current_stream()
    out = torch.empty(k, dtype=torch.int32, device="cuda")

    def timed(fn, reps=20):
        best = None
        for _ in range(reps + 2):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record(st)
            fn()
            e1.record(st)
            torch.cuda.synchronize()
            t = e0.elapsed_time(e1)
            best = t if best is None else min(best, t)
        return best

    build = timed(lambda: S.rebuild_async(st))
    draw = timed(lambda: S.draw_device(seed, k, 1, out, st))
    philox = timed(lambda: S.draw_philox_device(seed, k, out, st))
    step = timed(lambda: (S.rebuild_async(st), S.draw_device(seed, k, 1, out, st)))
    threads = os.cpu_count() or 1
    cpu_s, d = bench.cpu_reference_step(n, k, k, threads)
    print(json.dumps({
        "workload": "BASELINE configs[0]: n=1e6 uniform (reference generator, seed 42), "
                    "psa build + 1e7 draws",
        "gpu_build_ms": build, "gpu_draw_ms": draw, "gpu_draw_philox_ms": philox,
        "gpu_step_ms": step, "gpu_step_g_per_s": (n + k) / step / 1e6,
        "cpu_reference": {"kind": d["kind"], "threads": d["cores"], "build_ms": d["build_s"] * 1e3,
                          "draw_ms": d["draw_s_per_1e9"] * k / 1e9 * 1e3,
                          "step_ms": cpu_s * 1e3, "g_per_s": (n + k) / cpu_s / 1e9},
        "speedup_step": cpu_s * 1e3 / step}))


if __name__ == "__main__":
    main()
