"""Philox draw mode vs the reference-stream draws: 1e9 draws at table size n
(CUDA events, best of 3).
    python scripts/philox_probe.py [n]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1903_00227_b200 as wrs  # noqa: E402

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 10**8
k = 10**9
W = wrs.Weights.generate("uniform", 0.0, n, 42)
S = wrs.Sampler.build_psa(W, 0)
out = torch.empty(k, dtype=torch.int32, device="cuda")


def best(fn):
    fn()
    t = []
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        t.append(a.elapsed_time(b))
    return min(t)


rs = best(lambda: S.draw_device(7, k, 1, out))
ph = best(lambda: S.draw_philox_device(7, k, out))
print(f"n={n} k={k}: RngStream draws {rs:.3f} ms, Philox draws {ph:.3f} ms "
      f"({36 * k / ph / 1e6:.0f} GB/s at 36 B/sample)")
