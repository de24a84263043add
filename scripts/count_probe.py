"""Aggregated draws (configs[3] shape): n lognormal(0, 2) weights, 1e9 draws
-> (item, count) pairs, for launch-list profiling of the counting kernels.
    python scripts/count_probe.py [n] [k]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1903_00227_b200 as wrs  # noqa: E402

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 10**8
k = int(float(sys.argv[2])) if len(sys.argv) > 2 else 10**9
W = wrs.Weights.generate("lognormal", 2.0, n, 42)
S = wrs.Sampler.build(W, "psa", 1)
cap = min(n, k)
items = torch.empty(cap, dtype=torch.int32, device="cuda")
counts = torch.empty(cap, dtype=torch.int64, device="cuda")
m = torch.zeros(1, dtype=torch.int64, device="cuda")
for _ in range(2):
    S.draw_counts_device(42, k, 1, items, counts, m, None)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
S.draw_counts_device(42, k, 1, items, counts, m, None)
b.record()
torch.cuda.synchronize()
print(f"n={n} k={k} counts {a.elapsed_time(b):.3f} ms, {int(m.item())} distinct")
