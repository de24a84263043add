"""One build + one device draw of k samples at table size n, for launch-list
profiling of the draw kernels at sizes other than the bench's:
    ncu --metrics gpu__time_duration.sum python scripts/draw_probe.py n k"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

import paper_1903_00227_b200 as wrs

n = int(float(sys.argv[1]))
k = int(float(sys.argv[2]))
W = wrs.Weights.generate("uniform", 0.0, n, 42)
S = wrs.Sampler.build_psa(W, 0)
out = torch.empty(k, dtype=torch.int32, device="cuda")
for _ in range(2):
    S.draw_device(7, k, 1, out)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
S.draw_device(7, k, 1, out)
b.record()
torch.cuda.synchronize()
print(f"n={n} k={k} draw {a.elapsed_time(b):.3f} ms")
