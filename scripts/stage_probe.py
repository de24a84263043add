"""Per-kernel build times (CUDA events inside the library) for A/B builds:
    WRS_B200_LIB=... python scripts/stage_probe.py [n] [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: F401  (CUDA context)

import paper_1903_00227_b200 as wrs

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 10**8
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
W = wrs.Weights.generate("uniform", 0.0, n, 42)
S = wrs.Sampler.build_psa(W, 0)
names = ["K1", "K2a", "K2b", "K2c", "K3", "K4a", "K4b"]
best = None
for _ in range(reps):
    wrs.set_timing(True)
    S.rebuild_async(None)
    torch.cuda.synchronize()
    t = S.stage_times()
    wrs.set_timing(False)
    best = t if best is None else [min(a, b) for a, b in zip(best, t)]
print(" ".join(f"{k}={v:.3f}" for k, v in zip(names, best)), f"sum={sum(best[:7]):.3f}")
