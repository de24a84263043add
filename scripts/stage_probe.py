"""Per-kernel build times (CUDA events inside the library; stages then run
one after another) and the whole build as the bench runs it (concurrent
stages allowed), for A/B builds:
    WRS_B200_LIB=... python scripts/stage_probe.py [n] [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1903_00227_b200 as wrs  # noqa: E402

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
st = torch.cuda.Stream()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
builds = []
for _ in range(reps + 1):
    torch.cuda.synchronize()
    a.record(st)
    S.rebuild_async(st)
    b.record(st)
    torch.cuda.synchronize()
    builds.append(a.elapsed_time(b))
S.check()
print(" ".join(f"{k}={v:.3f}" for k, v in zip(names, best)), f"sum={sum(best[:7]):.3f}",
      f"build={min(builds[1:]):.3f}")
