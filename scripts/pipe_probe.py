"""Draw-stage chunk pipeline sweep: 1e9 draws from an n-item table with
WRS_B200_DRAW_PIPE set to each configuration on the command line, timed with
CUDA events (median of 5) and checked byte-equal to the unpipelined draw.
    python scripts/pipe_probe.py 1e8 1e9 1 2,2,3,2 4,2,3,2 ...
The pipeline was measured slower and reverted (profiles/r02_draw_pipeline_
experiment.md); the library now ignores WRS_B200_DRAW_PIPE, so this times the
shipped serial plan unless run against that experiment's build."""
import hashlib
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

import paper_1903_00227_b200 as wrs

n = int(float(sys.argv[1]))
k = int(float(sys.argv[2]))
cfgs = sys.argv[3:] or ["1"]
W = wrs.Weights.generate("uniform", 0.0, n, 42)
S = wrs.Sampler.build_psa(W, 0)
out = torch.empty(k, dtype=torch.int32, device="cuda")
ref = None
for cfg in cfgs:
    os.environ["WRS_B200_DRAW_PIPE"] = cfg
    for _ in range(2):
        S.draw_device(7, k, 1, out)
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        S.draw_device(7, k, 1, out)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    h = hashlib.sha256(out.cpu().numpy().tobytes()).hexdigest()[:16]
    if ref is None:
        ref = h
    ms = statistics.median(ts)
    print(f"n={n:.3g} k={k:.3g} pipe={cfg:>10} draw {ms:7.3f} ms  frac {36 * k / ms / 1e6 / 6443.2:.3f}"
          f"  sha {h} {'same' if h == ref else 'DIFF'}", flush=True)
S.check()
