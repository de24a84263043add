"""Direct vs region draw plan around the L2 size: 1e9 draws per table size
(WRS_B200_PLAN forces the plan).  Run on the GPU box with PYTHONPATH=."""
import os
import subprocess
import sys

code = r'''
import sys, torch, paper_1903_00227_b200 as wrs
n = int(sys.argv[1]); k = 10**9
W = wrs.Weights.generate_range("uniform", 0.0, n, 0, n, 42)
S = wrs.Sampler.build(W, "psa", 1)
out = torch.empty(k, dtype=torch.int32, device="cuda")
S.draw_device(7, k, 1, out); torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(); S.draw_device(7, k, 1, out); b.record(); torch.cuda.synchronize()
print(a.elapsed_time(b))
'''
for mb in (64, 96, 128, 160, 192, 256):
    n = mb * 2**20 // 16
    row = [f"{mb} MB"]
    for plan in ("direct", "region"):
        env = dict(os.environ, WRS_B200_PLAN=plan)
        r = subprocess.run([sys.executable, "-c", code, str(n)], env=env, capture_output=True, text=True)
        row.append(f"{plan} {float(r.stdout.strip().splitlines()[-1]):.2f} ms" if r.returncode == 0 else f"{plan} err")
    print(" | ".join(row), flush=True)
