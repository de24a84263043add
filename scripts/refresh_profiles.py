"""Regenerate profiles/ from a TAG run of scripts/gpu_round1_profile.sh
(gpurun_out/bench_<tag>.log, launches_<tag>.csv, prof_<tag>.ncu-rep):
r<tag>_launch_list.txt, r<tag>_ncu_kernels.txt, traffic.json, r<tag>_summary.md.

    python scripts/refresh_profiles.py [tag]
"""
import json
import os
import re
import subprocess
import sys

HERE = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
G = os.path.join(HERE, "gpurun_out")
P = os.path.join(HERE, "profiles")


def run(*a):
    return subprocess.run([sys.executable, *a], capture_output=True, text=True, check=True).stdout


launch = run(os.path.join(HERE, "scripts", "launch_table.py"), os.path.join(G, f"launches_{tag}.csv"))
open(os.path.join(P, f"{tag}_launch_list.txt"), "w").write(launch)
raw = subprocess.run(["ncu", "-i", os.path.join(G, f"prof_{tag}.ncu-rep"), "--page", "raw", "--csv"],
                     capture_output=True, text=True).stdout
open("/tmp/raw_prof.csv", "w").write(raw)
summ = run(os.path.join(HERE, "scripts", "ncu_summary.py"), "/tmp/raw_prof.csv").splitlines()
out, seen, i = [f"# ncu --set full --clock-control none, one launch of each kernel of a bench step "
                f"(n=1e8, k=1e9), 1x B200",
                f"# command: TAG={tag} bash scripts/gpu_round1_profile.sh (report "
                f"gpurun_out/prof_{tag}.ncu-rep)"], set(), 0
while i < len(summ):
    blk = [summ[i]]
    if i + 1 < len(summ) and summ[i + 1].startswith("    "):
        blk.append(summ[i + 1])
        i += 1
    i += 1
    name = blk[0].split(":")[0]
    if name not in seen:
        seen.add(name)
        out += blk
open(os.path.join(P, f"{tag}_ncu_kernels.txt"), "w").write("\n".join(out) + "\n")

b = json.loads(open(os.path.join(G, f"bench_{tag}.log")).read().strip().splitlines()[-1])
rows = []
for line in launch.splitlines():
    m = re.match(r"\s*(\d+) (.{40}) +([\d.]+) us  read +([\d.]+) GB  write +([\d.]+) GB", line)
    if m and 20 <= int(m.group(1)) <= 30:
        rows.append((m.group(2).strip(), float(m.group(3)), float(m.group(4)), float(m.group(5))))
assert len(rows) == 11, rows
names = ["K1", "K2a", "K2b", "K2c", "K3", "K4a", "K4b"]
bt = sum(r + w for _, _, r, w in rows[:7])
dt = sum(r + w for _, _, r, w in rows[7:])
json.dump({"draw_bytes_per_sample": round(dt, 2), "build_bytes_per_item": round(bt * 10, 1),
           "source": f"profiles/{tag}_launch_list.txt (launches 20-30, one bench step): ncu "
                     "dram__bytes_read.sum + dram__bytes_write.sum per launch, n=1e8 uniform, k=1e9 "
                     "draws (region plan: scatter %.2f GB + gather %.2f GB + unpermute %.2f GB; "
                     "build: %s GB)" % (rows[7][2] + rows[7][3], rows[9][2] + rows[9][3],
                                        rows[10][2] + rows[10][3],
                                        " + ".join("%s %.2f" % (n, r + w) for n, (_, _, r, w)
                                                   in zip(names, rows[:7])))},
          open(os.path.join(P, "traffic.json"), "w"), indent=2)
c = b["cpu_baseline"]
s = [f"# Round 1 evidence summary (1x B200, n = 1e8 uniform, k = 1e9 draws)\n",
     f"Bench line: `gpurun_out/bench_{tag}.log` (command `python bench.py`, driver defaults):\n",
     f"- step (rebuild + 1e9 draws): **{b['ms_per_step']:.2f} ms -> {b['value']:.1f} "
     f"G(items+samples)/s**; clocks {b['clocks']}",
     f"- build alone {b['build']['ms']:.2f} ms (roofline frac {b['build']['roofline']['frac']:.3f} "
     f"of {b['build']['roofline']['peak']} GB/s at 72 B/item); draws alone {b['sample']['ms']:.2f} ms "
     f"(frac {b['roofline']['frac']:.3f} at 36 B/sample)",
     f"- aggregate (configs[3] shape, 1 GPU): {b['aggregate']['ms']:.2f} ms per 1e9 draws",
     f"- e2e through the C ABI with host buffers: {b['e2e']['ms_per_step']:.1f} ms -> "
     f"{b['e2e']['value']:.2f} G/s (H2D {b['e2e']['h2d_bytes_per_step'] / 1e9:.1f} GB + D2H "
     f"{b['e2e']['d2h_bytes_per_step'] / 1e9:.1f} GB per step)",
     f"- reference CPU (oracle/_ref, {c['cores']} threads): {c['value']:.3f} G/s (build "
     f"{c['build_s']:.2f} s, draws {c['draw_s_per_1e9']:.2f} s per 1e9)\n",
     f"Per-kernel, one bench step (ncu launch list `{tag}_launch_list.txt`, launches 20-30; "
     "cold-cache, serialised):\n",
     "| kernel | time us | DRAM read GB | DRAM write GB | DRAM GB/s | of 6550 GB/s |",
     "|---|---|---|---|---|---|"]
for k, t, r, w in rows:
    bw = (r + w) / (t * 1e-6)
    s.append(f"| {k} | {t:.1f} | {r:.3f} | {w:.3f} | {bw:.0f} | {bw / 6550:.2f} |")
s += ["", f"Stall / issue breakdown per kernel: `{tag}_ncu_kernels.txt` (`--set full`).",
      f"Other configs: `{tag}_config0.json` (configs[0] vs the reference on the host), "
      f"`{tag}_size_sweep.md` (configs[4]), `{tag}_config3_shards.jsonl` (configs[2] per-GPU "
      f"shares), `{tag}_aggregate_shards.jsonl` (configs[3] per-GPU shares).",
      "Microbenchmarks behind the design choices (random 16-B gathers by load path, TMA gather4, "
      f"distributed shared memory, FP64 chain latencies): `{tag}_microbench_all.txt` (sources in "
      "`scripts/microbench/`)."]
open(os.path.join(P, f"{tag}_summary.md"), "w").write("\n".join(s) + "\n")
print("\n".join(s))
