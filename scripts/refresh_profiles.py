"""Regenerate profiles/ from a TAG run of scripts/gpu_round2_profile.sh
(gpurun_out/bench_<tag>.log, launches_<tag>.csv, prof_<tag>.ncu-rep):
<tag>_launch_list.txt, <tag>_launch_list.csv, <tag>_ncu_kernels.txt and
traffic.json (per-kernel DRAM bytes of one bench step).

    python scripts/refresh_profiles.py [tag]

One bench step is the first complete rebuild + draw in the launch list:
K1 .. K4b of the build, then the draw's scatter (full tiles + the partial last
tile), gather and unpermute.  The build kernels are found by name, so the
list adapts to fused / unfused K2 forms.
"""
import json
import os
import re
import shutil
import subprocess
import sys

HERE = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
tag = sys.argv[1] if len(sys.argv) > 1 else "r02b"
G = os.path.join(HERE, "gpurun_out")
P = os.path.join(HERE, "profiles")

BUILD = ["k_partition", "k_scan_blocks", "k_totals_kb", "k_scan_carry", "k_carry_ckpt",
         "k_ckpt_kb", "k_split", "k_pack", "k_assemble"]
DRAW = ["k_region_scatter", "k_region_gather", "k_region_unpermute"]


def run(*a):
    return subprocess.run([sys.executable, *a], capture_output=True, text=True, check=True).stdout


launch = run(os.path.join(HERE, "scripts", "launch_table.py"), os.path.join(G, f"launches_{tag}.csv"))
open(os.path.join(P, f"{tag}_launch_list.txt"), "w").write(launch)
shutil.copy(os.path.join(G, f"launches_{tag}.csv"), os.path.join(P, f"{tag}_launch_list.csv"))

rows = []
for line in launch.splitlines():
    m = re.match(r"\s*(\d+) (.{44}) *([\d.]+) us  read +([\d.]+) GB  write +([\d.]+) GB", line)
    if m:
        name = m.group(2).strip().replace("void ", "").split("<")[0]
        rows.append((int(m.group(1)), name, m.group(2).strip(), float(m.group(3)),
                     float(m.group(4)), float(m.group(5))))

# first k_partition* whose build is followed directly by a draw
step = None
for s, r in enumerate(rows):
    if not r[1].startswith("k_partition"):
        continue
    e = s + 1
    while e < len(rows) and any(rows[e][1].startswith(b) for b in BUILD):
        e += 1
    d = e
    while d < len(rows) and any(rows[d][1].startswith(b) for b in DRAW):
        d += 1
    if d > e:
        step = (s, e, d)
        break
assert step, "no rebuild + draw step in the launch list"
s, e, d = step
build, draw = rows[s:e], rows[e:d]
bt = sum(r[4] + r[5] for r in build)
dt = sum(r[4] + r[5] for r in draw)
n, k = 1e8, 1e9
json.dump({"draw_bytes_per_sample": round(dt * 1e9 / k, 2),
           "build_bytes_per_item": round(bt * 1e9 / n, 1),
           "source": f"profiles/{tag}_launch_list.txt (launches {rows[s][0]}-{rows[d - 1][0]}, one "
                     "bench step): ncu dram__bytes_read.sum + dram__bytes_write.sum per launch, "
                     "n=1e8 uniform, k=1e9 draws (build: " +
                     " + ".join(f"{r[1]} {r[4] + r[5]:.2f}" for r in build) + " GB; draw: " +
                     " + ".join(f"{r[1]} {r[4] + r[5]:.2f}" for r in draw) + " GB)",
           "build_kernel_us": round(sum(r[3] for r in build), 1),
           "draw_kernel_us": round(sum(r[3] for r in draw), 1)},
          open(os.path.join(P, "traffic.json"), "w"), indent=1)

rep = os.path.join(G, f"prof_{tag}.ncu-rep")
raw_csv = os.path.join(G, f"prof_{tag}_raw.csv")  # exported on the box when the report is too big to bring back
if os.path.exists(rep) or os.path.exists(raw_csv):
    if os.path.exists(rep):
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                             text=True).stdout
    else:
        raw = open(raw_csv).read()
    open("/tmp/raw_prof.csv", "w").write(raw)
    summ = run(os.path.join(HERE, "scripts", "ncu_summary.py"), "/tmp/raw_prof.csv").splitlines()
    out, seen, i = [f"# ncu --set full --clock-control none, one launch of each kernel of a bench "
                    f"step (n=1e8, k=1e9), 1x B200",
                    f"# command: TAG={tag} bash scripts/gpu_round2_profile.sh (report "
                    f"gpurun_out/prof_{tag}.ncu-rep; its raw page: profiles/{tag}_ncu_raw.csv)"], set(), 0
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

print(f"step launches {rows[s][0]}-{rows[d - 1][0]}")
print("| kernel | time us | DRAM read GB | DRAM write GB | DRAM GB/s |")
print("|---|---|---|---|---|")
for r in build + draw:
    print(f"| {r[2]} | {r[3]:.1f} | {r[4]:.3f} | {r[5]:.3f} | {(r[4] + r[5]) / (r[3] * 1e-6):.0f} |")
print(f"build {bt * 10:.1f} B/item, draw {dt:.2f} B/sample")
