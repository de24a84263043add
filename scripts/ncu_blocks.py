"""Group a kernel's SASS from an ncu report's source page by execution count
(loop bodies show up as runs of equal counts) with their share of
instructions and stall samples:
    python scripts/ncu_blocks.py REPORT.ncu-rep KERNEL_REGEX [min_share]"""
import csv
import io
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
mins = float(sys.argv[3]) if len(sys.argv) > 3 else 0.005
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-units", "base",
                      "-k", "regex:" + kre, "-c", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
start = [i for i, r in enumerate(rows) if r and r[0] == "Kernel Name"][0]
h = rows[start + 1]
data = []
for r in rows[start + 2:]:
    if not r or r[0] == "Kernel Name":
        break
    data.append(r)
ai, ie = h.index("Address"), h.index("Instructions Executed")
si, src = h.index("Warp Stall Sampling (All Samples)"), h.index("Source")
base = int(data[0][ai], 16)
out = [(int(r[ai], 16) - base, float(r[ie] or 0), float(r[si] or 0), r[src].strip()) for r in data]
T = sum(x[1] for x in out)
S = sum(x[2] for x in out) or 1
print(f"total warp instructions {T / 1e6:.1f}M")
cur = None
for a, n, s, t in out + [(0, -1, 0, "")]:
    if cur is None or abs(n - cur[1]) > 0.5:
        if cur and cur[1] * cur[3] / T > mins:
            print(f"{cur[0]:#06x}-{cur[2]:#06x} n={cur[1]:>10.0f} x{cur[3]:3d} = {cur[1] * cur[3] / 1e6:7.1f}M"
                  f" ({100 * cur[1] * cur[3] / T:4.1f}%) stall={100 * cur[4] / S:4.1f}%")
        cur = [a, n, a, 1, s]
    else:
        cur[2] = a
        cur[3] += 1
        cur[4] += s
