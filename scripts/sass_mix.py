"""Per-kernel SASS instruction mix of libwrs_b200.so: how many LDGSTS (sm_80
cp.async), UBLKCP (cp.async.bulk), UTMA* (tensor-map TMA), SYNCS (mbarrier),
LDG / STG / LDS / STS lines each kernel has.

    python scripts/sass_mix.py [lib] > profiles/r02_sass_mix.md
"""
import collections
import re
import subprocess
import sys

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_1903_00227_b200/libwrs_b200.so"
sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
OPS = ["LDGSTS", "UBLKCP", "UTMALDG", "UTMASTG", "SYNCS", "LDG", "STG", "LDS", "STS"]
cur, counts = None, collections.OrderedDict()
for line in sass.splitlines():
    m = re.match(r"\s*Function : (\S+)", line)
    if m:
        cur = subprocess.run(["c++filt", m.group(1)], capture_output=True, text=True).stdout.strip()
        cur = re.sub(r"\(.*", "", cur.replace("wrsb::", "").replace("void ", ""))
        counts[cur] = collections.Counter()
        continue
    if cur:
        for op in OPS:
            if re.search(r"\b" + op + r"(\.|\s)", line):
                counts[cur][op] += 1
print("# SASS instruction mix per kernel\n")
print(f"`python scripts/sass_mix.py` over `{lib}` (`cuobjdump -sass`), counting instruction "
      "lines by opcode prefix: LDGSTS = sm_80 cp.async, UBLKCP = cp.async.bulk (global<->shared), "
      "SYNCS = mbarrier operations.  Library (cub) and helper kernels omitted.\n")
print("| kernel | " + " | ".join(OPS) + " |")
print("|---" * (len(OPS) + 1) + "|")
for k, c in counts.items():
    if not k.startswith("k_") or "cub" in k:
        continue
    print(f"| `{k}` | " + " | ".join(str(c[o]) for o in OPS) + " |")
