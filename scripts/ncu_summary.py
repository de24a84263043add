"""Summarise an ncu --set full report (raw page CSV): per kernel launch the
time, DRAM traffic, occupancy, issue activity and the top stall reasons.

    ncu -i <rep> --page raw --csv > raw.csv && python scripts/ncu_summary.py raw.csv
"""
import csv
import sys

KEYS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "dram_rd"),
    ("dram__bytes_write.sum", "dram_wr"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_%"),
    ("lts__t_sector_hit_rate.pct", "l2_hit_%"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps_active_%"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_active_%"),
    ("launch__registers_per_thread", "regs"),
    ("smsp__inst_executed.sum", "warp_inst"),
]
PFX = "smsp__average_warps_issue_stalled_"
SFX = "_per_issue_active.ratio"


def main(path):
    rows = list(csv.reader(open(path)))
    h, units = rows[0], rows[1]
    stalls = [n for n in h if n.startswith(PFX) and n.endswith(SFX)]
    for r in rows[2:]:
        name = r[h.index("Kernel Name")].split("(")[0]
        parts = []
        for k, short in KEYS:
            if k in h:
                i = h.index(k)
                parts.append(f"{short}={r[i]}{units[i] if units[i] not in ('', '%') else ''}")
        st = sorted(((float(r[h.index(n)] or 0), n[len(PFX):-len(SFX)]) for n in stalls),
                    reverse=True)[:5]
        print(f"{name}: " + " ".join(parts))
        print("    stalls/issue: " + ", ".join(f"{n}={v:.2f}" for v, n in st))


if __name__ == "__main__":
    main(sys.argv[1])
