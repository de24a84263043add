"""Summarise an ncu --csv launch list: one row per launch with time and DRAM bytes."""
import csv
import sys


def main(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = next(r for r in rows if "Metric Name" in r)
    ki, mi, vi, ii = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
    launches = {}
    for r in rows:
        if r is hdr or r[mi] == "Metric Name":
            continue
        d = launches.setdefault(int(r[ii]), {"kernel": r[ki].split("(")[0].replace("wrsb::", "")})
        d[r[mi]] = float(r[vi].replace(",", ""))
    total = 0.0
    for i, d in sorted(launches.items()):
        t = d.get("gpu__time_duration.sum", 0) / 1e3
        total += t
        rd = d.get("dram__bytes_read.sum", 0) / 1e9
        wr = d.get("dram__bytes_write.sum", 0) / 1e9
        print(f"{i:4d} {d['kernel'][:40]:40s} {t:10.1f} us  read {rd:7.3f} GB  write {wr:7.3f} GB")
    print(f"total {total:.1f} us")


if __name__ == "__main__":
    main(sys.argv[1])
