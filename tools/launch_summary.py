"""Summarise an ncu launch list (gpu__time_duration.sum per launch): the last decode step's
kernels and the per-kernel median over the steady-state launches."""
import collections
import csv
import statistics
import sys


def main(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[start]
    ik, iv, iu = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    seq = []
    for r in rows[start + 1:]:
        v = float(r[iv].replace(",", ""))
        unit = r[iu]
        us = v / 1000.0 if unit in ("ns", "nsecond") else (v if unit in ("us", "usecond") else v * 1000.0)
        seq.append((r[ik].split("(")[0], us))
    by = collections.defaultdict(list)
    for name, us in seq[len(seq) // 2:]:
        by[name].append(us)
    print(f"{len(seq)} launches; per-kernel median over the second half (us):")
    tot = 0.0
    for name, v in by.items():
        m = statistics.median(v)
        print(f"  {m:9.2f}  x{len(v):3d}  {name}")
    print("last launches:")
    for name, us in seq[-8:]:
        print(f"  {us:9.2f}  {name}")


if __name__ == "__main__":
    main(sys.argv[1])
