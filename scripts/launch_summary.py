"""Summarise an ncu launch-list CSV (--metrics gpu__time_duration.sum --csv):
per kernel name, launch count and median duration; launches over 0.5 ms
listed separately (the timed repair steps vs the e2e pipeline's chunks)."""
import csv
import statistics
import sys
from collections import defaultdict


def main(path):
    rows = [r for r in csv.reader(open(path)) if r]
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    head = rows[h]
    ki, mi, vi = head.index("Kernel Name"), head.index("Metric Name"), head.index("Metric Value")
    ui = head.index("Metric Unit") if "Metric Unit" in head else None
    by = defaultdict(list)
    for r in rows[h + 1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        v = float(r[vi].replace(",", ""))
        unit = r[ui] if ui is not None else "us"
        us = v / 1000 if unit == "ns" else v * 1000 if unit == "ms" else v
        by[r[ki][:70]].append(us)
    for k, v in by.items():
        big = [x for x in v if x > 500]
        extra = f"  (launches > 0.5 ms: n={len(big)} median={statistics.median(big):.1f} us)" if big and len(big) != len(v) else ""
        print(f"{k:70s} n={len(v):4d} median={statistics.median(v):10.1f} us{extra}")


if __name__ == "__main__":
    main(sys.argv[1])
