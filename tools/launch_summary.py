"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv).

    python tools/launch_summary.py launches.csv > summary.txt
"""
import collections
import csv
import sys


def main():
    rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
    hdr = rows[0]
    ik, iv, iu = (hdr.index("Kernel Name"), hdr.index("Metric Value"),
                  hdr.index("Metric Unit"))
    scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3,
             "ms": 1e3, "msecond": 1e3}
    agg = collections.OrderedDict()
    for r in rows[1:]:
        name = r[ik].split("(")[0]
        us = float(r[iv].replace(",", "")) * scale.get(r[iu], 1.0)
        agg.setdefault(name, []).append(us)
    total = sum(sum(v) for v in agg.values())
    print(f"{'kernel':34s} {'launches':>8s} {'mean us':>10s} {'total us':>12s} {'share':>7s}")
    for k, v in agg.items():
        print(f"{k[:34]:34s} {len(v):8d} {sum(v) / len(v):10.1f} "
              f"{sum(v):12.1f} {100 * sum(v) / total:6.2f}%")


if __name__ == "__main__":
    main()
