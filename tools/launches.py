#!/usr/bin/env python
"""Summarise an ncu --csv launch list (gpu__time_duration + dram bytes) per kernel."""
import collections
import csv
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[hi]
    ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    per = collections.defaultdict(dict)
    names = {}
    for r in rows[hi + 1:]:
        per[int(r[ii])][r[mi]] = float(r[vi].replace(",", ""))
        names[int(r[ii])] = r[ki].split("(")[0]
    return per, names


def main(path):
    per, names = load(path)
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    total = 0.0
    for i, m in per.items():
        t = m.get("gpu__time_duration.sum", 0.0)
        b = m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
        a = agg[names[i]]
        a[0] += 1
        a[1] += t
        a[2] += b
        total += t
    print(f"{'kernel':45s} {'launches':>8s} {'ms':>10s} {'share':>7s} {'dram GB/launch':>15s} {'dram GB/s':>10s}")
    for k, (c, t, b) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k:45s} {c:8d} {t / 1e6:10.2f} {t / total:7.1%} {b / c / 1e9:15.2f} {b / (t * 1e-9) / 1e9:10.1f}")
    print(f"total device time {total / 1e6:.1f} ms over {len(per)} launches")


if __name__ == "__main__":
    main(sys.argv[1])
