#!/usr/bin/env python3
"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list:
per-kernel total device time, launches and share."""
import collections
import csv
import sys


def main(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.OrderedDict()
    for d in data:
        k = d["Kernel Name"].split("(")[0][:70]
        agg.setdefault(k, [0.0, 0])
        agg[k][0] += float(d["Metric Value"])
        agg[k][1] += 1
    tot = sum(v[0] for v in agg.values())
    print(f"{'total us':>10} {'n':>4} {'share':>6}  kernel   ({data[0]['Metric Unit'] if data else ''})")
    for k, (v, n) in sorted(agg.items(), key=lambda x: -x[1][0]):
        print(f"{v / 1e3:10.1f} {n:4d} {100 * v / tot:5.1f}%  {k}")


if __name__ == "__main__":
    main(sys.argv[1])
