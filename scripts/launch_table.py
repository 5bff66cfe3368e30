#!/usr/bin/env python
"""Per-kernel totals of an ncu launch list (--metrics gpu__time_duration.sum --csv --log-file)."""
import collections
import csv
import sys


def main(path, top=30):
    rows = list(csv.reader(open(path)))
    h = [r for r in rows if r and r[0] == "ID"][0]
    i0 = rows.index(h)
    d, n = collections.defaultdict(float), collections.Counter()
    for r in rows[i0 + 1:]:
        if len(r) < len(h):
            continue
        x = dict(zip(h, r))
        if x["Metric Name"] != "gpu__time_duration.sum":
            continue
        k = x["Kernel Name"].split("(")[0][-60:]
        d[k] += float(x["Metric Value"].replace(",", "")) / 1e3
        n[k] += 1
    tot = sum(d.values())
    for k, v in sorted(d.items(), key=lambda t: -t[1])[:top]:
        print(f"{v:10.1f} us {v / tot * 100:5.1f}%  x{n[k]:5d}  {k}")
    print(f"{tot:10.1f} us total")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)
