#!/usr/bin/env python
"""Summarise an ncu launch list (`ncu --metrics gpu__time_duration.sum --csv --log-file F ...`):
per kernel name the launch count, total and average duration, and its share of the listed time.

    python scripts/launch_summary.py gpurun_out/launches.csv "header line" > profiles/rNN_launches_summary.txt
"""
import csv
import sys
from collections import defaultdict


def main(path: str, header: str = ""):
    rows = [r for r in csv.reader(open(path)) if r and not r[0].startswith("==")]
    hdr = rows[0]
    ki, mi, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows[1:]:
        if r[mi] != "gpu__time_duration.sum":
            continue
        v = float(r[vi].replace(",", ""))
        scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
        v *= scale.get(r[ui], 1.0)  # -> us
        name = r[ki].split("(")[0].strip()
        tot[name] += v
        cnt[name] += 1
    all_us = sum(tot.values())
    if header:
        print(header)
    for name in sorted(tot, key=lambda k: -tot[k]):
        print(f"{name[:60]:60s} n={cnt[name]:5d} total_us={tot[name]:10.1f} avg_us={tot[name] / cnt[name]:9.2f} "
              f"share={100 * tot[name] / all_us:5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "")
