#!/usr/bin/env python
"""Aggregate an `ncu --page source --print-source cuda,sass --csv` export per CUDA source line:
warp-stall samples and executed instructions, top lines first.
Usage: ncu -i X.ncu-rep --page source --csv --kernel-name regex:K --print-source cuda,sass > s.csv
       python scripts/ncu_src_lines.py s.csv [top]"""
import csv
import sys


def num(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
    hdr = None
    agg = {}
    cur_line, cur_src = None, ""
    for r in rows:
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < len(hdr):
            continue
        if r[0]:
            cur_line, cur_src = int(r[0]), r[1]
        if not r[2]:
            continue
        samp = num(r[hdr.index("Warp Stall Sampling (All Samples)")])
        inst = num(r[hdr.index("Instructions Executed")])
        a = agg.setdefault(cur_line, [0.0, 0.0, cur_src])
        a[0] += samp
        a[1] += inst
    ts = sum(v[0] for v in agg.values()) or 1.0
    ti = sum(v[1] for v in agg.values()) or 1.0
    print(f"total samples {ts:.0f}, instructions {ti:.3e}")
    for ln, (s, i, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{ln:5d} {100 * s / ts:5.1f}% samp {100 * i / ti:5.1f}% inst  {src.strip()[:90]}")


if __name__ == "__main__":
    main()
