#!/usr/bin/env python
"""Summarise an ncu report of one kernel: headline metrics, instruction mix and hot SASS regions.
Usage: python scripts/ncu_hot.py gpurun_out/x.ncu-rep [window]"""
import collections
import csv
import io
import re
import subprocess
import sys


def main(rep, W=100):
    det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(det)))
    hdr = r[0]
    want = ("Duration", "Executed Ipc Active", "Registers Per Thread", "Achieved Active Warps Per SM",
            "Warp Cycles Per Issued Instruction", "DRAM Throughput", "L1/TEX Cache Throughput", "L2 Cache Throughput",
            "Compute (SM) Throughput", "Memory Throughput")
    for row in r[1:]:
        d = dict(zip(hdr, row))
        if d.get("Metric Name", "") in want:
            print(f"{d['Metric Name']:40s} {d['Metric Value']} {d.get('Metric Unit', '')}")
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(src)))
    h = rows[1]
    iS, iW, iI = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
    data = [x for x in rows[2:] if len(x) > iI]
    tot = sum(float(x[iI] or 0) for x in data)
    ts = sum(float(x[iW] or 0) for x in data)
    print(f"instructions {tot / 1e6:.1f} M")
    blk, stl = collections.Counter(), collections.Counter()
    for k, x in enumerate(data):
        blk[k // W] += float(x[iI] or 0)
        stl[k // W] += float(x[iW] or 0)
    print("region(start): M instr, % stall")
    print([(k * W, round(v / 1e6, 1), round(stl[k] / ts * 100, 1)) for k, v in sorted(blk.items()) if v > 0])
    op = collections.Counter()
    for x in data:
        s = re.sub(r"^@!?U?P\w+\s+", "", x[iS].strip())
        op[s.split()[0] if s else ""] += float(x[iI] or 0)
    print([(o, round(c / 1e6, 1)) for o, c in op.most_common(14)])
    top = sorted(range(len(data)), key=lambda k: -float(data[k][iW] or 0))[:15]
    for k in sorted(top):
        print(k, data[k][iI], data[k][iW], data[k][iS][:80])


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 100)
