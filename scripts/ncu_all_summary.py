#!/usr/bin/env python
"""Per-kernel table of an ncu --set full raw CSV covering a whole step (first launch of every
kernel): duration, DRAM bytes and GB/s against the measured HBM peak, FP64 pipe %, SM throughput,
issue-active %, and the two largest stall reasons.
Usage: python scripts/ncu_all_summary.py gpurun_out/r02v_all_raw.csv.gz "note" > profiles/r02/x.json"""
import csv
import gzip
import io
import json
import sys

HBM_GBS = 6559.0  # MEASURED_PEAKS.json hbm_gbs (copy bandwidth)
STALLS = ["long_scoreboard", "short_scoreboard", "wait", "barrier", "mio_throttle", "lg_throttle", "membar",
          "math_pipe_throttle", "branch_resolving", "no_instructions", "sleeping", "dispatch_stall"]


def main(path, note=""):
    opener = gzip.open if path.endswith(".gz") else open
    with opener(path, "rt") as f:
        rows = list(csv.reader(io.StringIO(f.read())))
    h, units = rows[0], rows[1]
    seen, out = set(), []
    for v in rows[2:]:
        d = dict(zip(h, v))
        name = d.get("Kernel Name", "").split("(")[0].replace("void ", "").replace("fsfem::", "")
        if name in seen or not name:
            continue
        seen.add(name)

        def num(k):
            try:
                return float(d[k].replace(",", ""))
            except (KeyError, ValueError):
                return None
        t_us = num("gpu__time_duration.sum")
        unit_t = dict(zip(h, units)).get("gpu__time_duration.sum", "")
        if unit_t == "ms":
            t_us *= 1e3
        elif unit_t == "ns":
            t_us /= 1e3
        mb = {}
        for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            u = dict(zip(h, units)).get(k, "")
            x = num(k) or 0.0
            mb[k] = x * {"Gbyte": 1e3, "Mbyte": 1.0, "Kbyte": 1e-3, "byte": 1e-6}.get(u, 1.0)
        dram_mb = mb["dram__bytes_read.sum"] + mb["dram__bytes_write.sum"]
        gbs = dram_mb / t_us * 1e3 if t_us else None  # MB/us -> GB/s
        stalls = []
        for s in STALLS:
            x = num(f"smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio")
            if x is not None:
                stalls.append((x, s))
        stalls.sort(reverse=True)
        out.append({
            "kernel": name, "time_us": round(t_us, 2) if t_us else None, "dram_MB": round(dram_mb, 2),
            "dram_GBs": round(gbs, 1) if gbs else None, "dram_frac_of_measured_peak": round(gbs / HBM_GBS, 3) if gbs else None,
            "fp64_pipe_pct": num("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
            "sm_throughput_pct": num("sm__throughput.avg.pct_of_peak_sustained_elapsed"),
            "issue_active_pct": num("sm__inst_issued.avg.pct_of_peak_sustained_active"),
            "warps_active_pct": num("sm__warps_active.avg.pct_of_peak_sustained_active"),
            "top_stalls_per_issue": [[s, round(x, 2)] for x, s in stalls[:2]],
        })
    out.sort(key=lambda r: -(r["time_us"] or 0))
    print(json.dumps({"source": path.split("/")[-1], "note": note, "hbm_peak_GBs": HBM_GBS, "kernels": out}, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "")
