"""Summarise ncu reports / launch lists for profiles/ (run on the CPU box).

    python scripts/ncu_summary.py rep  <file.ncu-rep> [label]      -> key metrics per launch (JSON)
    python scripts/ncu_summary.py launches <launches.csv>           -> per-kernel time share
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram__bytes.sum.per_second",
    "lts__t_sector_hit_rate.pct", "lts__t_bytes.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__occupancy_limit_registers", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__inst_executed.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__average_warp_latency_issue_stalled_long_scoreboard.ratio",
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")]}
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                d[k] = f"{r[i]} {units[i]}".strip()
        res.append(d)
    return res


def stalls(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    keep = {}
    for r in csv.reader(io.StringIO(out)):
        if len(r) > 14 and r[12] in ("Warp Cycles Per Issued Instruction", "DRAM Throughput", "Memory Throughput",
                                     "Achieved Occupancy", "Theoretical Occupancy", "Mem Busy",
                                     "Max Bandwidth", "L2 Hit Rate", "Eligible Warps Per Scheduler"):
            keep[r[12]] = f"{r[14]} {r[13]}"
    return keep


def launches(path):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[h]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    d = defaultdict(list)
    for r in rows[h + 1:]:
        if len(r) > vi:
            d[r[ki].split("(")[0]].append(float(r[vi].replace(",", "")))
    tot = sum(sum(v) for v in d.values())
    out = []
    for k, v in sorted(d.items(), key=lambda x: -sum(x[1])):
        out.append({"kernel": k, "launches": len(v), "total_us": sum(v) / 1e3, "avg_us": sum(v) / len(v) / 1e3,
                    "share": sum(v) / tot})
    return out


if __name__ == "__main__":
    mode, path = sys.argv[1], sys.argv[2]
    if mode == "rep":
        print(json.dumps({"report": path, "label": sys.argv[3] if len(sys.argv) > 3 else "",
                          "launches": raw(path), "details": stalls(path)}, indent=1))
    else:
        print(json.dumps(launches(path), indent=1))
