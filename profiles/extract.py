#!/usr/bin/env python
"""Summarise an ncu report (--set full) or a launch-list CSV into JSON.

  python profiles/extract.py report.ncu-rep  > summary.json
  python profiles/extract.py --launches launches.csv > shares.json
"""
import collections
import csv
import json
import subprocess
import sys

DETAILS = ["Duration", "Elapsed Cycles", "SM Active Cycles", "DRAM Throughput", "L2 Cache Throughput",
           "L2 Hit Rate", "Issue Slots Busy", "Registers Per Thread", "Achieved Active Warps Per SM",
           "Eligible Warps Per Scheduler", "Executed Instructions", "Dynamic Shared Memory Per Block",
           "Grid Size", "Block Size", "SM Frequency", "DRAM Frequency"]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum", "lts__t_bytes.sum",
       "sm__inst_executed_pipe_tma.sum", "smsp__inst_executed.sum",
       "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
       "smsp__issue_active.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct",
       "sm__cycles_elapsed.avg.per_second", "launch__registers_per_thread"]


def report(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h = rows[0]
    ki, ni, ui, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Unit"), h.index("Metric Value")
    res = {"kernel": rows[1][ki] if len(rows) > 1 else None, "details": {}, "raw": {}, "stalls_pct": {}}
    for r in rows[1:]:
        if len(r) > vi and r[ni] in DETAILS and r[ni] not in res["details"]:
            res["details"][r[ni]] = f"{r[vi]} {r[ui]}".strip()
    raw = list(csv.reader(subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                                         text=True).stdout.splitlines()))
    H, U, V = raw[0], raw[1], raw[2]
    for a in RAW:
        if a in H:
            res["raw"][a] = f"{V[H.index(a)]} {U[H.index(a)]}"
    st = {a.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(b.replace(",", "")) for a, b in zip(H, V)
          if a.startswith("smsp__pcsamp_warps_issue_stalled_") and not a.endswith("not_issued") and b}
    tot = sum(st.values()) or 1.0
    res["stalls_pct"] = {k: round(v / tot * 100, 1) for k, v in sorted(st.items(), key=lambda x: -x[1]) if v}
    return res


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    h = rows[0]
    ki, ni, ui, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Unit"), h.index("Metric Value")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        if r[ni] != "gpu__time_duration.sum":
            continue
        v = float(r[vi].replace(",", ""))
        v *= {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(r[ui], 1e-3)
        name = r[ki].split("(")[0]
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(a[1] for a in agg.values()) or 1.0
    return [{"kernel": k, "launches": n, "total_us": round(t, 1), "share_pct": round(t / tot * 100, 2)}
            for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1])]


if __name__ == "__main__":
    if sys.argv[1] == "--launches":
        print(json.dumps(launches(sys.argv[2]), indent=1))
    else:
        print(json.dumps(report(sys.argv[1]), indent=1))
