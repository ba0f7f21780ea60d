#!/usr/bin/env python
"""Summarise ncu captures for profiles/ (run here, on the CPU box).

    python tools/ncu_summary.py launches <launches.csv>          # per-kernel launch list
    python tools/ncu_summary.py full <prof.ncu-rep> [algorithmic_bytes | n:<elements>]
(n:<elements>: algorithmic bytes = n * the element size read off each kernel's
template arguments -- 8 for double / 64-bit integer kernels, else 4)
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__bytes_read.sum.per_second", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__occupancy_limit_registers", "launch__waves_per_multiprocessor",
    "sm__cycles_elapsed.avg.per_second", "dram__cycles_elapsed.avg.per_second",
    "lts__t_bytes.sum", "smsp__inst_executed.sum",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
]


def launches(path):
    text = open(path).read()
    lines = [l for l in text.splitlines() if l.startswith('"')]
    rows = list(csv.reader(io.StringIO("\n".join(lines))))
    h = rows[0]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = defaultdict(list)
    order = []
    for r in rows[1:]:
        name = r[ki]
        if name not in agg:
            order.append(name)
        agg[name].append(float(r[vi].replace(",", "")) * (1e-3 if r[ui] == "ns" else 1.0))
    total = sum(sum(v) for v in agg.values())
    out = []
    for name in order:
        v = agg[name]
        out.append({"kernel": name, "launches": len(v), "mean_us": sum(v) / len(v),
                    "total_us": sum(v), "share": sum(v) / total})
    return out


def full(path, alg_bytes=None):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    res = []
    for vals in rows[2:]:
        d = {"kernel": vals[h.index("Kernel Name")]}
        for k in KEYS:
            if k in h:
                d[k] = f"{vals[h.index(k)]} {units[h.index(k)]}".strip()
        stalls = {}
        for i, k in enumerate(h):
            if k.startswith("smsp__average_warps_issue_stalled") and k.endswith("per_issue_active.ratio"):
                try:
                    v = float(vals[i])
                except ValueError:
                    continue
                if v >= 0.05:
                    stalls[k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", "")] = v
        d["stalls_per_issue"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1]))
        if alg_bytes:
            if str(alg_bytes).startswith("n:"):
                kn = d["kernel"]
                wide = any(t in kn for t in ("double", "unsigned long", "Float64", "<long"))
                alg = int(str(alg_bytes)[2:]) * (8 if wide else 4)
            else:
                alg = float(alg_bytes)
            d["algorithmic_bytes"] = alg
            rd = float(vals[h.index("dram__bytes_read.sum")]) * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1}[units[h.index("dram__bytes_read.sum")]]
            wr = float(vals[h.index("dram__bytes_write.sum")]) * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1}[units[h.index("dram__bytes_write.sum")]]
            d["traffic_bytes"] = rd + wr
            d["traffic_over_algorithmic"] = (rd + wr) / float(alg)
        res.append(d)
    return res


if __name__ == "__main__":
    mode, path = sys.argv[1], sys.argv[2]
    if mode == "launches":
        print(json.dumps(launches(path), indent=1))
    else:
        print(json.dumps(full(path, sys.argv[3] if len(sys.argv) > 3 else None), indent=1))
