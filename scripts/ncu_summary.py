#!/usr/bin/env python
"""Summarise ncu --set full reports into a small JSON (committed under profiles/).

    python scripts/ncu_summary.py gpurun_out/attn_c2.ncu-rep [...] > profiles/xxx.json
"""
import csv
import io
import json
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "launch__occupancy_limit_shared_mem",
    "launch__occupancy_limit_registers", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
]
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "ms": 1e-3,
        "nsecond": 1e-9, "usecond": 1e-6,
        "msecond": 1e-3}


def summarize(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    head, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[head.index("Kernel Name")][:120], "report": path}
        for k in KEYS:
            if k in head:
                i = head.index(k)
                v = r[i].replace(",", "")
                try:
                    x = float(v)
                except ValueError:
                    continue
                u = units[i]
                if u in UNIT:
                    x *= UNIT[u]
                    u = "s" if u.endswith("s") and "byte" not in u else "B"
                d[k] = {"value": x, "unit": u}
        rb = d.get("dram__bytes_read.sum", {}).get("value", 0)
        wb = d.get("dram__bytes_write.sum", {}).get("value", 0)
        d["dram_bytes_per_launch"] = rb + wb
        t = d.get("gpu__time_duration.sum", {}).get("value")
        if t:
            d["dram_GBps_under_ncu"] = round((rb + wb) / t / 1e9, 1)
        res.append(d)
    return res


if __name__ == "__main__":
    allr = []
    for p in sys.argv[1:]:
        allr += summarize(p)
    json.dump(allr, sys.stdout, indent=1)
