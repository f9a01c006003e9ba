"""Summarise an ncu --set full report (one row per captured launch) into the
per-kernel metrics committed under profiles/: duration, DRAM bytes, DRAM and
tensor-pipe utilisation, warps active, L2 hit rate.

    python scripts/ncu_summary.py report.ncu-rep > summary.json
"""
import csv
import io
import json
import subprocess
import sys

KEYS = ["launch__grid_size", "launch__registers_per_thread", "gpu__time_duration.sum", "dram__bytes_read.sum",
        "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct"]
raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
head, units = rows[0], rows[1]
out = []
for r in rows[2:]:
    rec = {"Kernel Name": r[head.index("Kernel Name")]}
    for k in KEYS:
        if k in head:
            i = head.index(k)
            rec[k] = f"{r[i]} {units[i]}".strip()
    out.append(rec)
json.dump(out, sys.stdout, indent=1)
