#!/usr/bin/env python
"""Per-launch DRAM traffic and key counters of each kernel in an ncu --set full
report, as the JSON bench.py reads for roofline.traffic.
Usage: python scripts/ncu_traffic_json.py report.ncu-rep out.json "source description" """
import csv
import io
import json
import subprocess
import sys

rep, out, src = sys.argv[1], sys.argv[2], sys.argv[3]
rows = list(csv.reader(io.StringIO(subprocess.run(
    ["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout)))
h, units = rows[0], rows[1]
col = {n: i for i, n in enumerate(h)}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "usecond": 1e3, "ns": 1, "us": 1e3, "ms": 1e6,
         "msecond": 1e6, "second": 1e9}


def val(r, name):
    """Value in base units (bytes, nanoseconds)."""
    try:
        i = col[name]
        return float(r[i].replace(",", "")) * SCALE.get(units[i], 1)
    except (KeyError, ValueError):
        return None


kernels = {}
for r in rows[2:]:
    name = r[col["Kernel Name"]].split("(")[0].split("::")[-1].split("<")[0].strip()
    if name in kernels:
        continue
    rd = val(r, "dram__bytes_read.sum") or 0.0
    wr = val(r, "dram__bytes_write.sum") or 0.0
    kernels[name] = {
        "dram_read_bytes": rd, "dram_write_bytes": wr, "traffic_bytes": rd + wr,
        "duration_us": (val(r, "gpu__time_duration.sum") or 0.0) / 1e3,
        "smem_wavefronts": val(r, "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"),
        "tensor_pipe_active_pct": val(r, "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"),
        "issue_active_pct": val(r, "smsp__issue_active.avg.pct_of_peak_sustained_active"),
        "sm_cycles_active_avg": val(r, "sm__cycles_active.avg"),
    }
json.dump({"source": src, "kernels": kernels}, open(out, "w"), indent=1)
print(json.dumps(kernels, indent=1))
