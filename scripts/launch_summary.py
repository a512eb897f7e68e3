#!/usr/bin/env python
"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel.
Usage: python scripts/launch_summary.py launches.csv "command" > summary.txt"""
import csv
import sys
from collections import defaultdict

path, cmd = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else ""
rows = [r for r in csv.reader(open(path)) if len(r) > 10]
h = rows[0]
col = {n: i for i, n in enumerate(h)}
t = defaultdict(list)
geo = {}
for r in rows[1:]:
    if r[col["Metric Name"]] != "gpu__time_duration.sum":
        continue
    name = r[col["Kernel Name"]].split("(")[0].split("::")[-1].split("<")[0]
    if name == "spin_kernel":
        continue
    v = float(r[col["Metric Value"]].replace(",", ""))
    unit = r[col["Metric Unit"]]
    t[name].append(v / 1e3 if unit in ("nsecond", "ns") else v * (1e3 if unit in ("msecond", "ms") else 1))
    geo[name] = (r[col["Grid Size"]], r[col["Block Size"]])
tot = sum(sum(v) for v in t.values())
print("ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised launches;")
print("the profiling hold kernel spin_kernel of pgb_profile_steps is excluded)")
print(f"command: {cmd}")
print(f"{'kernel':40s} launches   mean_us  share  grid/block")
for name, v in sorted(t.items(), key=lambda kv: -sum(kv[1])):
    print(f"{name:40s} {len(v):8d} {sum(v) / len(v):9.2f} {100 * sum(v) / tot:5.1f}%  {geo[name]}")
