#!/usr/bin/env python
"""Summarise an ncu report: key metrics, stall reasons and hottest source
lines per kernel.  Usage: python scripts/ncu_summary.py report.ncu-rep [max_kernels]"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
maxk = int(sys.argv[2]) if len(sys.argv) > 2 else 4


def ncu(*args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


rows = list(csv.reader(io.StringIO(ncu("--page", "raw", "--csv"))))
h = rows[0]
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "lts__t_bytes.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"]
seen = set()
for idx, r in enumerate(rows[2:]):
    name = r[h.index("Kernel Name")]
    short = name.split("(")[0][-40:]
    if short in seen or len(seen) >= maxk:
        continue
    seen.add(short)
    print(f"== {short}")
    for k in KEYS:
        if k in h:
            print(f"   {k:70s} {r[h.index(k)]} {rows[1][h.index(k)]}")
    st = []
    for i, n in enumerate(h):
        if n.startswith("smsp__pcsamp_warps_issue_stalled_") and not n.endswith("not_issued"):
            try:
                st.append((float(r[i].replace(",", "")), n[33:]))
            except ValueError:
                pass
    tot = sum(v for v, _ in st) or 1
    print("   stalls: " + ", ".join(f"{n} {100 * v / tot:.0f}%" for v, n in sorted(st, reverse=True)[:6]))
    src = ncu("--page", "source", "--csv", "--print-source", "cuda,sass", "--launch-skip", str(idx),
              "--launch-count", "1")
    cur = line = None
    agg = defaultdict(lambda: [0, 0])
    text = {}
    for rr in csv.reader(io.StringIO(src)):
        if len(rr) == 2 and rr[0] == "File Path":
            cur = rr[1].split("/")[-1]
            continue
        if len(rr) < 8 or rr[0] == "Line No":
            continue
        if rr[0] != "":
            line = (cur, int(rr[0]))
            text[line] = rr[1].strip()[:70]
            continue
        try:
            agg[line][0] += int(rr[4])
            agg[line][1] += int(rr[7])
        except ValueError:
            pass
    ts = sum(v[0] for v in agg.values()) or 1
    ti = sum(v[1] for v in agg.values()) or 1
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:12]:
        print(f"   {100 * v[0] / ts:5.1f}% samp {100 * v[1] / ti:5.1f}% inst  {k[0]}:{k[1]}  {text.get(k, '')}")
