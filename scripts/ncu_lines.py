#!/usr/bin/env python
"""Per-source-line stall breakdown of one kernel in an ncu report.
Usage: python scripts/ncu_lines.py report.ncu-rep <launch-index> [file-substring] [line-lo line-hi]"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep, idx = sys.argv[1], sys.argv[2]
fsub = sys.argv[3] if len(sys.argv) > 3 else ""
lo, hi = (int(sys.argv[4]), int(sys.argv[5])) if len(sys.argv) > 5 else (0, 10 ** 9)
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "--launch-skip", idx, "--launch-count", "1"], capture_output=True,
                     text=True).stdout
hdr = None
cur = line = None
agg = defaultdict(lambda: defaultdict(float))
text = {}
for r in csv.reader(io.StringIO(out)):
    if len(r) == 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if len(r) > 8 and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8:
        continue
    if r[0] != "":
        line = (cur, int(r[0]))
        text[line] = r[1].strip()[:60]
        continue
    for i, n in enumerate(hdr):
        if (n.startswith("stall_") and "Not Issued" not in n or n == "Instructions Executed"
                or n in ("L1 Wavefronts Shared", "L1 Wavefronts Shared Ideal")):
            try:
                agg[line][n] += float(r[i])
            except ValueError:
                pass
tot = sum(sum(v for k, v in d.items() if k.startswith("stall_")) for d in agg.values()) or 1
for k in sorted(agg, key=lambda k: (k[0], k[1])):
    if fsub not in k[0] or not lo <= k[1] <= hi:
        continue
    d = agg[k]
    s = sum(v for kk, v in d.items() if kk.startswith("stall_"))
    top = sorted(((v, kk[6:]) for kk, v in d.items() if kk.startswith("stall_")), reverse=True)[:3]
    print(f"{k[1]:4d} {100 * s / tot:5.1f}% inst {d['Instructions Executed']:9.0f} "
          f"smem-wf {d['L1 Wavefronts Shared']:8.0f} (ideal {d['L1 Wavefronts Shared Ideal']:7.0f}) " +
          " ".join(f"{n}:{v:.0f}" for v, n in top if v) + f"   {text.get(k, '')}")
