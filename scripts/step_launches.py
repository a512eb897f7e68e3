"""One step of an ncu launch list (gpu__time_duration.sum, --csv): the kernels
between two aggregation launches, in order, with grid and time (us)."""
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
c = {n: i for i, n in enumerate(h)}
seq = []
for r in rows[1:]:
    if r[c["Metric Name"]] != "gpu__time_duration.sum":
        continue
    name = r[c["Kernel Name"]].split("(")[0].replace("void ", "").replace("pgb::", "")
    v = float(r[c["Metric Value"]].replace(",", ""))
    u = r[c["Metric Unit"]]
    us = v / 1e3 if u in ("nsecond", "ns") else v * (1e3 if u in ("msecond", "ms") else 1)
    seq.append((name[:40], r[c["Grid Size"]], us))
idx = [i for i, (n, g, u) in enumerate(seq) if n.startswith("aggregate")]
a, b = idx[0], idx[1]
tot = 0.0
for n, g, us in seq[a + 1:b + 1]:
    print(f"{n:42s} {g:16s} {us:9.1f}")
    tot += us
print(f"step total {tot:.1f} us")
