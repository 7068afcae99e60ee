"""Warp-stall and instruction mix summary of a one-kernel ncu capture
(gpurun_out/one_sass.csv + one_details.csv from scripts/ncu_blend_l0.sh)."""
import csv
import sys
from collections import Counter

d = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out"
rows = list(csv.reader(open(f"{d}/one_details.csv")))
h = rows[0]
for r in rows[1:]:
    m = dict(zip(h, r))
    if m["Metric Name"] in ("Duration", "DRAM Throughput", "Issue Slots Busy", "Registers Per Thread",
                            "Achieved Occupancy", "Warp Cycles Per Issued Instruction", "Grid Size", "Block Size"):
        print(m["Metric Name"], m["Metric Value"])
rows = list(csv.reader(open(f"{d}/one_sass.csv")))
h, data = rows[1], rows[2:]
I, S = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
tot = sum(int(r[I] or 0) for r in data)
ts = sum(int(r[S] or 0) for r in data)
print("warp instructions", tot, "stall samples", ts)
c = Counter()
for r in data:
    op = r[1].strip().split()
    if op:
        o = op[1] if op[0].startswith("@") else op[0]
        c[o.split(".")[0]] += int(r[I] or 0)
print("mix:", ", ".join(f"{o} {100 * v / tot:.1f}%" for o, v in c.most_common(14)))
top = sorted(range(len(data)), key=lambda i: -int(data[i][S] or 0))[:10]
for i in top:
    ctx = data[i - 1][1].strip()[:40] if i else ""
    print(f"{100 * int(data[i][S] or 0) / ts:5.1f}%  {data[i][1].strip()[:60]:60s}  after: {ctx}")
