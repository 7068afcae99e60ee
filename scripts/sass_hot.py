#!/usr/bin/env python
"""Summarise an `ncu --page source --csv --print-source sass` export: total
executed warp instructions, per-opcode counts and the hottest instructions
(by stall samples)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix = {n: i for i, n in enumerate(hdr)}
body = [r for r in rows[2:] if len(r) == len(hdr)]
def num(r, k):
    try:
        return float(r[ix[k]] or 0)
    except (ValueError, KeyError):
        return 0.0
tot = sum(num(r, "Instructions Executed") for r in body)
samp = sum(num(r, "Warp Stall Sampling (All Samples)") for r in body)
print(f"{rows[0][1]}: {len(body)} SASS lines, {tot:.4g} warp inst, {samp:.0f} stall samples")
ops = collections.Counter()
for r in body:
    op = r[ix["Source"]].split()[0] if r[ix["Source"]].split() else "?"
    if op.startswith("@"):
        op = r[ix["Source"]].split()[1]
    ops[op.split(".")[0]] += num(r, "Instructions Executed")
print("opcodes:", ", ".join(f"{k} {v / tot:.1%}" for k, v in ops.most_common(18)))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
for r in sorted(body, key=lambda r: -num(r, "Warp Stall Sampling (All Samples)"))[:n]:
    print(f"{r[ix['Address']]:>6} {num(r, 'Warp Stall Sampling (All Samples)'):6.0f} "
          f"{num(r, 'Instructions Executed'):10.0f}  {r[ix['Source']][:90]}")
