#!/usr/bin/env python
"""Attribute ncu per-instruction executed counts / stall samples to source
lines: join an `ncu --page source --csv --print-source sass` export (one
launch) with `nvdisasm -g -c` of the same cubin (line-info comments).
usage: sass_lines.py export.csv module.cubin mangled_function_name [n]"""
import collections
import csv
import re
import subprocess
import sys

exp, cubin, fn = sys.argv[1:4]
n = int(sys.argv[4]) if len(sys.argv) > 4 else 40
rows = list(csv.reader(open(exp)))
hdr = rows[1]
ix = {k: i for i, k in enumerate(hdr)}
body = [r for r in rows[2:] if len(r) == len(hdr)]
seen, uniq = set(), []
for r in body:  # exports can repeat the listing; keep the first copy
    if r[ix["Address"]] in seen:
        break
    seen.add(r[ix["Address"]])
    uniq.append(r)
dis = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
sec = dis.split(f".text.{fn}:")[1].split(".L_x_")[0] if False else dis.split(f".text.{fn}:")[1]
sec = sec.split("//---------------------")[0]
line = None
lines = []
for t in sec.splitlines():
    m = re.search(r'//## File "([^"]+)", line (\d+)', t)
    if m:
        line = f'{m.group(1).split("/")[-1]}:{m.group(2)}'
        continue
    if re.search(r"/\*[0-9a-f]{4,}\*/", t):
        lines.append(line)
if len(lines) != len(uniq):
    print(f"warning: {len(lines)} disassembled vs {len(uniq)} profiled instructions")
agg = collections.defaultdict(lambda: [0.0, 0.0])
def f(r, k):
    try:
        return float(r[ix[k]] or 0)
    except ValueError:
        return 0.0
for r, ln in zip(uniq, lines):
    agg[ln][0] += f(r, "Instructions Executed")
    agg[ln][1] += f(r, "Warp Stall Sampling (All Samples)")
ti = sum(v[0] for v in agg.values())
ts = sum(v[1] for v in agg.values()) or 1
print(f"{ti:.4g} warp inst, {ts:.0f} samples")
for ln, (ie, st) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:n]:
    print(f"{str(ln):24s} inst {ie / ti:6.1%}  stall {st / ts:6.1%}")
