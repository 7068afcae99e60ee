#!/usr/bin/env python
"""Summarise one kernel block of an `ncu --page source --csv --print-source sass`
export: instruction mix by opcode and the hottest instructions by warp
instructions executed and by stall samples.
usage: sass_hot.py FILE BLOCK_INDEX [TOP]"""
import csv
import sys
from collections import Counter


def blocks(path):
    cur, hdr, name = None, None, None
    for row in csv.reader(open(path)):
        if row and row[0] == "Kernel Name":
            if cur is not None:
                yield name, hdr, cur
            name, cur, hdr = row[1], [], None
        elif hdr is None:
            hdr = row
        else:
            cur.append(row)
    if cur is not None:
        yield name, hdr, cur


def main(path, bi, top=25):
    for i, (name, hdr, rows) in enumerate(blocks(path)):
        if i != bi:
            continue
        ix = {h: j for j, h in enumerate(hdr)}
        ie, iss = ix["Instructions Executed"], ix["Warp Stall Sampling (All Samples)"]
        tot = sum(float(r[ie] or 0) for r in rows)
        stot = sum(float(r[iss] or 0) for r in rows)
        print(f"{name}: {tot / 1e6:.2f} M warp instructions, {stot:.0f} stall samples")
        mix = Counter()
        for r in rows:
            op = r[ix["Source"]].split()[0] if r[ix["Source"]].split() else "?"
            if op.startswith("@"):
                op = r[ix["Source"]].split()[1]
            mix[op.split(".")[0]] += float(r[ie] or 0)
        print("mix:", ", ".join(f"{k} {v / tot * 100:.1f}%" for k, v in mix.most_common(18)))
        print("-- by executed")
        for r in sorted(rows, key=lambda r: -float(r[ie] or 0))[:top]:
            print(f"{r[ix['Address']]:>6} {float(r[ie] or 0) / 1e3:9.1f}K {float(r[iss] or 0):7.0f}  {r[ix['Source']][:90]}")
        print("-- by stall samples")
        for r in sorted(rows, key=lambda r: -float(r[iss] or 0))[:top]:
            print(f"{r[ix['Address']]:>6} {float(r[ie] or 0) / 1e3:9.1f}K {float(r[iss] or 0):7.0f}  {r[ix['Source']][:90]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]), int(sys.argv[3]) if len(sys.argv) > 3 else 25)
