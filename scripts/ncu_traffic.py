#!/usr/bin/env python
"""Per-kernel DRAM traffic of one steady-state frame from an
`ncu --set full --page raw --csv` export of a short bench run, keyed like the
bench's per-launch profiler ("k_blend_level/3" = 4th blend launch of a frame).
Writes/updates profiles/ncu_traffic.json and prints a summary table.
usage: ncu_traffic.py raw.csv config [frames]"""
import collections
import csv
import json
import os
import sys

FAMILY = {"k_warp_t": "k_warp", "k_detect9": "k_detect", "k_detect": "k_detect", "k_pyr_down2": "k_pyr_down", "k_describe6": "k_describe",
          "k_blend_lean": "k_blend_level", "k_blend_level": "k_blend_level",
          "k_match_query_split": "k_match_query", "k_match_query_warp": "k_match_query"}
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "ns": 1e-9, "us": 1e-6, "ms": 1e-3,
        "msecond": 1e-3, "second": 1}


def main(path, cfg, frames=None):
    rows = list(csv.reader(open(path)))
    hdr, units = rows[0], rows[1]
    ix = {n: i for i, n in enumerate(hdr)}
    launches = []
    for r in rows[2:]:
        if len(r) != len(hdr):
            continue
        name = r[ix["Kernel Name"]].split("(")[0].split("<")[0].split("::")[-1].replace("void ", "").strip()
        fam = FAMILY.get(name, name)

        def val(m):
            i = ix[m]
            return float(r[i].replace(",", "")) * UNIT.get(units[i], 1)
        def opt(m):
            return val(m) if m in ix and r[ix[m]] else None
        launches.append((fam, val("dram__bytes_read.sum") + val("dram__bytes_write.sum"),
                         val("gpu__time_duration.sum"),
                         {"issue_active_pct": opt("sm__inst_issued.avg.pct_of_peak_sustained_active"),
                          "fp64_pipe_pct": opt("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
                          "dram_pct": opt("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
                          "warps_active_pct": opt("sm__warps_active.avg.pct_of_peak_sustained_active"),
                          "registers": opt("launch__registers_per_thread")}))
    per = collections.defaultdict(list)
    for fam, b, t, lim in launches:
        per[fam].append((b, t, lim))
    if frames is None:
        frames = max(1, len(per.get("k_detect", [])))
    out = {}
    for fam, lst in per.items():
        n = max(1, len(lst) // frames)
        for occ, (b, t, lim) in enumerate(lst[-n:]):
            out[f"{fam}/{occ}"] = {"traffic_bytes": b, "ncu_us": t * 1e6, "limiter": lim}
    dst = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "ncu_traffic.json")
    allj = json.load(open(dst)) if os.path.exists(dst) else {}
    allj[cfg] = out
    json.dump(allj, open(dst, "w"), indent=1, sort_keys=True)
    for k, v in sorted(out.items(), key=lambda kv: -kv[1]["ncu_us"]):
        print(f"{k:22s} {v['ncu_us']:9.1f} us  {v['traffic_bytes'] / 1e6:9.2f} MB")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else None)
