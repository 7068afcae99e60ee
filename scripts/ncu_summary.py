#!/usr/bin/env python
"""One line per captured launch from an `ncu --page raw --csv` export: time,
DRAM traffic, throughput fractions, pipe utilisation, occupancy."""
import csv
import sys

COLS = [("time_us", "gpu__time_duration.sum", 1),
        ("dram_rd_MB", "dram__bytes_read.sum", 1e-6), ("dram_wr_MB", "dram__bytes_write.sum", 1e-6),
        ("dram%", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1),
        ("sm%", "sm__throughput.avg.pct_of_peak_sustained_elapsed", 1),
        ("l1%", "l1tex__throughput.avg.pct_of_peak_sustained_active", 1),
        ("issue%", "sm__inst_issued.avg.pct_of_peak_sustained_active", 1),
        ("fp64%", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", 1),
        ("alu%", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", 1),
        ("fma%", "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", 1),
        ("lsu%", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", 1),
        ("warps%", "sm__warps_active.avg.pct_of_peak_sustained_active", 1),
        ("regs", "launch__registers_per_thread", 1),
        ("winst_M", "smsp__inst_executed.sum", 1e-6)]


def main(path):
    rows = list(csv.reader(open(path)))
    hdr = rows[0]
    ix = {n: i for i, n in enumerate(hdr)}
    units = rows[1]
    print("kernel".ljust(34) + " ".join(c[0].rjust(10) for c in COLS))
    for r in rows[2:]:
        if len(r) != len(hdr):
            continue
        out = []
        for name, m, scale in COLS:
            i = ix.get(m)
            if i is None or not r[i]:
                out.append("-".rjust(10))
                continue
            v = float(r[i].replace(",", ""))
            u = units[i]
            if m.startswith("dram__bytes"):
                v *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
            if m == "gpu__time_duration.sum":
                v *= {"nsecond": 1e-3, "usecond": 1, "msecond": 1e3, "ns": 1e-3, "us": 1, "ms": 1e3}.get(u, 1)
            out.append(f"{v * scale:10.2f}")
        print(r[ix["Kernel Name"]].split("(")[0][-34:].ljust(34) + " ".join(out))


if __name__ == "__main__":
    main(sys.argv[1])
