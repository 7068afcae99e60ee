#!/usr/bin/env python
"""Per-kernel DRAM bytes and L2 read hit rate of one frame from two
`ncu --metrics ... --csv` launch lists (long format, one row per metric):
warm (--cache-control none) next to cold (--cache-control all).
usage: ncu_warm_summary.py warm.csv cold.csv"""
import collections
import csv
import sys

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "ns": 1e-3, "usecond": 1, "us": 1, "msecond": 1e3, "sector": 1}


def load(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ix = {n: i for i, n in enumerate(hdr)}
    per = collections.OrderedDict()
    for r in rows[1:]:
        if r[ix["ID"]] == "ID":
            continue
        k = (int(r[ix["ID"]]), r[ix["Kernel Name"]].split("(")[0].replace("void ", ""))
        v = float(r[ix["Metric Value"]].replace(",", "")) * UNIT.get(r[ix["Metric Unit"]], 1)
        per.setdefault(k, {})[r[ix["Metric Name"]]] = v
    return list(per.items())


def main(warm, cold):
    W, C = load(warm), load(cold)
    print(f"{'kernel':28s} {'warm_us':>8s} {'warm_MB':>8s} {'l2_hit%':>8s} {'cold_us':>8s} {'cold_MB':>8s}")
    tw = tc = 0.0
    for (kw, mw), (kc, mc) in zip(W, C):
        bw = (mw.get("dram__bytes_read.sum", 0) + mw.get("dram__bytes_write.sum", 0)) / 1e6
        bc = (mc.get("dram__bytes_read.sum", 0) + mc.get("dram__bytes_write.sum", 0)) / 1e6
        look = mw.get("lts__t_sectors_srcunit_tex_op_read.sum", 0)
        hit = 100.0 * mw.get("lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum", 0) / look if look else float("nan")
        tw += bw
        tc += bc
        print(f"{kw[1][:28]:28s} {mw.get('gpu__time_duration.sum', 0):8.1f} {bw:8.1f} {hit:8.1f} "
              f"{mc.get('gpu__time_duration.sum', 0):8.1f} {bc:8.1f}")
    print(f"{'frame total':28s} {'':8s} {tw:8.1f} {'':8s} {'':8s} {tc:8.1f}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
