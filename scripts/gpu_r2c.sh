#!/bin/bash
# Roofline-by-pipe check (cfg3, cfg1, cfg4) + source-level ncu of the compositor's level-0 kernels.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --out gpurun_out/rf_cfg3.json > gpurun_out/rf_cfg3.log 2>&1
timeout 600 python bench.py --config cfg1 --steps 200 --warmup 10 --no-cpu-baseline --out gpurun_out/rf_cfg1.json > gpurun_out/rf_cfg1.log 2>&1
timeout 600 python bench.py --config cfg4 --steps 30 --warmup 3 --no-cpu-baseline --out gpurun_out/rf_cfg4.json > gpurun_out/rf_cfg4.log 2>&1
tail -2 gpurun_out/rf_cfg*.log | cut -c1-300
KREGEX='k_pyr_down|k_blend_level|k_mask0|k_warp|k_detect' KSKIP=14 KCOUNT=14 TAG=src_cfg3 bash scripts/ncu_capture.sh
python scripts/ncu_summary.py gpurun_out/src_cfg3_raw.csv
