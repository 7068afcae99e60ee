#!/bin/bash
# One --set full capture (with source counters) of the level-0 k_blend_lean
# launch of a steady-state config-3 frame; source page exported as CSV.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
export LPB_GRAPHS=0
K=${KERNEL:-k_blend_lean<64>}
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"${KREGEX:-k_blend_lean}" -s ${SKIP:-8} -c 1 \
  -o gpurun_out/one -f python bench.py --config ${CFG:-cfg3} --steps 3 --warmup 1 --no-e2e --no-cpu-baseline \
  --no-profile --no-parity > gpurun_out/one.log 2>&1
ncu -i gpurun_out/one.ncu-rep --page details --csv > gpurun_out/one_details.csv 2>/dev/null
ncu -i gpurun_out/one.ncu-rep --page source --csv --print-source sass > gpurun_out/one_sass.csv 2>/dev/null
ncu -i gpurun_out/one.ncu-rep --page raw --csv > gpurun_out/one_raw.csv 2>/dev/null
ls -la gpurun_out/one*
