#!/bin/bash
# One ncu --set full capture of the kernels matching $KREGEX from a short
# bench run (single GPU), plus its raw-page CSV, under gpurun_out/.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
CFG=${CFG:-cfg3}
TAG=${TAG:-cap}
LPB_GRAPHS=0 timeout ${NCU_TIMEOUT:-900} ncu --set full --clock-control none --import-source on ${NCU_EXTRA} \
    -k regex:"${KREGEX:-k_detect}" -s ${KSKIP:-4} -c ${KCOUNT:-4} \
    -o gpurun_out/$TAG -f python bench.py --config $CFG --steps ${STEPS:-3} --warmup 1 --no-e2e \
    --no-cpu-baseline --no-profile > gpurun_out/${TAG}_run.log 2>&1
tail -3 gpurun_out/${TAG}_run.log
ncu -i gpurun_out/$TAG.ncu-rep --page raw --csv > gpurun_out/${TAG}_raw.csv 2>/dev/null
# per-instruction source pages of the captured launches (stall sampling)
ncu -i gpurun_out/$TAG.ncu-rep --page source --csv --print-source sass > gpurun_out/${TAG}_sass.csv 2>/dev/null
# and per CUDA source line (-lineinfo build)
ncu -i gpurun_out/$TAG.ncu-rep --page source --csv --print-source cuda > gpurun_out/${TAG}_cuda.csv 2>/dev/null
# the full report only when asked (gpurun brings back <= 64 MiB)
[ "${KEEP_REP:-0}" = "1" ] || rm -f gpurun_out/$TAG.ncu-rep
ls -la gpurun_out
