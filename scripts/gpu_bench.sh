#!/bin/bash
# Bench + ncu evidence in one GPU round-trip (outputs under gpurun_out/).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
CFG=${CFG:-cfg3}
timeout 900 python bench.py --config $CFG --steps ${STEPS:-20} --warmup ${WARMUP:-5} --out gpurun_out/bench_$CFG.json 2>&1 | tail -5
# launch list (cold-cache, serialised: compare shares)
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c ${NLAUNCH:-120} --csv \
    --log-file gpurun_out/launches_$CFG.csv python bench.py --config $CFG --steps 3 --warmup 1 \
    --no-e2e --no-cpu-baseline --no-profile > gpurun_out/ncu_launch_run.log 2>&1
tail -3 gpurun_out/ncu_launch_run.log
# full capture of the heavy kernels of a steady-state frame
timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:"${KREGEX:-k_blend_level|k_warp|k_detect|k_pyr_down|k_seam}" -s ${KSKIP:-12} -c ${KCOUNT:-10} \
    -o gpurun_out/prof_$CFG -f python bench.py --config $CFG --steps 2 --warmup 1 --no-e2e \
    --no-cpu-baseline --no-profile > gpurun_out/ncu_full_run.log 2>&1
tail -3 gpurun_out/ncu_full_run.log
ls -la gpurun_out
