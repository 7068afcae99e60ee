#!/bin/bash
# Round profile set (one GPU): the launch list of a short bench run (ncu
# gpu__time_duration, clocks untouched) and one `--set full` capture of a
# steady-state frame for config 3 and config 1, summarised by
# scripts/ncu_summary.py and scripts/ncu_traffic.py. Outputs: gpurun_out/.
# usage: TAG=v7 bash scripts/profile_round.sh
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${TAG:-v10}
export LPB_GRAPHS=0   # individual launches (graph nodes are otherwise one launch)
[ "${SKIP_LAUNCHES:-0}" = "1" ] || timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches_cfg3_$TAG.csv python bench.py --steps 2 --warmup 1 --no-e2e \
    --no-cpu-baseline --no-profile > gpurun_out/launches_cfg3_$TAG.log 2>&1
# frame 0 registers (18 kernels); config 3 then runs 13 per frame, config 1 (re-registering
# every frame) 18: capture the third frame whole, starting at its k_detect9
for CFG in cfg3 cfg1; do
  if [ $CFG = cfg3 ]; then SKIP=${SKIP3:-33}; CNT=${CNT3:-14}; else SKIP=${SKIP1:-38}; CNT=${CNT1:-19}; fi
  timeout 900 ncu --set full --clock-control none -k regex:"^(lpb::)?k_" -s $SKIP -c $CNT \
      -o gpurun_out/frame_$CFG -f python bench.py --config $CFG --steps 3 --warmup 1 --no-e2e \
      --no-cpu-baseline --no-profile > gpurun_out/frame_${CFG}_$TAG.log 2>&1
  ncu -i gpurun_out/frame_$CFG.ncu-rep --page raw --csv > gpurun_out/frame_${CFG}_${TAG}_raw.csv 2>/dev/null
  python scripts/ncu_summary.py gpurun_out/frame_${CFG}_${TAG}_raw.csv > gpurun_out/frame_${CFG}_${TAG}_summary.txt 2>&1
  rm -f gpurun_out/frame_$CFG.ncu-rep
done
ls -la gpurun_out | tail -12
