#!/bin/bash
# DRAM traffic of one steady-state config-3 frame with the L2 left as the
# previous kernel left it (--cache-control none), next to the default
# cold-cache capture (--cache-control all, ncu flushes L2 before every kernel).
# Kernels still run one at a time under ncu (no stream overlap), so this is the
# serialised frame's traffic with L2 reuse between producer and consumer.
# Outputs: gpurun_out/warm_cfg3_<TAG>.csv, gpurun_out/cold_cfg3_<TAG>.csv
# usage: TAG=r2v8 bash scripts/ncu_warm_traffic.sh
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${TAG:-r2v8}
export LPB_GRAPHS=0
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum,lts__t_sectors_srcunit_tex_op_read.sum
for CC in none all; do
  N=$([ $CC = none ] && echo warm || echo cold)
  timeout 900 ncu --metrics $M --cache-control $CC --clock-control none -k regex:"^(lpb::)?k_" -s ${SKIP3:-33} -c ${CNT3:-14} \
      --csv --log-file gpurun_out/${N}_cfg3_$TAG.csv python bench.py --config cfg3 --steps 3 --warmup 1 --no-e2e \
      --no-cpu-baseline --no-profile --no-parity > gpurun_out/${N}_cfg3_$TAG.log 2>&1
done
python scripts/ncu_warm_summary.py gpurun_out/warm_cfg3_$TAG.csv gpurun_out/cold_cfg3_$TAG.csv > gpurun_out/warm_cold_cfg3_$TAG.txt 2>&1
cat gpurun_out/warm_cold_cfg3_$TAG.txt
