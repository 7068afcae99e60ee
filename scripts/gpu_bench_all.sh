#!/bin/bash
# All bench configurations + the reference arm, one GPU round trip (outputs under gpurun_out/).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nproc > gpurun_out/host.txt; lscpu | grep "Model name" >> gpurun_out/host.txt
timeout 600 python bench.py --out gpurun_out/bench_cfg3.json 2>&1 | tail -1 | cut -c1-200
timeout 600 python bench.py --config cfg1 --steps 300 --warmup 10 --no-cpu-baseline --out gpurun_out/bench_cfg1.json 2>&1 | tail -1 | cut -c1-200
timeout 600 python bench.py --config cfg2 --steps 100 --warmup 5 --no-cpu-baseline --out gpurun_out/bench_cfg2.json 2>&1 | tail -1 | cut -c1-200
timeout 600 python bench.py --config cfg4 --steps 50 --warmup 3 --no-cpu-baseline --out gpurun_out/bench_cfg4.json 2>&1 | tail -1 | cut -c1-200
timeout 600 python bench.py --config cfg5 --steps 8 --warmup 6 --out gpurun_out/bench_cfg5.json 2>&1 | tail -1 | cut -c1-200
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_cfg3.json 2>gpurun_out/bench_ref.err; tail -1 gpurun_out/bench_ref_cfg3.json | cut -c1-300
