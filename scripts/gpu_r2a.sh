#!/bin/bash
# Round-2 first GPU call: pipe peaks, TMA re-check, full-size parity, bench cfg3.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > gpurun_out/nvsmi.txt
timeout 120 ./build/pipe_peaks > gpurun_out/peaks_fp64_int.json 2>&1
timeout 120 ./build/tma_probe2 > gpurun_out/tma2.json 2>&1
timeout 300 compute-sanitizer ./build/tma_probe2 > gpurun_out/tma2_sanitizer.txt 2>&1
timeout 2400 python -m pytest tests -q -m gpu --timeout 1200 -p no:cacheprovider -rA ${PYTEST_ARGS} > gpurun_out/pytest_gpu.txt 2>&1
tail -30 gpurun_out/pytest_gpu.txt
timeout 900 python bench.py --steps 100 --warmup 5 --out gpurun_out/b_cfg3.json > gpurun_out/b_cfg3.log 2>&1
tail -c 3000 gpurun_out/b_cfg3.log
