#!/bin/bash
# tests + bench without ncu
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 1200 python -m pytest tests -q -m gpu -x --timeout 900 -p no:cacheprovider ${PYTEST_ARGS} 2>&1 | tee gpurun_out/pytest_gpu.txt | tail -30
timeout 900 python bench.py --config ${CFG:-cfg3} --steps ${STEPS:-200} --warmup ${WARMUP:-10} ${BENCH_ARGS} --out gpurun_out/bench_${CFG:-cfg3}.json 2>&1 | tail -3
