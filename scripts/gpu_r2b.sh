#!/bin/bash
# Round-2 check: smoke, the whole GPU suite (incl. full-size parity vs oracle/_ref), bench cfg3.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > gpurun_out/nvsmi.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
timeout 2400 python -m pytest tests -q -m gpu --timeout 1200 -p no:cacheprovider -rA --durations=15 ${PYTEST_ARGS} > gpurun_out/pytest_gpu.txt 2>&1
tail -40 gpurun_out/pytest_gpu.txt
timeout 900 python bench.py --steps 100 --warmup 5 --out gpurun_out/b_cfg3.json > gpurun_out/b_cfg3.log 2>&1
tail -c 1500 gpurun_out/b_cfg3.log
