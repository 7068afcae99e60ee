#!/bin/bash
# One GPU round-trip: smoke, the GPU parity suite, and (optionally) a bench line.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv | tee gpurun_out/nvsmi.txt
nproc; lscpu | grep "Model name"
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -20
timeout ${TEST_TIMEOUT:-1500} python -m pytest tests -q -m gpu --timeout 900 -p no:cacheprovider ${PYTEST_ARGS} 2>&1 | tee gpurun_out/pytest_gpu.txt | tail -60
