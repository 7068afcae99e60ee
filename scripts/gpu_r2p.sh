#!/bin/bash
# Round-2 evidence after the compositor rework: smoke + GPU suite, every bench
# config + the reference arm, the launch list and full-set frame captures.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 1500 python -m pytest tests -q -m gpu --timeout 900 -p no:cacheprovider 2>&1 | tee gpurun_out/pytest_gpu.txt | tail -3
bash scripts/gpu_bench_all.sh
TAG=${TAG:-r2v3} bash scripts/profile_round.sh
