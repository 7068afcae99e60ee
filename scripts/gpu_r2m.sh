#!/bin/bash
# Drop-in engine: Pipelined variants (threads x device depth) at cfg1, 3 repeats, + acceptance 9.
cd "$(dirname "$0")/.."
for t in 1 0; do for d in 1 2 3; do
  r=""
  for i in 1 2 3; do
    v=$(LPB_ENGINE_THREADS=$t LPB_ENGINE_DEPTH=$d ./build/ref_unit/engine_bench_b200 cfg1 300 pipelined | python -c "import json,sys; print(round(json.load(sys.stdin)['frames_per_second']))")
    r="$r $v"
  done
  echo "threads=$t depth=$d cfg1 pipelined fps:$r"
done; done
for i in 1 2 3; do ./build/ref_unit/engine_bench_b200 cfg1 300 serial | python -c "import json,sys; print('serial', round(json.load(sys.stdin)['frames_per_second']))"; done
for t in 1 0; do for d in 2 3; do
  echo "threads=$t depth=$d"; for i in 1 2 3; do LPB_ENGINE_THREADS=$t LPB_ENGINE_DEPTH=$d ./build/ref_unit/acceptance_b200 | grep -E "^\[(PASS|FAIL)\] +9:" | cut -c1-120; done
done; done
