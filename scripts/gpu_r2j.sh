#!/bin/bash
# Round-2 evidence: all bench configs + the reference arm, launch list, full-set frame captures.
cd "$(dirname "$0")/.."
bash scripts/gpu_bench_all.sh
TAG=${TAG:-r2v2} bash scripts/profile_round.sh
