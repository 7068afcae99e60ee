#!/bin/bash
# TMA pyramid staging: parity tests + A/B bench (LPB_TMA=1 vs 0) at cfg3.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -m gpu -x -p no:cacheprovider -k "tma or pyramid or blend or full_size or cfg3 or chain" 2>&1 | tail -5
for m in 1 0; do
LPB_TMA=$m timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-e2e --out gpurun_out/tma$m.json > /dev/null 2>&1
python -c "
import json;d=json.load(open('gpurun_out/tma$m.json'));k=d['kernel_ms'];print('TMA=$m', round(d['value'],1), {x:k[x] for x in k if 'pyr' in x or 'blend' in x})"
done
