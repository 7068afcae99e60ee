#!/bin/bash
# frames/s and the compositing kernels' per-launch ms for the given configs
cd "$(dirname "$0")/.."
for c in ${CFGS:-cfg3 cfg4}; do
  timeout 600 python bench.py --config $c --steps ${STEPS:-200} --warmup 5 --no-cpu-baseline --no-e2e --no-parity --out /tmp/b.json > /dev/null 2>&1
  python -c "import json; d=json.load(open('/tmp/b.json')); k=d['kernel_ms']; print('$c', round(d['value'],1), {n: k[n] for n in k if n[0]=='k'})"
done
