#!/bin/bash
# A/B of an environment knob on one box: VAR=name VALS="0 1" CFGS="cfg3 cfg4" bash scripts/ab_env.sh
cd "$(dirname "$0")/.."
for rep in 1 2; do for c in ${CFGS:-cfg3 cfg4}; do for v in ${VALS:-0 1}; do
  env $VAR=$v timeout 600 python bench.py --config $c --steps ${STEPS:-200} --warmup 5 --no-cpu-baseline --no-e2e --no-parity --no-profile --out /tmp/b.json > /dev/null 2>&1
  python -c "import json; d=json.load(open('/tmp/b.json')); print('$c $VAR=$v', round(d['value'],1), d['ms_per_step'])"
done; done; done
