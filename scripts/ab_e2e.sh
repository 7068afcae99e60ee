#!/bin/bash
# A/B of an environment knob on the end-to-end number (host frames in, panorama out)
cd "$(dirname "$0")/.."
for rep in 1 2; do for c in ${CFGS:-cfg3}; do for v in ${VALS:-0 1}; do
  env $VAR=$v timeout 600 python bench.py --config $c --steps ${STEPS:-100} --warmup 5 --no-cpu-baseline --no-parity --no-profile --out /tmp/b.json > /dev/null 2>&1
  python -c "import json; d=json.load(open('/tmp/b.json')); print('$c $VAR=$v', round(d['value'],1), 'e2e', round(d['e2e']['value'],1))"
done; done; done
