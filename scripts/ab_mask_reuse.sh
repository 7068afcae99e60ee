#!/bin/bash
# A/B of the seam-mask reuse (LPB_MASK_REUSE) on one box: frames/s and the
# compositing kernels' per-launch ms, two alternating repetitions
cd "$(dirname "$0")/.."
for rep in 1 2; do for c in ${CFGS:-cfg3 cfg4 cfg1 cfg2}; do for u in 0 1; do
  LPB_MASK_REUSE=$u timeout 600 python bench.py --config $c --steps 200 --warmup 5 --no-cpu-baseline --no-e2e --no-parity --out /tmp/b.json > /dev/null 2>&1
  python -c "import json; d=json.load(open('/tmp/b.json')); k=d['kernel_ms']; print('$c reuse=$u', round(d['value'],1), {n: k[n] for n in k if n.split('/')[0] in ('k_runs','k_mask0','k_pyr_down','k_warp')})"
done; done; done
