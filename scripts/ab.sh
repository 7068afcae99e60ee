#!/bin/bash
# per-kernel device times of the product build and every build/variants/* library (cfg3 by default)
cd "$(dirname "$0")/.."
CFG=${CFG:-cfg3}
for lib in paper_1810_03988_b200/_lib/liblorbpano_b200.so build/variants/*/liblorbpano_b200.so; do
  LPB_LIB=$lib timeout 300 python bench.py --config $CFG --steps ${STEPS:-100} --warmup 5 --no-e2e --no-cpu-baseline --out /tmp/ab.json > /dev/null 2>&1
  python -c "
import json,sys; d=json.load(open('/tmp/ab.json')); k=d['kernel_ms']
print(sys.argv[1].split('/')[-2], round(d['value'],1), {n: k[n] for n in list(k)[:6]}, d['rank_checksums'], 'parity', (d.get('parity') or {}).get('equal'))" $lib
done
