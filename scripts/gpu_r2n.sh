#!/bin/bash
# async re-registration: full GPU suite, then cfg1/cfg2/cfg4 bench async vs LPB_ASYNC=0 + cfg3 sanity.
cd "$(dirname "$0")/.."
timeout 1500 python -m pytest tests -q -m gpu -x -p no:cacheprovider --timeout 900 2>&1 | tail -6
for c in cfg1 cfg2 cfg4; do for a in 1 0; do
  LPB_ASYNC=$a timeout 600 python bench.py --config $c --steps 200 --warmup 10 --no-cpu-baseline --out /tmp/b.json > /dev/null 2>&1
  python -c "import json; d=json.load(open('/tmp/b.json')); print('$c async=$a', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), d['rank_checksums'])"
done; done
timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-e2e --out /tmp/b.json > /dev/null 2>&1; python -c "import json; d=json.load(open('/tmp/b.json')); print('cfg3', round(d['value'],1), d['kernel_ms']['k_warp/0'])"
