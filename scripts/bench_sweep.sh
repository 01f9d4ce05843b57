#!/bin/bash
# quick throughput sweep (no CPU baseline, no e2e) over kernel variants
CFG=${CFG:-c2}
run() { echo -n "$CFG $* : "; env "$@" timeout 300 python bench.py --config $CFG --steps 3 --warmup 2 --no-cpu --e2e-steps 0 $EXTRA 2>&1 | tail -1 | python -c "import json,sys
try:
  d=json.loads(sys.stdin.read()); print(round(d['value']/1e6,2), 'M/s frac', round(d['roofline']['frac'],3), 'loss', round(d['mean_loss'],5))
except Exception as e: print('ERR', e)"; }
for v in "$@"; do run $v; done
