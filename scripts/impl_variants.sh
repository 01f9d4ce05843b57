#!/bin/bash
# kernel-only timing of the default bench workload under implementation
# switches given as arguments (each "VAR=value [VAR=value]" or "" for default)
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
for v in "$@"; do
  echo "== $v" >> gpurun_out/variants.log
  env $v timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu --e2e-steps 0 ${BENCH_ARGS} 2>>gpurun_out/variants.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e6,3), 'M', round(d['roofline']['frac'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'], 'loss', round(d['mean_loss'],6))" >> gpurun_out/variants.log
done
