#!/bin/bash
# Kernel-only samples/s against the number of pairs in flight (the Hogwild
# window; the bench default is the config's batch B) for c2 and c3, for the
# default kernel family and the register-streamed one-warp-per-pair kernel.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
out=gpurun_out/window_sweep.log
: > $out
for c in c2 c3; do
  for impl in "" "HEAT_HOGWILD_IMPL=wide"; do
    for w in 512 1024 2048 4096; do
      echo -n "$c ${impl:-default} window $w: " >> $out
      env $impl timeout 300 python bench.py --config $c --window $w --steps 5 --warmup 3 --no-cpu \
        --e2e-steps 0 2>>gpurun_out/window_sweep.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e6,2), 'M samples/s, frac', round(d['roofline']['frac'],3), 'loss', round(d['mean_loss'],5))" >> $out
    done
  done
done
cat $out
