#!/bin/bash
# Bench lines for every config plus the extras (no profiler in this call).
mkdir -p gpurun_out
for c in c2 c1 c3 c4 c5; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
timeout 600 python scripts/measure_extras.py > gpurun_out/extras.jsonl 2> gpurun_out/extras.err
timeout 300 python scripts/e2e_breakdown.py c2 > gpurun_out/e2e_breakdown.jsonl 2>&1
echo done
