#!/bin/bash
# Round profiling pass (1 GPU): bench lines per config, extras, launch list and
# one ncu --set full capture of the Hogwild kernel on the default (c2) bench.
set -x
mkdir -p gpurun_out
for c in c2 c1 c3 c4; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
timeout 600 python scripts/measure_extras.py > gpurun_out/extras.jsonl 2> gpurun_out/extras.err
CMD="python bench.py --steps 2 --warmup 1 --no-cpu --e2e-steps 0"
KREGEX=${KREGEX:-hogwild}
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
$CMD > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:$KREGEX -s 1 -c 1 -f -o gpurun_out/prof_hogwild $CMD > gpurun_out/ncu_full.log 2>&1
echo done
