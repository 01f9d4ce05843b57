#!/bin/bash
# One ncu --set full capture of the training kernel of bench.py --config $1
# (run only after the same command exits 0 without ncu; one ncu per call).
CFG=${1:-c2}
KREGEX=${KREGEX:-hogwild}
CMD="python bench.py --config $CFG --steps 1 --warmup 1 --no-cpu --e2e-steps 0"
mkdir -p gpurun_out
$CMD > gpurun_out/plain_$CFG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:$KREGEX -s 1 -c 1 -f \
    -o gpurun_out/prof_$CFG $CMD > gpurun_out/ncu_full_$CFG.log 2>&1
tail -2 gpurun_out/ncu_full_$CFG.log
