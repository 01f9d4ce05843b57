#!/bin/bash
# ncu --set full of the recall/NDCG kernel on c2 (run only after the plain command exits 0)
mkdir -p gpurun_out
CMD="python scripts/measure_extras.py eval c2"
$CMD > gpurun_out/plain_eval.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:eval_fr -s 1 -c 1 -f \
    -o gpurun_out/prof_eval $CMD > gpurun_out/ncu_full_eval.log 2>&1
tail -1 gpurun_out/plain_eval.log; tail -2 gpurun_out/ncu_full_eval.log
