#!/bin/bash
# ncu capture of the hogwild kernel on the c2 bench (1 GPU), after a plain run.
set -e
mkdir -p gpurun_out
HEAT_STAGES=3 HEAT_CROSS=0 python bench.py --steps 1 --warmup 1 --no-cpu --e2e-steps 1 > gpurun_out/plain.log 2>&1
HEAT_STAGES=3 HEAT_CROSS=0 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 1 --warmup 1 --no-cpu --e2e-steps 1 > gpurun_out/ncu_launch.log 2>&1
HEAT_STAGES=3 HEAT_CROSS=0 ncu --set full --clock-control none --import-source on -k regex:hogwild -s 1 -c 1 \
    -o gpurun_out/prof_hogwild -f python bench.py --steps 1 --warmup 1 --no-cpu --e2e-steps 0 > gpurun_out/ncu_full.log 2>&1
