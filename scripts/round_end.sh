#!/bin/bash
# Round-end evidence in one call: the GPU test suite, both bench arms on the
# default workload, the ncu launch list of the same command, the other
# configs' lines and the sharded step code at N = 1.  No number printed under
# ncu is used as a bench value.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
O=gpurun_out/round_end; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/gputest.log 2>&1; echo "pytest rc=$?" >> $O/gputest.log
timeout 600 python bench.py --impl reference > $O/bench_ref_c4.json 2> $O/bench_ref_c4.err
timeout 900 python bench.py > $O/bench_c4.json 2> $O/bench_c4.err
for c in c2 c3 c5; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 > $O/bench_$c.json 2> $O/bench_$c.err
done
: > $O/sharded_n1.jsonl
for c in c4 c5 c3; do
  timeout 900 python bench.py --config $c --sharded --steps 5 --warmup 3 --no-cpu --e2e-steps 0 >> $O/sharded_n1.jsonl 2>> $O/sharded.err
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $O/launches_c4.csv python bench.py --steps 2 --warmup 1 --e2e-steps 2 --no-cpu > $O/ncu_launches.log 2>&1
tail -2 $O/gputest.log
