#!/bin/bash
# Scaling sweep of the user-sharded path on one node: bench.py at N = 1, 2, 4, 8
# GPUs (one rank per GPU, NCCL), then the parallel efficiency
# value(N) / (N * value(1)) per config.  Needs a box with >= 8 GPUs.
#   bash scripts/scale_sweep.sh [c4 c5 ...]
CONFIGS=${@:-c4 c5}
mkdir -p gpurun_out
for c in $CONFIGS; do
  out=gpurun_out/scale_$c.jsonl
  rm -f $out
  # N = 1 through the same sharded step code (--sharded), so the ratio
  # isolates the exchange and the sharding
  timeout 1200 python bench.py --config $c --sharded --steps 3 --warmup 2 --no-cpu \
      --e2e-steps 0 >> $out 2> gpurun_out/scale_${c}_1.err
  for n in 2 4 8; do
    timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n \
        --master-addr 127.0.0.1 --master-port $((29500 + n)) bench.py --gpus $n \
        --config $c --steps 3 --warmup 2 --e2e-steps 0 >> $out 2> gpurun_out/scale_${c}_$n.err
  done
  python - "$out" <<'PY'
import json, sys
rows = [json.loads(l) for l in open(sys.argv[1]) if l.startswith("{")]
base = next((r["value"] for r in rows if r["n_gpus"] == 1), None)
for r in rows:
    eff = r["value"] / (r["n_gpus"] * base) if base else None
    print(json.dumps({"config": r["config"]["workload"], "n_gpus": r["n_gpus"],
                      "samples_per_s": r["value"], "efficiency": eff}))
PY
done
