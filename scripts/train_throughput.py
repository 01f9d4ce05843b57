"""Throughput of the public train() entry point (trainer.py:480-533) on a
BASELINE config: device-resident tables across epochs, the epoch orders from
the host prefetcher, no evaluation until the end.

    python scripts/train_throughput.py [c2] [epochs]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2304_07334_b200 import LossParams, TrainingConfig  # noqa: E402
from paper_2304_07334_b200.embeddings import InitSpec, init_matrix  # noqa: E402
from workloads import make_dataset  # noqa: E402
from paper_2304_07334_b200.trainer import configure, train  # noqa: E402

cfg_name = sys.argv[1] if len(sys.argv) > 1 else "c2"
epochs = int(sys.argv[2]) if len(sys.argv) > 2 else 20
tr, te, sp = make_dataset(cfg_name)
configure(mode="hogwild", window=sp.batch)
cfg = TrainingConfig(emb_dim=sp.dim, num_negatives=sp.negatives, learning_rate=sp.learning_rate,
                     num_threads=8, epochs=epochs, loss=LossParams(mu=sp.mu, theta=sp.theta))
S = init_matrix(tr.num_users, sp.dim, InitSpec(seed=0))
T = init_matrix(tr.num_items, sp.dim, InitSpec(seed=0))
train(S, T, tr, te, TrainingConfig(**{**cfg.__dict__, "epochs": 2}))  # warm-up (JIT-free, caches)
S = init_matrix(tr.num_users, sp.dim, InitSpec(seed=0))
T = init_matrix(tr.num_items, sp.dim, InitSpec(seed=0))
t0 = time.perf_counter()
res = train(S, T, tr, te, cfg)
wall = time.perf_counter() - t0
ep = [r.wall_time for r in res.reports]
print(json.dumps({"what": "train_throughput", "config": cfg_name, "epochs": epochs,
                  "wall_s": wall, "median_epoch_ms": sorted(ep)[len(ep) // 2] * 1e3,
                  "samples_per_s_median_epoch": tr.num_pairs / sorted(ep)[len(ep) // 2],
                  "recall@20": res.final_metrics.recall_at_k}))
