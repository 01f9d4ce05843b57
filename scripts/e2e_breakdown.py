"""Where the time of one public train_epoch call goes (c2, host numpy tables):
host->device upload, kernel, device->host write-back, and the rest."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2304_07334_b200 import TrainingConfig, LossParams  # noqa: E402
from paper_2304_07334_b200.embeddings import EmbeddingMatrix, InitSpec, init_matrix  # noqa: E402
from workloads import make_dataset  # noqa: E402
from paper_2304_07334_b200.trainer import configure, train_epoch  # noqa: E402

cfg_name = sys.argv[1] if len(sys.argv) > 1 else "c2"
tr, _, sp = make_dataset(cfg_name)
S = init_matrix(tr.num_users, sp.dim, InitSpec(seed=0))
T = init_matrix(tr.num_items, sp.dim, InitSpec(seed=0))
cfg = TrainingConfig(emb_dim=sp.dim, num_negatives=sp.negatives, learning_rate=sp.learning_rate,
                     num_threads=8, loss=LossParams(mu=sp.mu, theta=sp.theta))
configure(mode="hogwild", window=sp.batch)
for e in range(3):
    train_epoch(S, T, tr, cfg, epoch=e)
rows = []
for e in range(3, 13):
    t0 = time.perf_counter()
    r = train_epoch(S, T, tr, cfg, epoch=e, collect_phases=True)
    rows.append((time.perf_counter() - t0, r.phase_times["read_emb"], r.phase_times["similarity"],
                 r.phase_times["update"]))
a = np.median(np.array(rows), axis=0) * 1e3
print(json.dumps({"what": "e2e_breakdown", "config": cfg_name, "wall_ms": a[0], "upload_ms": a[1],
                  "kernel_ms": a[2], "writeback_ms": a[3], "other_ms": a[0] - a[1] - a[2] - a[3],
                  "pairs": int(tr.num_pairs)}))
# plain copy rates for reference (best of 5 per direction)
x = torch.empty(64 << 20, dtype=torch.uint8).pin_memory()
y = torch.empty(64 << 20, dtype=torch.uint8, device="cuda")
for _ in range(3):
    y.copy_(x, non_blocking=True)
torch.cuda.synchronize()
h2d = d2h = float("inf")
for _ in range(5):
    t0 = time.perf_counter(); y.copy_(x, non_blocking=True); torch.cuda.synchronize()
    h2d = min(h2d, time.perf_counter() - t0)
    t0 = time.perf_counter(); x.copy_(y, non_blocking=True); torch.cuda.synchronize()
    d2h = min(d2h, time.perf_counter() - t0)
print(json.dumps({"what": "pcie", "h2d_GBps": (64 << 20) / h2d / 1e9, "d2h_GBps": (64 << 20) / d2h / 1e9}))
