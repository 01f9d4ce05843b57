"""Config 5 at full size (the scale-out data path):
10 M users x 2 M items, 500 M interactions, K 128, N 1000, B 8192.

The host data path runs end to end:
* generation: synth.make_dataset with a process pool, one seeded stream per
  block;
* CSR: built per block, with no global sort;
* epoch order: numpy-identical native shuffle of 500 M pairs, computed on a
  host thread one epoch ahead into page-locked buffers while the GPU trains;
* upload: 4 GB of pairs per epoch.
The tables (6.1 GB) are device-resident across epochs, as in train().
One JSON line with the timings."""

import json
import os
import sys
import threading
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2304_07334_b200 import _native as N  # noqa: E402
from paper_2304_07334_b200.dataset import epoch_pairs  # noqa: E402
from paper_2304_07334_b200.device import DeviceModel  # noqa: E402
from paper_2304_07334_b200.embeddings import InitSpec, init_matrix  # noqa: E402
from paper_2304_07334_b200.rng import epoch_stream, shuffle_seed  # noqa: E402
from workloads import make_dataset  # noqa: E402

EPOCHS = int(os.environ.get("C5_EPOCHS", "2"))
out = {"what": "c5_full", "epochs": EPOCHS}
t0 = time.perf_counter()
train, _, spec = make_dataset("c5", workers=os.cpu_count() or 8)
out["generate_s"] = time.perf_counter() - t0
out["pairs"] = int(train.num_pairs)
P = train.num_pairs

t0 = time.perf_counter()
S = init_matrix(spec.num_users, spec.dim, InitSpec(seed=0)).values
T = init_matrix(spec.num_items, spec.dim, InitSpec(seed=0)).values
out["init_s"] = time.perf_counter() - t0
t0 = time.perf_counter()
model = DeviceModel(S, T)
torch.cuda.synchronize()
out["tables_h2d_s"] = time.perf_counter() - t0
out["tables_gb"] = (S.nbytes + T.nbytes) / 1e9
del S, T

pin = [(torch.empty(P, dtype=torch.int32, pin_memory=True),
        torch.empty(P, dtype=torch.int32, pin_memory=True)) for _ in range(2)]
shuffle_s = {}


def shuffle_into(e):
    t = time.perf_counter()
    u, i = pin[e % 2]
    epoch_pairs(train, shuffle_seed(0, e), out=(u.numpy(), i.numpy()))
    shuffle_s[e] = time.perf_counter() - t


shuffle_into(0)
du = torch.empty(P, dtype=torch.int32, device="cuda")
di = torch.empty(P, dtype=torch.int32, device="cuda")
rows = []
for e in range(EPOCHS):
    t_wall = time.perf_counter()
    nxt = None
    u, i = pin[e % 2]
    du.copy_(u, non_blocking=True)
    di.copy_(i, non_blocking=True)
    torch.cuda.synchronize()
    t_up = time.perf_counter() - t_wall
    if e + 1 < EPOCHS:  # next epoch's order on a host thread while this one trains
        nxt = threading.Thread(target=shuffle_into, args=(e + 1,))
        nxt.start()
    p = model.params(n_neg=spec.negatives, lr=spec.learning_rate, l2=0.0, mu=spec.mu,
                     theta=spec.theta, cosine=True, mode=N.MODE_HOGWILD,
                     stream_base=epoch_stream(0, e), window=spec.batch)
    model.counters.reset()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    model.train_range(du, di, 0, P, p)
    ev1.record()
    c = model.counters.read()
    k = ev0.elapsed_time(ev1) / 1e3
    if nxt is not None:
        nxt.join()
    wall = time.perf_counter() - t_wall
    rows.append({"epoch": e, "kernel_s": k, "samples_per_s": P / k, "wall_s": wall,
                 "wall_samples_per_s": P / wall, "pairs_upload_s": t_up,
                 "mean_loss": c.loss / P, "active_per_pair": c.active / P, "pairs": c.pairs})
out["epochs_detail"] = rows
out["shuffle_s"] = shuffle_s
bytes_pair = 4 * spec.dim * (spec.negatives + 2) + 8
k_med = float(np.median([r["kernel_s"] for r in rows]))
a_med = float(np.median([r["active_per_pair"] for r in rows]))
alg = P * (bytes_pair + 4 * spec.dim * (2 + a_med))
try:
    with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
        peak = float(json.load(f)["hbm_gbs"])
except Exception:
    peak = 6443.2
out["samples_per_s"] = P / k_med
out["achieved_GBps"] = alg / k_med / 1e9
out["roofline_frac"] = out["achieved_GBps"] / peak
print(json.dumps(out), flush=True)
