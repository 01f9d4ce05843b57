"""Timings beside the headline bench: EXACT (bit-parity) mode throughput, the
recall@20 evaluator, and the Hogwild kernel per config.  One JSON line per
measurement (CUDA events, after warm-up, L2 flushed before each timed call)."""

import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2304_07334_b200 import _native as N  # noqa: E402
from paper_2304_07334_b200.config import TrainingConfig  # noqa: E402
from paper_2304_07334_b200.dataset import epoch_pairs  # noqa: E402
from paper_2304_07334_b200.device import DeviceModel  # noqa: E402
from paper_2304_07334_b200.embeddings import InitSpec, init_matrix  # noqa: E402
from paper_2304_07334_b200.evaluator import evaluate_device  # noqa: E402
from paper_2304_07334_b200.rng import epoch_stream, shuffle_seed  # noqa: E402
from workloads import make_dataset  # noqa: E402

flush = torch.empty(128 * 1024 * 1024, dtype=torch.float32, device="cuda")


def timed(fn):
    flush.zero_()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / 1e3


def exact(cfg_name, npairs):
    tr, _, sp = make_dataset(cfg_name)
    S = init_matrix(tr.num_users, sp.dim, InitSpec(seed=0)).values
    T = init_matrix(tr.num_items, sp.dim, InitSpec(seed=0)).values
    m = DeviceModel(S, T)
    u, i = epoch_pairs(tr, shuffle_seed(0, 0))
    n = min(npairs, len(u))
    du, di = m.upload_pairs(u[:n], i[:n])
    p = m.params(n_neg=sp.negatives, lr=sp.learning_rate, l2=0.0, mu=sp.mu, theta=sp.theta,
                 cosine=True, mode=N.MODE_EXACT, stream_base=epoch_stream(0, 0))
    m.train_range(du, di, 0, min(n, 256), p)
    torch.cuda.synchronize()
    import ctypes
    st = (ctypes.c_ulonglong * 8)()
    N.lib().heat_exact_stats(st, 1)
    dt = timed(lambda: m.train_range(du, di, 0, n, p))
    N.lib().heat_exact_stats(st, 1)
    pairs = max(1, st[5])
    print(json.dumps({"what": "exact_mode", "config": cfg_name, "pairs": n, "seconds": dt,
                      "samples_per_s": n / dt,
                      "cycles_per_pair": {"speculate": st[0] / pairs, "wait": st[1] / pairs,
                                          "commit": st[2] / pairs},
                      "recompute_frac": {"partial": st[3] / pairs, "full": st[4] / pairs}}),
          flush=True)


def agg_hogwild(cfg_name="c2", K=128, NN=64, H=100, mb=32, window=4096, epochs=3):
    """H-ACCL: SimpleX aggregation, throughput mode, on the Gowalla-shaped c2
    data with the paper's Table-8 setting (K 128, N 64, 100 history items;
    PAPER.md:811 reports 2.13 s/epoch on 2x64-core EPYC with local
    accumulation).  Whole epochs on the device, CUDA events."""
    from paper_2304_07334_b200.config import AggregatorConfig
    from paper_2304_07334_b200.device import DeviceAggregator
    tr, _, sp = make_dataset(cfg_name)
    S = init_matrix(tr.num_users, K, InitSpec(seed=0)).values
    T = init_matrix(tr.num_items, K, InitSpec(seed=0)).values
    m = DeviceModel(S, T)
    acfg = AggregatorConfig(enabled=True, gamma=0.5, max_history=H, mini_batch_size=mb)
    agg = DeviceAggregator(np.eye(K, dtype=np.float32), tr, acfg, sp.learning_rate, m.device)
    times = []
    for e in range(epochs + 1):
        u, i = epoch_pairs(tr, shuffle_seed(0, e))
        du, di = m.upload_pairs(u, i)
        p = m.params(n_neg=NN, lr=sp.learning_rate, l2=0.0, mu=sp.mu, theta=sp.theta,
                     cosine=True, mode=N.MODE_HOGWILD, stream_base=epoch_stream(0, e),
                     window=window)
        m.counters.reset()
        dt = timed(lambda: m.train_range(du, di, 0, len(u), p, agg=agg))
        c = m.counters.read()
        if e > 0:
            times.append(dt)
    dt = float(np.median(times))
    hist = np.minimum(np.diff(tr.offsets), H)
    mean_hist = float((hist[np.repeat(np.arange(tr.num_users), np.diff(tr.offsets))]).mean())
    print(json.dumps({"what": "agg_hogwild", "config": f"{cfg_name}-shaped K{K} N{NN} H{H} mb{mb}",
                      "pairs": len(u), "window": window, "seconds_per_epoch": dt,
                      "samples_per_s": len(u) / dt, "mean_history_rows": mean_hist,
                      "mean_loss": c.loss / len(u),
                      "paper_seconds_per_epoch": 2.13, "paper_source": "PAPER.md:811 Gowalla"}),
          flush=True)


def quality(cfg_name="c2", epochs=20):
    """Statistical parity at full config-2 scale: recall@20 / NDCG@20 on the
    held-out split after `epochs` epochs of the throughput kernel (B = 1024
    pairs in flight) against the deterministic kernel, which is bit-identical
    to the reference's single thread (BASELINE config 2: 20 epochs)."""
    from paper_2304_07334_b200 import LossParams, TrainingConfig
    from paper_2304_07334_b200.embeddings import EmbeddingMatrix
    tr, te, sp = make_dataset(cfg_name)
    out = {"what": "quality", "config": cfg_name, "epochs": epochs}
    for mode in ("hogwild", "exact"):
        S = init_matrix(tr.num_users, sp.dim, InitSpec(seed=0))
        T = init_matrix(tr.num_items, sp.dim, InitSpec(seed=0))
        m = DeviceModel(S.values, T.values)
        t0 = time.perf_counter()
        losses = []
        for e in range(epochs):
            u, i = epoch_pairs(tr, shuffle_seed(0, e))
            du, di = m.upload_pairs(u, i)
            p = m.params(n_neg=sp.negatives, lr=sp.learning_rate, l2=0.0, mu=sp.mu,
                         theta=sp.theta, cosine=True,
                         mode=N.MODE_HOGWILD if mode == "hogwild" else N.MODE_EXACT,
                         stream_base=epoch_stream(0, e), window=sp.batch)
            m.counters.reset()
            m.train_range(du, di, 0, len(u), p)
            losses.append(m.counters.read().loss / len(u))
        dt = time.perf_counter() - t0
        cfg = TrainingConfig(emb_dim=sp.dim, num_negatives=sp.negatives,
                             loss=LossParams(mu=sp.mu, theta=sp.theta))
        r = evaluate_device(m, S, T, tr, te, cfg, k=20)
        out[mode] = {"recall@20": r.recall_at_k, "ndcg@20": r.ndcg_at_k,
                     "first_loss": losses[0], "last_loss": losses[-1], "train_seconds": dt}
    out["recall_gap"] = abs(out["hogwild"]["recall@20"] - out["exact"]["recall@20"])
    print(json.dumps(out), flush=True)


def agg_quality(cfg_name="c2", K=128, NN=64, H=100, mb=32, epochs=5):
    """H-ACCL parity at full scale: aggregated-query recall@20 after `epochs`
    epochs, throughput aggregator (4096-pair steps) vs the deterministic one
    (bit-identical to the reference's single thread)."""
    from paper_2304_07334_b200 import LossParams, TrainingConfig
    from paper_2304_07334_b200.config import AggregatorConfig
    from paper_2304_07334_b200.device import DeviceAggregator
    tr, te, sp = make_dataset(cfg_name)
    acfg = AggregatorConfig(enabled=True, gamma=0.5, max_history=H, mini_batch_size=mb)
    out = {"what": "agg_quality", "config": f"{cfg_name}-shaped K{K} N{NN} H{H} mb{mb}",
           "epochs": epochs}
    for mode in ("hogwild", "exact"):
        S = init_matrix(tr.num_users, K, InitSpec(seed=0))
        T = init_matrix(tr.num_items, K, InitSpec(seed=0))
        m = DeviceModel(S.values, T.values)
        agg = DeviceAggregator(np.eye(K, dtype=np.float32), tr, acfg, sp.learning_rate, m.device)
        t0 = time.perf_counter()
        for e in range(epochs):
            u, i = epoch_pairs(tr, shuffle_seed(0, e))
            du, di = m.upload_pairs(u, i)
            p = m.params(n_neg=NN, lr=sp.learning_rate, l2=0.0, mu=sp.mu, theta=sp.theta,
                         cosine=True,
                         mode=N.MODE_HOGWILD if mode == "hogwild" else N.MODE_EXACT,
                         stream_base=epoch_stream(0, e), window=4096)
            m.counters.reset()
            agg.reset_epoch()
            m.train_range(du, di, 0, len(u), p, agg=agg)
            loss = m.counters.read().loss / len(u)
        dt = time.perf_counter() - t0
        cfg = TrainingConfig(emb_dim=K, num_negatives=NN, loss=LossParams(mu=sp.mu, theta=sp.theta),
                             aggregator=acfg)
        r = evaluate_device(m, S, T, tr, te, cfg, weights=agg.W, k=20)
        out[mode] = {"recall@20": r.recall_at_k, "ndcg@20": r.ndcg_at_k, "last_loss": loss,
                     "train_seconds": dt}
    out["recall_gap"] = abs(out["hogwild"]["recall@20"] - out["exact"]["recall@20"])
    print(json.dumps(out), flush=True)


def evaluation(cfg_name):
    tr, te, sp = make_dataset(cfg_name)
    S = init_matrix(tr.num_users, sp.dim, InitSpec(seed=0))
    T = init_matrix(tr.num_items, sp.dim, InitSpec(seed=0))
    m = DeviceModel(S.values, T.values)
    cfg = TrainingConfig(emb_dim=sp.dim, num_negatives=1)
    evaluate_device(m, S, T, tr, te, cfg, k=20)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = evaluate_device(m, S, T, tr, te, cfg, k=20)
    dt = time.perf_counter() - t0
    users = r.users_evaluated
    flops = 2.0 * users * tr.num_items * sp.dim
    print(json.dumps({"what": "evaluate", "config": cfg_name, "users": users,
                      "items": tr.num_items, "seconds": dt, "recall@20": r.recall_at_k,
                      "score_gflop": flops / 1e9, "gflops": flops / dt / 1e9}), flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "exact":
        exact("c1", 20000)
        exact("c2", 50000)
        sys.exit(0)
    if len(sys.argv) > 1 and sys.argv[1] == "agg_quality":
        agg_quality()
        sys.exit(0)
    if len(sys.argv) > 1 and sys.argv[1] == "quality":
        quality()
        sys.exit(0)
    if len(sys.argv) > 1 and sys.argv[1] == "eval":
        for c in sys.argv[2:] or ["c2"]:
            evaluation(c)
        sys.exit(0)
    if len(sys.argv) > 1 and sys.argv[1] == "agg":
        agg_hogwild()
        sys.exit(0)
    exact("c1", 20000)
    exact("c2", 50000)
    evaluation("c2")
    agg_hogwild()
