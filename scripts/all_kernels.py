"""Small invocations of every kernel family in one process: the EXACT
kernels (speculative and serial), the Hogwild families (resident, several
warps per pair, staged cp.async / TMA, registers, generic) in plain and DELTA
mode, the sampler, the evaluator variants, both aggregators and the shard
runtime.  Each asserts every pair trained and a finite loss.

Written to run under compute-sanitizer (memcheck / racecheck / synccheck:
sizes are tiny because the tools slow kernels 10-100x).  The GPU pool used
in this round refuses compute-sanitizer runs, so it serves as a quick
all-families check:  python scripts/all_kernels.py
"""

from __future__ import annotations

import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2304_07334_b200 import _native as N  # noqa: E402
from paper_2304_07334_b200.device import DeviceModel  # noqa: E402


def tables(rng, U, I, K):
    S = (rng.standard_normal((U, K)) * 0.1).astype(np.float32)
    T = (rng.standard_normal((I, K)) * 0.1).astype(np.float32)
    return S, T


def run(name, K, n_neg, pairs=64, mode=N.MODE_HOGWILD, window=32, env=None, l2=0.0,
        theta=0.1, delta=False):
    for k in ("HEAT_HOGWILD_IMPL", "HEAT_EXACT_SERIAL"):
        os.environ.pop(k, None)
    os.environ.update(env or {})
    rng = np.random.default_rng(K * 1000 + n_neg)
    S, T = tables(rng, 48, 300, K)
    m = DeviceModel(S, T, "cuda:0")
    u = rng.integers(0, 48, pairs).astype(np.int32)
    i = rng.integers(0, 300, pairs).astype(np.int32)
    du, di = m.upload_pairs(u, i)
    p = m.params(n_neg=n_neg, lr=0.01, l2=l2, mu=2.0, theta=theta, cosine=True, mode=mode,
                 stream_base=99, window=window)
    m.counters.reset()
    d = None
    if delta:
        cap = pairs * (n_neg + 1)
        d = (torch.empty(cap, dtype=torch.int32, device="cuda"),
             torch.empty((cap, K), dtype=torch.float32, device="cuda"),
             torch.zeros(1, dtype=torch.int64, device="cuda"), cap)
        p.mode = N.MODE_DELTA
    m.train_range(du, di, 0, pairs, p, delta=d)
    c = m.counters.read()
    assert c.pairs == pairs and np.isfinite(c.loss), (name, c)
    print(f"ok {name}: loss {c.loss:.4f}", flush=True)


def main():
    torch.cuda.set_device(0)
    E = N.MODE_EXACT
    run("exact-spec K32 N10", 32, 10, mode=E)
    run("exact-spec K64 N100 l2", 64, 100, mode=E, l2=0.01)
    run("exact-serial K32 N10", 32, 10, mode=E, env={"HEAT_EXACT_SERIAL": "1"})
    run("resident K64 N100", 64, 100)
    run("resident K32 N50 theta<0", 32, 50, theta=-0.2)
    run("resident K64 N100 delta", 64, 100, delta=True)
    run("multi K64 N300", 64, 300)
    run("multi K32 N300 delta", 32, 300, delta=True)
    run("staged K128 N100", 128, 100)
    run("staged K128 N300 l2 (spill)", 128, 300, l2=0.01)
    run("staged K128 N100 delta", 128, 100, delta=True)
    run("staged-tma K64 N100", 64, 100, env={"HEAT_HOGWILD_IMPL": "tma"})
    run("regs K64 N100", 64, 100, env={"HEAT_HOGWILD_IMPL": "regs"})
    run("generic K48 N20", 48, 20, env={"HEAT_HOGWILD_IMPL": "generic"})
    for k in ("HEAT_HOGWILD_IMPL", "HEAT_EXACT_SERIAL"):
        os.environ.pop(k, None)

    # sampler
    out = torch.empty(64 * 10, dtype=torch.int32, device="cuda")
    N.check(N.lib().heat_sample_negatives(7, 0, 64, 10, 300, ctypes_p(out), None))
    torch.cuda.synchronize()
    print("ok sampler", flush=True)

    # evaluator (plain and register-blocked variants) and the shard runtime
    from paper_2304_07334_b200 import TrainingConfig
    from paper_2304_07334_b200.dataset import from_user_lists
    from paper_2304_07334_b200.embeddings import EmbeddingMatrix
    from paper_2304_07334_b200.evaluator import evaluate
    rng = np.random.default_rng(5)
    S, T = tables(rng, 60, 500, 64)
    tr = from_user_lists({x: rng.choice(500, 6, replace=False) for x in range(60)},
                         num_users=60, num_items=500)
    te = from_user_lists({x: rng.choice(500, 3, replace=False) for x in range(0, 60, 2)},
                         num_users=60, num_items=500)
    for env in ({}, {"HEAT_EVAL_FMA": "1"}, {"HEAT_EVAL_PLAIN": "1"}):
        for k in ("HEAT_EVAL_FMA", "HEAT_EVAL_PLAIN"):
            os.environ.pop(k, None)
        os.environ.update(env)
        met = evaluate(EmbeddingMatrix(S), EmbeddingMatrix(T), tr, te,
                       TrainingConfig(emb_dim=64, num_negatives=10), k=20)
        print(f"ok evaluate {env}: recall {met.recall_at_k:.4f}", flush=True)

    # behaviour aggregation: deterministic (serial kernel) and throughput, with
    # the history gradient, plus the aggregated evaluation queries
    from paper_2304_07334_b200.config import AggregatorConfig
    from paper_2304_07334_b200.dataset import epoch_pairs
    from paper_2304_07334_b200.device import DeviceAggregator
    Wa = (np.eye(64) + rng.standard_normal((64, 64)) * 0.01).astype(np.float32)
    u, i = epoch_pairs(tr, 2)
    for mode in (N.MODE_EXACT, N.MODE_HOGWILD):
        m = DeviceModel(S, T, "cuda:0")
        agg = DeviceAggregator(Wa.copy(), tr, AggregatorConfig(enabled=True, gamma=0.5,
                                                               mini_batch_size=8,
                                                               max_history=5,
                                                               history_grad=True),
                               0.01, m.device)
        du, di = m.upload_pairs(u, i)
        p = m.params(n_neg=20, lr=0.01, l2=0.0, mu=2.0, theta=0.1, cosine=True, mode=mode,
                     stream_base=13, window=16)
        m.counters.reset()
        m.train_range(du, di, 0, len(u), p, agg=agg)
        assert m.counters.read().pairs == len(u)
        print(f"ok aggregator mode {mode}", flush=True)
    met = evaluate(EmbeddingMatrix(S), EmbeddingMatrix(T), tr, te,
                   TrainingConfig(emb_dim=64, num_negatives=10,
                                  aggregator=AggregatorConfig(enabled=True, gamma=0.5,
                                                              max_history=5)),
                   weights=Wa, k=20)
    print(f"ok aggregated evaluate: recall {met.recall_at_k:.4f}", flush=True)

    from paper_2304_07334_b200.parallel import NativeShardTrainer
    m = DeviceModel(S, T, "cuda:0")
    sh = NativeShardTrainer(m, 1, 0)
    u, i = epoch_pairs(tr, 3)
    p = m.params(n_neg=20, lr=0.01, l2=0.0, mu=2.0, theta=0.1, cosine=True, mode=N.MODE_DELTA,
                 stream_base=11, window=16)
    m.counters.reset()
    st = sh.train_epoch(u, i, p, 64)
    assert m.counters.read().pairs == len(u)
    sh.close()
    print(f"ok shard runtime: {st.steps} steps, {st.entries} entries", flush=True)


def ctypes_p(t):
    import ctypes
    return ctypes.c_void_p(t.data_ptr())


if __name__ == "__main__":
    main()
