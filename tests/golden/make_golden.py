"""Generate golden vectors from the REFERENCE implementation (heatcf).

Run in the build container, where /root/reference exists:

    PYTHONPATH=/root/reference/pkg/src:/root/repo PYTHONDONTWRITEBYTECODE=1 \
    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

Outputs (committed, read by tests on CPU and on the GPU box; nothing at test
time reads /root/reference):

- rng.json            SplitMix64 stream values (rng.py) — the reference's own
                      tests pin no literal constants, so these are the pins.
- c1_epoch.npz        config 1 (BASELINE.json configs[0]) trained with the
                      reference's per-chunk JIT loop exactly as
                      train_epoch(num_threads=1) runs it, one _train_chunk call
                      per step of B=256 pairs: running
                      loss_out / degen_out after every step, negative ids of
                      the first 64 pairs, final S/T after epochs 0 and 1, and
                      each epoch's EpochReport.mean_loss from train_epoch.
- edge_cases.npz      small hand-made cases over the branches of
                      trainer.py:176-293 (dot, l2, theta<0 with zero rows,
                      mu=0, duplicate/pos==neg ids, odd K) — initial and final
                      tables plus per-epoch mean losses.
- c2_prefix.json      first 8 steps (B=1024) of config 2 epoch 0: running
                      loss and sha256 of S/T after each step.
- c2_epoch0.json      config 2's whole epoch 0 (805 steps of B=1024): running
                      loss / degenerate count and S/T sha256 after every step.
- c3_prefix.json,     first 8 steps of configs 3 (B=1024, K 64, N 500) and 4
  c4_prefix.json      (B=2048, K 128, N 1000): the same records.
- eval.npz            evaluate() on c1-shaped data with a 20 % split (trained
                      tables from c1_epoch, k=20 and k=5, cosine and dot),
                      top-k lists of the first 64 users; evaluate() on the
                      config-2 split at init.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

import heatcf  # noqa: E402  (the reference)
from heatcf import trainer as rtrainer  # noqa: E402
from heatcf.dataset import InteractionSet as RSet, epoch_pairs as r_epoch_pairs  # noqa: E402
from heatcf.embeddings import EmbeddingMatrix as RMat, InitSpec as RInit, init_matrix as r_init  # noqa: E402
from heatcf.evaluator import evaluate as r_evaluate, _topk_from_scores  # noqa: E402
from heatcf.kernels import LossParams as RLoss  # noqa: E402
from heatcf.rng import SplitMix64, derive_stream, stream_state  # noqa: E402

from workloads import make_dataset  # noqa: E402  (data only)


def rset(s) -> RSet:
    return RSet(s.num_users, s.num_items, s.offsets.copy(), s.items.copy())


def run_steps(S, T, train, cfg, epoch, B, record_negs=0):
    """train_epoch(num_threads=1) unrolled into per-step _train_chunk calls
    (trainer.py:390-429 with chunk = B)."""
    ep_users, ep_items = r_epoch_pairs(train, stream_state(cfg.seed, 0x53485546, epoch)[0] >> 1)
    st = rtrainer._ThreadState(cfg, T, (0x45504F43, epoch, 0))
    w = np.zeros((1, 1), dtype=np.float32)
    agg = cfg.aggregator
    losses, degens, negs = [], [], []
    n = len(ep_users)

    def call(a, b):
        rtrainer._train_chunk(
            S.values, T.values, ep_users, ep_items, a, b, False, T.rows, st.rng_state,
            st.tile_ids, st.tile_emb, st.tile_ctr, cfg.sampler.refresh_interval,
            cfg.similarity == "cosine", cfg.num_negatives, cfg.learning_rate, cfg.l2_reg,
            cfg.loss.mu, cfg.loss.theta, False, w, agg.gamma, cfg.learning_rate,
            agg.mini_batch_size, False, train.offsets, train.items, agg.max_history,
            st.agg_accu, st.agg_ctr, st.ubuf, st.pooled, st.ugrad, st.wh, st.pos_buf,
            st.neg_buf, st.neg_ids, st.tts, st.sts, st.sims, st.dnegs, st.loss_out,
            st.degen_out, st.phase_cycles, False)

    i = 0
    while i < n:
        stop = min(n, i + B)
        if i < record_negs:
            for p in range(i, min(stop, record_negs)):
                call(p, p + 1)
                negs.append(st.neg_ids.copy())
            if min(stop, record_negs) < stop:
                call(min(stop, record_negs), stop)
        else:
            call(i, stop)
        losses.append(float(st.loss_out[0]))
        degens.append(int(st.degen_out[0]))
        i = stop
    return np.array(losses), np.array(degens, dtype=np.int64), np.array(negs, dtype=np.int32)


def rng_golden():
    out = {
        "derive_stream": [
            [0, [], derive_stream(0)],
            [42, [7, 3], derive_stream(42, 7, 3)],
            [0, [0x45504F43, 0, 0], derive_stream(0, 0x45504F43, 0, 0)],
            [0, [0x45504F43, 1, 0], derive_stream(0, 0x45504F43, 1, 0)],
            [7, [0x45504F43, 3, 2], derive_stream(7, 0x45504F43, 3, 2)],
            [0, [0x53485546, 0], derive_stream(0, 0x53485546, 0)],
            [2**64 - 1, [2**63], derive_stream(2**64 - 1, 2**63)],
        ],
    }
    s = SplitMix64(42, 7, 3)
    out["next_u64_42_7_3"] = [s.next_u64() for _ in range(32)]
    s = SplitMix64(9)
    out["below17_9"] = [s.below(17) for _ in range(200)]
    s = SplitMix64(0, 0x45504F43, 0, 0)
    out["below2000_epoch0"] = [s.below(2000) for _ in range(1000)]
    s = SplitMix64(5)
    out["below_2pow31m1_5"] = [s.below(2**31 - 1) for _ in range(256)]
    s = SplitMix64(5)
    out["below_92000_5"] = [s.below(92000) for _ in range(256)]
    with open(os.path.join(HERE, "rng.json"), "w") as f:
        json.dump({k: [[str(x) if isinstance(x, int) and x > 2**53 else x for x in row]
                       if isinstance(row, list) else (str(row) if row > 2**53 else row)
                       for row in v] for k, v in out.items()}, f)


def c1_golden():
    train, _, spec = make_dataset("c1")
    rtrain = rset(train)
    cfg = rtrainer.TrainingConfig(emb_dim=32, num_negatives=10, learning_rate=1e-3, epochs=2,
                                  num_threads=1, loss=RLoss(mu=10.0, theta=0.5), seed=0)
    S = r_init(train.num_users, 32, RInit(seed=0))
    T = r_init(train.num_items, 32, RInit(seed=0))
    res = {"offsets": train.offsets, "items": train.items}
    for e in range(2):
        losses, degens, negs = run_steps(S, T, rtrain, cfg, e, 256, record_negs=64 if e == 0 else 0)
        res[f"step_loss_e{e}"] = losses
        res[f"step_degen_e{e}"] = degens
        if e == 0:
            res["negs_e0"] = negs
        res[f"S_e{e}"] = S.values.copy()
        res[f"T_e{e}"] = T.values.copy()
    # the same two epochs through the public train_epoch: EpochReport values
    S2 = r_init(train.num_users, 32, RInit(seed=0))
    T2 = r_init(train.num_items, 32, RInit(seed=0))
    ml = []
    for e in range(2):
        rep = rtrainer.train_epoch(S2, T2, rtrain, cfg, epoch=e)
        ml.append(rep.mean_loss)
    assert S2.values.tobytes() == res["S_e1"].tobytes(), "per-step unroll != train_epoch"
    assert T2.values.tobytes() == res["T_e1"].tobytes()
    res["mean_loss"] = np.array(ml)
    np.savez_compressed(os.path.join(HERE, "c1_epoch.npz"), **res)
    return S2, T2


def edge_golden():
    rng = np.random.Generator(np.random.PCG64(2024))
    cases = {}

    def lists_to_set(lists, nu, ni):
        return heatcf.dataset.from_user_lists(lists, num_users=nu, num_items=ni)

    def add(name, train, S0, T0, cfg, epochs):
        S = RMat(S0.copy())
        T = RMat(T0.copy())
        ml = []
        for e in range(epochs):
            ml.append(rtrainer.train_epoch(S, T, train, cfg, epoch=e).mean_loss)
        cases[name] = dict(offsets=train.offsets, items=train.items, nu=train.num_users,
                           ni=train.num_items, S0=S0, T0=T0, S=S.values.copy(), T=T.values.copy(),
                           mean_loss=np.array(ml), K=cfg.emb_dim, N=cfg.num_negatives,
                           lr=cfg.learning_rate, l2=cfg.l2_reg, mu=cfg.loss.mu,
                           theta=cfg.loss.theta, cosine=int(cfg.similarity == "cosine"),
                           seed=cfg.seed, epochs=epochs)

    # clustered-ish random data, dot similarity + l2
    lists = {u: rng.integers(0, 240, size=int(rng.integers(1, 30))) for u in range(60)}
    tr = lists_to_set(lists, 60, 240)
    S0 = r_init(60, 16, RInit(seed=1)).values
    T0 = r_init(240, 16, RInit(seed=2)).values
    add("dot_l2", tr, S0, T0, rtrainer.TrainingConfig(
        emb_dim=16, num_negatives=8, learning_rate=0.01, similarity="dot", l2_reg=0.01,
        loss=RLoss(mu=1.0, theta=0.2), seed=7), 2)
    add("cos_l2", tr, S0, T0, rtrainer.TrainingConfig(
        emb_dim=16, num_negatives=8, learning_rate=0.05, l2_reg=0.05,
        loss=RLoss(mu=2.0, theta=0.1), seed=3), 2)
    # theta < 0 with zero rows: degenerate sims count as active for the loss
    S0z = S0.copy()
    S0z[[3, 17]] = 0.0
    T0z = T0.copy()
    T0z[[0, 5, 9, 100, 200]] = 0.0
    add("neg_theta_zero_rows", tr, S0z, T0z, rtrainer.TrainingConfig(
        emb_dim=16, num_negatives=8, learning_rate=0.05, loss=RLoss(mu=1.0, theta=-0.3),
        seed=11), 2)
    add("neg_theta_zero_rows_l2", tr, S0z, T0z, rtrainer.TrainingConfig(
        emb_dim=16, num_negatives=8, learning_rate=0.05, l2_reg=0.1,
        loss=RLoss(mu=1.0, theta=-0.3), seed=11), 1)
    # mu = 0 (negatives move only by decay)
    add("mu0_l2", tr, S0, T0, rtrainer.TrainingConfig(
        emb_dim=16, num_negatives=4, learning_rate=0.05, l2_reg=0.1,
        loss=RLoss(mu=0.0, theta=0.8), seed=5), 1)
    # tiny universe: duplicate negatives and pos == neg collisions
    tiny = lists_to_set({0: [0, 1], 1: [2], 2: [0, 1, 2]}, 3, 3)
    S0t = r_init(3, 8, RInit(seed=4)).values
    T0t = r_init(3, 8, RInit(seed=5)).values
    add("tiny_dups", tiny, S0t, T0t, rtrainer.TrainingConfig(
        emb_dim=8, num_negatives=8, learning_rate=0.05, loss=RLoss(mu=1.0, theta=-0.9),
        seed=2), 3)
    # item matrix larger than the train universe (T.rows is the sampling range)
    lists = {u: rng.integers(0, 50, size=int(rng.integers(1, 10))) for u in range(20)}
    small = lists_to_set(lists, 20, 50)
    T0big = r_init(80, 6, RInit(seed=9)).values
    S0s = r_init(25, 6, RInit(seed=8)).values
    add("odd_K_big_T", small, S0s, T0big, rtrainer.TrainingConfig(
        emb_dim=6, num_negatives=5, learning_rate=0.05, loss=RLoss(mu=1.0, theta=0.0),
        seed=13), 3)
    # larger K, large N, realistic theta
    lists = {u: rng.integers(0, 500, size=int(rng.integers(1, 40))) for u in range(100)}
    mid = lists_to_set(lists, 100, 500)
    add("K128_N300", mid, r_init(100, 128, RInit(seed=0)).values,
        r_init(500, 128, RInit(seed=0)).values, rtrainer.TrainingConfig(
            emb_dim=128, num_negatives=300, learning_rate=1e-3, loss=RLoss(mu=300.0, theta=0.1),
            seed=0), 1)
    flat = {}
    for name, d in cases.items():
        for k, v in d.items():
            flat[f"{name}/{k}"] = np.asarray(v)
    np.savez_compressed(os.path.join(HERE, "edge_cases.npz"), names=np.array(list(cases)), **flat)


def c2_prefix_golden(steps=8, B=1024):
    train, _, spec = make_dataset("c2")
    rtrain = rset(train)
    cfg = rtrainer.TrainingConfig(emb_dim=64, num_negatives=100, learning_rate=1e-3,
                                  num_threads=1, loss=RLoss(mu=150.0, theta=0.9), seed=0)
    S = r_init(train.num_users, 64, RInit(seed=0))
    T = r_init(train.num_items, 64, RInit(seed=0))
    ep_users, ep_items = r_epoch_pairs(rtrain, stream_state(0, 0x53485546, 0)[0] >> 1)
    n = steps * B
    sub_u, sub_i = ep_users[:n].copy(), ep_items[:n].copy()
    st = rtrainer._ThreadState(cfg, T, (0x45504F43, 0, 0))
    w = np.zeros((1, 1), dtype=np.float32)
    out = {"steps": steps, "B": B, "loss": [], "degen": [], "S_sha256": [], "T_sha256": []}
    for s in range(steps):
        rtrainer._train_chunk(
            S.values, T.values, sub_u, sub_i, s * B, (s + 1) * B, False, T.rows, st.rng_state,
            st.tile_ids, st.tile_emb, st.tile_ctr, 1, True, 100, 1e-3, 0.0, 150.0, 0.9, False,
            w, 0.5, 1e-3, 32, False, rtrain.offsets, rtrain.items, 100, st.agg_accu,
            st.agg_ctr, st.ubuf, st.pooled, st.ugrad, st.wh, st.pos_buf, st.neg_buf,
            st.neg_ids, st.tts, st.sts, st.sims, st.dnegs, st.loss_out, st.degen_out,
            st.phase_cycles, False)
        out["loss"].append(float(st.loss_out[0]))
        out["degen"].append(int(st.degen_out[0]))
        out["S_sha256"].append(hashlib.sha256(S.values.tobytes()).hexdigest())
        out["T_sha256"].append(hashlib.sha256(T.values.tobytes()).hexdigest())
    out["pairs_sha256"] = hashlib.sha256(sub_u.tobytes() + sub_i.tobytes()).hexdigest()
    with open(os.path.join(HERE, "c2_prefix.json"), "w") as f:
        json.dump(out, f, indent=1)


def shape_golden(name: str, steps: int | None, fname: str, hash_every: int = 1):
    """Config `name` (workloads.CONFIGS) trained by the reference exactly as
    train_epoch(num_threads=1) does, one _train_chunk call per step of the
    config's B pairs: running loss / degenerate count after every step and
    sha256 of S and T after every `hash_every`-th step (and the last).
    `steps` None = the whole of epoch 0."""
    train, _, spec = make_dataset(name)
    rtrain = rset(train)
    K, N, B = spec.dim, spec.negatives, spec.batch
    S = r_init(train.num_users, K, RInit(seed=0))
    T = r_init(train.num_items, K, RInit(seed=0))
    ep_users, ep_items = r_epoch_pairs(rtrain, stream_state(0, 0x53485546, 0)[0] >> 1)
    total = len(ep_users) if steps is None else min(len(ep_users), steps * B)
    nsteps = (total + B - 1) // B
    cfg = rtrainer.TrainingConfig(emb_dim=K, num_negatives=N, learning_rate=spec.learning_rate,
                                  num_threads=1, loss=RLoss(mu=spec.mu, theta=spec.theta), seed=0)
    st = rtrainer._ThreadState(cfg, T, (0x45504F43, 0, 0))
    w = np.zeros((1, 1), dtype=np.float32)
    out = {"config": name, "steps": nsteps, "B": B, "pairs": total, "K": K, "N": N,
           "theta": spec.theta, "mu": spec.mu, "lr": spec.learning_rate,
           "loss": [], "degen": [], "hash_steps": [], "S_sha256": [], "T_sha256": []}
    for s in range(nsteps):
        a, b = s * B, min(total, (s + 1) * B)
        rtrainer._train_chunk(
            S.values, T.values, ep_users, ep_items, a, b, False, T.rows, st.rng_state,
            st.tile_ids, st.tile_emb, st.tile_ctr, 1, True, N, spec.learning_rate, 0.0,
            spec.mu, spec.theta, False, w, 0.5, spec.learning_rate, 32, False, rtrain.offsets,
            rtrain.items, 100, st.agg_accu, st.agg_ctr, st.ubuf, st.pooled, st.ugrad, st.wh,
            st.pos_buf, st.neg_buf, st.neg_ids, st.tts, st.sts, st.sims, st.dnegs, st.loss_out,
            st.degen_out, st.phase_cycles, False)
        out["loss"].append(float(st.loss_out[0]))
        out["degen"].append(int(st.degen_out[0]))
        if (s + 1) % hash_every == 0 or s == nsteps - 1:
            out["hash_steps"].append(s)
            out["S_sha256"].append(hashlib.sha256(S.values.tobytes()).hexdigest())
            out["T_sha256"].append(hashlib.sha256(T.values.tobytes()).hexdigest())
    out["pairs_sha256"] = hashlib.sha256(ep_users[:total].tobytes() +
                                         ep_items[:total].tobytes()).hexdigest()
    with open(os.path.join(HERE, fname), "w") as f:
        json.dump(out, f, indent=0)


def shapes_golden():
    """The graded shapes: config 2's whole epoch 0, and prefixes of configs 3
    and 4 (K 64 / N 500, K 128 / N 1000)."""
    shape_golden("c2", None, "c2_epoch0.json", hash_every=1)
    print("c2 epoch 0 done")
    shape_golden("c3", 8, "c3_prefix.json")
    print("c3 prefix done")
    shape_golden("c4", 8, "c4_prefix.json")
    print("c4 prefix done")


def eval_golden(S_c1, T_c1):
    tr, te, _ = make_dataset("c1", test_fraction=0.2)
    rtr, rte = rset(tr), rset(te)
    res = {"tr_offsets": tr.offsets, "tr_items": tr.items, "te_offsets": te.offsets,
           "te_items": te.items}
    for sim in ("cosine", "dot"):
        cfg = rtrainer.TrainingConfig(emb_dim=32, num_negatives=1, similarity=sim)
        for k in (20, 5):
            m = r_evaluate(S_c1, T_c1, rtr, rte, cfg, k=k)
            res[f"{sim}_k{k}"] = np.array([m.recall_at_k, m.ndcg_at_k, m.users_evaluated])
        # top-20 lists for the first 64 evaluated users
        item64 = T_c1.values.astype(np.float64)
        norms = np.sqrt(np.einsum("ij,ij->i", item64, item64))
        tops = []
        users = [u for u in range(te.num_users) if len(te.slice(u))][:64]
        for u in users:
            top = heatcf.evaluator.topk_items(S_c1.values[u], T_c1, rtr.slice(u), 20, sim)
            tops.append(np.asarray(top, dtype=np.int64))
        res[f"{sim}_top20_users"] = np.array(users)
        res[f"{sim}_top20"] = np.stack(tops)
    # config-2 split at init (S == T[:U] at init, as the CLI does)
    tr2, te2, _ = make_dataset("c2")
    S = r_init(tr2.num_users, 64, RInit(seed=0))
    T = r_init(tr2.num_items, 64, RInit(seed=0))
    cfg = rtrainer.TrainingConfig(emb_dim=64, num_negatives=1)
    m = r_evaluate(S, T, rset(tr2), rset(te2), cfg, k=20)
    res["c2_init_k20"] = np.array([m.recall_at_k, m.ndcg_at_k, m.users_evaluated])
    np.savez_compressed(os.path.join(HERE, "eval.npz"), **res)


def agg_golden():
    """SimpleX behaviour aggregation (trainer.py:148-173, 299-331) through the
    reference train_epoch(num_threads=1): final S, T, W and per-epoch loss."""
    from heatcf.aggregator import AggregatorConfig as RAgg, init_weights
    rng = np.random.Generator(np.random.PCG64(77))
    lists = {u: rng.integers(0, 240, size=int(rng.integers(0, 30))) for u in range(60)}
    tr = heatcf.dataset.from_user_lists(lists, num_users=60, num_items=240)
    cases = {}

    def add(name, K, N, agg, epochs, **kw):
        S0 = r_init(60, K, RInit(seed=1)).values
        T0 = r_init(240, K, RInit(seed=2)).values
        W0 = init_weights(K, 9)
        cfg = rtrainer.TrainingConfig(emb_dim=K, num_negatives=N, aggregator=agg, **kw)
        S, T, W = RMat(S0.copy()), RMat(T0.copy()), W0.copy()
        ml = [rtrainer.train_epoch(S, T, tr, cfg, W, epoch=e).mean_loss for e in range(epochs)]
        cases[name] = dict(S0=S0, T0=T0, W0=W0, S=S.values.copy(), T=T.values.copy(), W=W.copy(),
                           mean_loss=np.array(ml), K=K, N=N, lr=cfg.learning_rate, l2=cfg.l2_reg,
                           mu=cfg.loss.mu, theta=cfg.loss.theta,
                           cosine=int(cfg.similarity == "cosine"), seed=cfg.seed, epochs=epochs,
                           gamma=agg.gamma, agg_lr=agg.learning_rate or cfg.learning_rate,
                           mb=agg.mini_batch_size, max_history=agg.max_history,
                           hist_prop=int(agg.history_grad))

    add("basic", 16, 8, RAgg(enabled=True, gamma=0.5, max_history=20, mini_batch_size=32), 2,
        learning_rate=0.05, loss=RLoss(mu=1.0, theta=0.2), seed=7)
    add("hist_grad_l2", 16, 8, RAgg(enabled=True, gamma=0.3, max_history=5, mini_batch_size=7,
                                    history_grad=True, learning_rate=0.02), 2,
        learning_rate=0.05, l2_reg=0.01, loss=RLoss(mu=2.0, theta=0.1), seed=3)
    add("gamma0_dot", 8, 4, RAgg(enabled=True, gamma=0.0, max_history=100, mini_batch_size=1),
        1, learning_rate=0.01, similarity="dot", loss=RLoss(mu=1.0, theta=0.5), seed=5)
    add("gamma1", 16, 8, RAgg(enabled=True, gamma=1.0, max_history=10, mini_batch_size=3,
                              history_grad=True), 1,
        learning_rate=0.05, loss=RLoss(mu=1.0, theta=0.0), seed=11)
    add("K64_N50", 64, 50, RAgg(enabled=True, gamma=0.5, max_history=100, mini_batch_size=32,
                                history_grad=True), 1,
        learning_rate=1e-3, loss=RLoss(mu=50.0, theta=0.3), seed=0)
    flat = {"offsets": tr.offsets, "items": tr.items}
    for name, d in cases.items():
        for k, v in d.items():
            flat[f"{name}/{k}"] = np.asarray(v)
    np.savez_compressed(os.path.join(HERE, "agg_cases.npz"), names=np.array(list(cases)), **flat)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "shapes":
        shapes_golden()
        sys.exit(0)
    if len(sys.argv) > 1 and sys.argv[1] == "agg":
        agg_golden()
        print("agg done")
        sys.exit(0)
    rng_golden()
    print("rng done")
    S, T = c1_golden()
    print("c1 done")
    edge_golden()
    print("edge done")
    c2_prefix_golden()
    print("c2 prefix done")
    eval_golden(S, T)
    print("eval done")
    shapes_golden()
    agg_golden()
    print("agg done")
