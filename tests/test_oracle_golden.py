"""Pin the CPU oracle to vectors produced by the reference itself.

tests/golden/* were written by tests/golden/make_golden.py running the
unmodified reference (heatcf) in the build container.  Every check here is
bit-exact: the oracle restates trainer.py:114-297 operation for operation.
"""

import hashlib
import json
import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_2304_07334_b200 import rng as hrng
from paper_2304_07334_b200.embeddings import InitSpec, init_matrix
from workloads import make_dataset

from conftest import GOLDEN


def _rng_json():
    with open(os.path.join(GOLDEN, "rng.json")) as f:
        raw = json.load(f)

    def conv(x):
        return int(x) if isinstance(x, str) else x

    return {k: [[conv(y) for y in r] if isinstance(r, list) else conv(r) for r in v]
            for k, v in raw.items()}


def test_rng_streams_match_reference():
    g = _rng_json()
    for seed, words, want in g["derive_stream"]:
        words = [int(w) if isinstance(w, str) else w for w in words]
        assert O.derive_stream(int(seed), *words) == int(want)
        assert hrng.derive_stream(int(seed), *words) == int(want)
    s = hrng.SplitMix64(42, 7, 3)
    assert [s.next_u64() for _ in range(32)] == [int(x) for x in g["next_u64_42_7_3"]]
    s = hrng.SplitMix64(9)
    assert [s.below(17) for _ in range(200)] == g["below17_9"]


def test_counter_form_equals_sequential_stream():
    g = _rng_json()
    s0 = hrng.derive_stream(0, hrng.EPOCH_SALT, 0, 0)
    got = [hrng.counter_draw(s0, n) % 2000 for n in range(1000)]
    assert got == g["below2000_epoch0"]
    ids, _ = O.sample_negatives(s0, 100, 10, 2000)
    assert ids.ravel().tolist() == g["below2000_epoch0"]
    s5 = hrng.derive_stream(5)
    assert [hrng.counter_draw(s5, n) % (2**31 - 1) for n in range(256)] == g["below_2pow31m1_5"]
    assert [hrng.counter_draw(s5, n) % 92000 for n in range(256)] == g["below_92000_5"]


def test_c1_generator_matches_golden_data():
    z = np.load(os.path.join(GOLDEN, "c1_epoch.npz"))
    train, _, _ = make_dataset("c1")
    assert np.array_equal(train.offsets, z["offsets"])
    assert np.array_equal(train.items, z["items"])


@pytest.mark.parametrize("B", [256, 1000])
def test_oracle_c1_two_epochs_bit_exact(B):
    z = np.load(os.path.join(GOLDEN, "c1_epoch.npz"))
    offsets, items = z["offsets"], z["items"]
    S = init_matrix(1000, 32, InitSpec(seed=0)).values
    T = init_matrix(2000, 32, InitSpec(seed=0)).values
    for e in range(2):
        ep_u, ep_i = O.epoch_pairs(offsets, items, 1000, O.shuffle_seed(0, e))
        state = O.derive_stream(0, 0x45504F43, e, 0)
        loss = 0.0
        losses, negs = [], []
        n = len(ep_u)
        for s0 in range(0, n, B):
            if e == 0 and s0 == 0 and B == 256:
                for p in range(64):
                    r = O.train_range(S, T, ep_u, ep_i, p, p + 1, state, n_neg=10, lr=1e-3,
                                      mu=10.0, theta=0.5, loss0=loss)
                    state, loss = r.state, r.loss
                    negs.append(r.last_neg_ids.copy())
                r = O.train_range(S, T, ep_u, ep_i, 64, min(n, B), state, n_neg=10, lr=1e-3,
                                  mu=10.0, theta=0.5, loss0=loss)
            else:
                r = O.train_range(S, T, ep_u, ep_i, s0, min(n, s0 + B), state, n_neg=10,
                                  lr=1e-3, mu=10.0, theta=0.5, loss0=loss)
            state, loss = r.state, r.loss
            losses.append(loss)
        if B == 256:
            assert np.array_equal(np.array(losses), z[f"step_loss_e{e}"])
        else:
            assert losses[-1] == z[f"step_loss_e{e}"][-1]
        if negs:
            assert np.array_equal(np.stack(negs), z["negs_e0"])
        assert S.tobytes() == z[f"S_e{e}"].tobytes()
        assert T.tobytes() == z[f"T_e{e}"].tobytes()
        assert loss / n == z["mean_loss"][e]


def test_oracle_edge_cases_bit_exact():
    z = np.load(os.path.join(GOLDEN, "edge_cases.npz"))
    for name in z["names"]:
        g = {k.split("/", 1)[1]: z[k] for k in z.files if k.startswith(f"{name}/")}
        S = g["S0"].copy()
        T = g["T0"].copy()
        nu = int(g["nu"])
        for e in range(int(g["epochs"])):
            ep_u, ep_i = O.epoch_pairs(g["offsets"], g["items"], nu,
                                       O.shuffle_seed(int(g["seed"]), e))
            state = O.derive_stream(int(g["seed"]), 0x45504F43, e, 0)
            r = O.train_range(S, T, ep_u, ep_i, 0, len(ep_u), state, n_neg=int(g["N"]),
                              lr=float(g["lr"]), l2=float(g["l2"]), mu=float(g["mu"]),
                              theta=float(g["theta"]), cosine=bool(g["cosine"]))
            assert r.loss / len(ep_u) == g["mean_loss"][e], name
        assert S.tobytes() == g["S"].tobytes(), name
        assert T.tobytes() == g["T"].tobytes(), name


def test_oracle_c2_prefix_bit_exact():
    with open(os.path.join(GOLDEN, "c2_prefix.json")) as f:
        g = json.load(f)
    train, _, _ = make_dataset("c2")
    S = init_matrix(train.num_users, 64, InitSpec(seed=0)).values
    T = init_matrix(train.num_items, 64, InitSpec(seed=0)).values
    ep_u, ep_i = O.epoch_pairs(train.offsets, train.items, train.num_users, O.shuffle_seed(0, 0))
    B, steps = g["B"], g["steps"]
    sub_u, sub_i = ep_u[:B * steps].copy(), ep_i[:B * steps].copy()
    assert hashlib.sha256(sub_u.tobytes() + sub_i.tobytes()).hexdigest() == g["pairs_sha256"]
    state = O.derive_stream(0, 0x45504F43, 0, 0)
    loss = 0.0
    for s in range(steps):
        r = O.train_range(S, T, sub_u, sub_i, s * B, (s + 1) * B, state, n_neg=100, lr=1e-3,
                          mu=150.0, theta=0.9, loss0=loss)
        state, loss = r.state, r.loss
        assert loss == g["loss"][s]
        assert hashlib.sha256(S.tobytes()).hexdigest() == g["S_sha256"][s]
        assert hashlib.sha256(T.tobytes()).hexdigest() == g["T_sha256"][s]


@pytest.mark.parametrize("fname,hash_stride", [("c3_prefix.json", 1), ("c4_prefix.json", 1),
                                             ("c2_epoch0.json", 100)])
def test_oracle_graded_shapes_bit_exact(fname, hash_stride):
    """The graded shapes from the reference: config 2's whole epoch 0 (817
    steps), and the first 8 steps of configs 3 (K 64, N 500) and 4 (K 128,
    N 1000).  The oracle's running loss equals the reference's after every
    step; S/T hashes are checked every `hash_stride`-th recorded step and at
    the end."""
    from workloads import CONFIGS
    with open(os.path.join(GOLDEN, fname)) as f:
        g = json.load(f)
    spec = CONFIGS[g["config"]]
    train, _, _ = make_dataset(g["config"])
    S = init_matrix(train.num_users, spec.dim, InitSpec(seed=0)).values
    T = init_matrix(train.num_items, spec.dim, InitSpec(seed=0)).values
    ep_u, ep_i = O.epoch_pairs(train.offsets, train.items, train.num_users, O.shuffle_seed(0, 0))
    n, B = g["pairs"], g["B"]
    assert hashlib.sha256(ep_u[:n].tobytes() + ep_i[:n].tobytes()).hexdigest() == g["pairs_sha256"]
    hashed = dict(zip(g["hash_steps"], zip(g["S_sha256"], g["T_sha256"])))
    check = set(g["hash_steps"][::hash_stride]) | {g["hash_steps"][-1]}
    state = O.derive_stream(0, 0x45504F43, 0, 0)
    loss = 0.0
    for s in range(g["steps"]):
        r = O.train_range(S, T, ep_u, ep_i, s * B, min(n, (s + 1) * B), state, n_neg=spec.negatives,
                          lr=spec.learning_rate, mu=spec.mu, theta=spec.theta, loss0=loss)
        state, loss = r.state, r.loss
        assert loss == g["loss"][s], s
        if s in check:
            assert (hashlib.sha256(S.tobytes()).hexdigest(),
                    hashlib.sha256(T.tobytes()).hexdigest()) == hashed[s], s


def test_oracle_evaluator_matches_reference():
    z = np.load(os.path.join(GOLDEN, "eval.npz"))
    c1 = np.load(os.path.join(GOLDEN, "c1_epoch.npz"))
    S, T = c1["S_e1"], c1["T_e1"]
    for sim in ("cosine", "dot"):
        for k in (20, 5):
            (rec, ndcg, n), tops = O.evaluate_ref(
                S, T, z["tr_offsets"], z["tr_items"], 1000, z["te_offsets"], z["te_items"],
                1000, k=k, similarity=sim, return_per_user=True)
            want = z[f"{sim}_k{k}"]
            assert rec == want[0] and ndcg == want[1] and n == int(want[2])
            if k == 20:
                for u, top in zip(z[f"{sim}_top20_users"], z[f"{sim}_top20"]):
                    assert list(tops[int(u)]) == list(top)


@pytest.mark.slow
def test_oracle_evaluator_c2_init():
    z = np.load(os.path.join(GOLDEN, "eval.npz"))
    tr, te, _ = make_dataset("c2")
    S = init_matrix(tr.num_users, 64, InitSpec(seed=0)).values
    T = init_matrix(tr.num_items, 64, InitSpec(seed=0)).values
    rec, ndcg, n = O.evaluate_ref(S, T, tr.offsets, tr.items, tr.num_users, te.offsets,
                                  te.items, te.num_users, k=20)
    want = z["c2_init_k20"]
    assert rec == want[0] and ndcg == want[1] and n == int(want[2])


def test_threaded_oracle_single_thread_equals_sequential():
    z = np.load(os.path.join(GOLDEN, "c1_epoch.npz"))
    S = init_matrix(1000, 32, InitSpec(seed=0)).values
    T = init_matrix(2000, 32, InitSpec(seed=0)).values
    ep_u, ep_i = O.epoch_pairs(z["offsets"], z["items"], 1000, O.shuffle_seed(0, 0))
    loss, _, _ = O.train_epoch_threads(S, T, ep_u, ep_i, seed=0, epoch=0, num_threads=1,
                                       n_neg=10, lr=1e-3, mu=10.0, theta=0.5)
    assert S.tobytes() == z["S_e0"].tobytes()
    assert loss / len(ep_u) == z["mean_loss"][0]


def test_threaded_oracle_hogwild_runs():
    z = np.load(os.path.join(GOLDEN, "c1_epoch.npz"))
    S = init_matrix(1000, 32, InitSpec(seed=0)).values
    T = init_matrix(2000, 32, InitSpec(seed=0)).values
    ep_u, ep_i = O.epoch_pairs(z["offsets"], z["items"], 1000, O.shuffle_seed(0, 0))
    loss, _, _ = O.train_epoch_threads(S, T, ep_u, ep_i, seed=0, epoch=0, num_threads=4,
                                       chunk_pairs=512, n_neg=10, lr=1e-3, mu=10.0, theta=0.5)
    assert np.isfinite(loss) and np.isfinite(S).all() and np.isfinite(T).all()
    assert abs(loss / len(ep_u) - z["mean_loss"][0]) < 0.05 * abs(z["mean_loss"][0])


def _agg_cases():
    z = np.load(os.path.join(GOLDEN, "agg_cases.npz"))
    for name in z["names"]:
        g = {k.split("/", 1)[1]: z[k] for k in z.files if k.startswith(f"{name}/")}
        yield str(name), g, z["offsets"], z["items"]


def test_oracle_aggregator_bit_exact():
    """trainer.py:148-173 / 299-331 (SimpleX aggregation, per-thread
    accumulator flushed every mini_batch pairs, optional history gradient)."""
    for name, g, offsets, items in _agg_cases():
        S, T, W = g["S0"].copy(), g["T0"].copy(), g["W0"].copy()
        for e in range(int(g["epochs"])):
            u, i = O.epoch_pairs(offsets, items, 60, O.shuffle_seed(int(g["seed"]), e))
            ag = O.AggState(W, offsets, items, gamma=float(g["gamma"]), lr=float(g["agg_lr"]),
                            mini_batch=int(g["mb"]), max_history=int(g["max_history"]),
                            history_grad=bool(g["hist_prop"]))  # fresh per epoch (trainer.py:398)
            r = O.train_range(S, T, u, i, 0, len(u), O.derive_stream(int(g["seed"]), 0x45504F43, e, 0),
                              n_neg=int(g["N"]), lr=float(g["lr"]), l2=float(g["l2"]),
                              mu=float(g["mu"]), theta=float(g["theta"]), cosine=bool(g["cosine"]),
                              agg=ag)
            assert r.loss / len(u) == g["mean_loss"][e], name
        assert S.tobytes() == g["S"].tobytes(), name
        assert T.tobytes() == g["T"].tobytes(), name
        assert W.tobytes() == g["W"].tobytes(), name
