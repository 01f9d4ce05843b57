"""GPU parity: the CUDA path (through the C ABI) against the oracle and the
reference-generated golden vectors.

Bit-exact targets: negative ids (always), S/T/loss in EXACT mode.  Hogwild
mode is checked statistically (recall@20 / loss) like the reference's own
thread-count parity test (test_trainer.py:199-208).
"""

import hashlib
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    assert torch.cuda.is_available()
    from paper_2304_07334_b200 import _native
    _native.lib()
    return torch


def _dev_pairs(model, u, i):
    return model.upload_pairs(u, i)


def _neg_ids_device(torch_cuda, s0, first, npairs, n_neg, num_items):
    import ctypes
    from paper_2304_07334_b200 import _native as N
    out = torch_cuda.empty(npairs * n_neg, dtype=torch_cuda.int32, device="cuda")
    rc = N.lib().heat_sample_negatives(s0, first, npairs, n_neg, num_items,
                                       ctypes.c_void_p(out.data_ptr()), None)
    N.check(rc)
    return out.cpu().numpy().reshape(npairs, n_neg)


def _counter_draws_np(s0, first, npairs, n_neg, num_items):
    n = (np.arange(first * n_neg, (first + npairs) * n_neg, dtype=np.uint64) + np.uint64(1))
    with np.errstate(over="ignore"):
        z = np.uint64(s0) + n * np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return (z % np.uint64(num_items)).astype(np.int64).reshape(npairs, n_neg)


def test_sampler_matches_reference_stream(torch_cuda):
    from paper_2304_07334_b200.rng import epoch_stream
    z = np.load(os.path.join(GOLDEN, "c1_epoch.npz"))
    s0 = epoch_stream(0, 0)
    got = _neg_ids_device(torch_cuda, s0, 0, 64, 10, 2000)
    assert np.array_equal(got, z["negs_e0"])
    with open(os.path.join(GOLDEN, "rng.json")) as f:
        g = json.load(f)
    assert got.ravel()[:1000].tolist() == g["below2000_epoch0"][:640]


@pytest.mark.parametrize("num_items", [1, 2, 3, 2000, 92000, 2_000_000, 2**31 - 1, 1 << 30])
def test_sampler_fast_mod_exact(torch_cuda, num_items):
    s0 = 0x0123456789ABCDEF
    for first in (0, 123_456_789):
        got = _neg_ids_device(torch_cuda, s0, first, 4096, 37, num_items)
        want = _counter_draws_np(s0, first, 4096, 37, num_items)
        assert np.array_equal(got, want)


def _run_exact_steps(model, users, items, B, params, loss0=0.0):
    from paper_2304_07334_b200.device import DeviceCounters  # noqa: F401
    du, di = model.upload_pairs(users, items)
    model.counters.reset(loss0)
    n = len(users)
    losses = []
    for s in range(0, n, B):
        model.train_range(du, di, s, min(n, s + B), params)
        losses.append(model.counters.read().loss)
    return losses


def test_exact_c1_two_epochs_bit_exact(torch_cuda):
    from paper_2304_07334_b200 import _native as N
    from paper_2304_07334_b200.dataset import epoch_pairs
    from paper_2304_07334_b200.device import DeviceModel
    from paper_2304_07334_b200.embeddings import InitSpec, init_matrix
    from paper_2304_07334_b200.rng import epoch_stream, shuffle_seed
    from workloads import make_dataset
    z = np.load(os.path.join(GOLDEN, "c1_epoch.npz"))
    train, _, _ = make_dataset("c1")
    S = init_matrix(1000, 32, InitSpec(seed=0)).values
    T = init_matrix(2000, 32, InitSpec(seed=0)).values
    model = DeviceModel(S, T)
    for e in range(2):
        u, i = epoch_pairs(train, shuffle_seed(0, e))
        p = model.params(n_neg=10, lr=1e-3, l2=0.0, mu=10.0, theta=0.5, cosine=True,
                         mode=N.MODE_EXACT, stream_base=epoch_stream(0, e))
        losses = _run_exact_steps(model, u, i, 256, p)
        assert np.array_equal(np.array(losses), z[f"step_loss_e{e}"]), e
        model.download(S, T)
        assert S.tobytes() == z[f"S_e{e}"].tobytes()
        assert T.tobytes() == z[f"T_e{e}"].tobytes()
    c = model.counters.read()
    assert c.loss / len(u) == z["mean_loss"][1]


def test_exact_edge_cases_bit_exact(torch_cuda):
    from paper_2304_07334_b200 import _native as N
    from paper_2304_07334_b200.dataset import InteractionSet, epoch_pairs
    from paper_2304_07334_b200.device import DeviceModel
    from paper_2304_07334_b200.rng import epoch_stream, shuffle_seed
    z = np.load(os.path.join(GOLDEN, "edge_cases.npz"))
    for name in z["names"]:
        g = {k.split("/", 1)[1]: z[k] for k in z.files if k.startswith(f"{name}/")}
        S, T = g["S0"].copy(), g["T0"].copy()
        train = InteractionSet(int(g["nu"]), int(g["ni"]), g["offsets"], g["items"])
        model = DeviceModel(S, T)
        for e in range(int(g["epochs"])):
            u, i = epoch_pairs(train, shuffle_seed(int(g["seed"]), e))
            p = model.params(n_neg=int(g["N"]), lr=float(g["lr"]), l2=float(g["l2"]),
                             mu=float(g["mu"]), theta=float(g["theta"]), cosine=bool(g["cosine"]),
                             mode=N.MODE_EXACT, stream_base=epoch_stream(int(g["seed"]), e))
            losses = _run_exact_steps(model, u, i, 7, p)
            assert losses[-1] / len(u) == g["mean_loss"][e], name
        model.download(S, T)
        assert S.tobytes() == g["S"].tobytes(), name
        assert T.tobytes() == g["T"].tobytes(), name


def test_exact_c2_prefix_bit_exact(torch_cuda):
    from paper_2304_07334_b200 import _native as N
    from paper_2304_07334_b200.dataset import epoch_pairs
    from paper_2304_07334_b200.device import DeviceModel
    from paper_2304_07334_b200.embeddings import InitSpec, init_matrix
    from paper_2304_07334_b200.rng import epoch_stream, shuffle_seed
    from workloads import make_dataset
    with open(os.path.join(GOLDEN, "c2_prefix.json")) as f:
        g = json.load(f)
    train, _, _ = make_dataset("c2")
    S = init_matrix(train.num_users, 64, InitSpec(seed=0)).values
    T = init_matrix(train.num_items, 64, InitSpec(seed=0)).values
    u, i = epoch_pairs(train, shuffle_seed(0, 0))
    B, steps = g["B"], g["steps"]
    u, i = u[:B * steps], i[:B * steps]
    model = DeviceModel(S, T)
    du, di = model.upload_pairs(u, i)
    p = model.params(n_neg=100, lr=1e-3, l2=0.0, mu=150.0, theta=0.9, cosine=True,
                     mode=N.MODE_EXACT, stream_base=epoch_stream(0, 0))
    model.counters.reset()
    for s in range(steps):
        model.train_range(du, di, s * B, (s + 1) * B, p)
        c = model.counters.read()
        assert c.loss == g["loss"][s]
        assert c.degenerate == g["degen"][s]
        model.download(S, T)
        assert hashlib.sha256(S.tobytes()).hexdigest() == g["S_sha256"][s]
        assert hashlib.sha256(T.tobytes()).hexdigest() == g["T_sha256"][s]


@pytest.mark.parametrize("K,N,cos,l2,theta", [(1, 3, True, 0.0, -0.5), (3, 7, True, 0.05, 0.0),
                                              (8, 33, False, 0.01, 0.3), (33, 600, True, 0.0, 0.2),
                                              (130, 64, True, 0.02, -1.0), (64, 100, True, 0.0, 0.9)])
def test_exact_matches_oracle_random(torch_cuda, K, N, cos, l2, theta):
    from oracle import oracle as O
    from paper_2304_07334_b200 import _native as NN
    from paper_2304_07334_b200.device import DeviceModel
    rng = np.random.default_rng(K * 1000 + N)
    nu, ni, P = 50, 300, 2000
    S = (rng.standard_normal((nu, K)) * 0.1).astype(np.float32)
    T = (rng.standard_normal((ni, K)) * 0.1).astype(np.float32)
    S[3] = 0.0
    T[7] = 0.0
    u = rng.integers(0, nu, P).astype(np.int32)
    i = rng.integers(0, ni, P).astype(np.int32)
    s0 = 0xDEADBEEF12345678
    S2, T2 = S.copy(), T.copy()
    r = O.train_range(S2, T2, u, i, 0, P, s0, n_neg=N, lr=0.05, l2=l2, mu=2.0, theta=theta,
                      cosine=cos)
    model = DeviceModel(S, T)
    du, di = model.upload_pairs(u, i)
    p = model.params(n_neg=N, lr=0.05, l2=l2, mu=2.0, theta=theta, cosine=cos,
                     mode=NN.MODE_EXACT, stream_base=s0)
    model.counters.reset()
    model.train_range(du, di, 0, P, p)
    c = model.counters.read()
    model.download(S, T)
    assert S.tobytes() == S2.tobytes()
    assert T.tobytes() == T2.tobytes()
    assert c.loss == r.loss and c.degenerate == r.degenerate and c.active == r.active


def test_train_epoch_api_exact_equals_reference(torch_cuda):
    from paper_2304_07334_b200 import LossParams, TrainingConfig, init_matrix, InitSpec
    from workloads import make_dataset
    from paper_2304_07334_b200.trainer import train_epoch
    z = np.load(os.path.join(GOLDEN, "c1_epoch.npz"))
    train, _, _ = make_dataset("c1")
    cfg = TrainingConfig(emb_dim=32, num_negatives=10, learning_rate=1e-3, num_threads=1,
                         loss=LossParams(mu=10.0, theta=0.5), seed=0)
    S = init_matrix(1000, 32, InitSpec(seed=0))
    T = init_matrix(2000, 32, InitSpec(seed=0))
    for e in range(2):
        rep = train_epoch(S, T, train, cfg, epoch=e, collect_phases=True)
        assert rep.mean_loss == z["mean_loss"][e]
        assert rep.num_pairs == 20000 and rep.num_threads == 1
        assert rep.phase_times["read_emb"] > 0
        assert sum(rep.phase_times.values()) <= rep.wall_time
    assert S.values.tobytes() == z["S_e1"].tobytes()
    assert T.values.tobytes() == z["T_e1"].tobytes()


def test_hogwild_descends_and_matches_oracle_quality(torch_cuda):
    from oracle import oracle as O
    from paper_2304_07334_b200 import LossParams, TrainingConfig, init_matrix, InitSpec
    from paper_2304_07334_b200.evaluator import evaluate
    from workloads import make_clustered
    from paper_2304_07334_b200.trainer import configure, train_epoch
    from paper_2304_07334_b200.dataset import epoch_pairs
    from paper_2304_07334_b200.rng import shuffle_seed
    train, test = make_clustered(800, 1600, 16, 40, affinity=0.97, seed=11)
    cfg = TrainingConfig(emb_dim=32, num_negatives=16, learning_rate=0.05, num_threads=8,
                         loss=LossParams(mu=1.0, theta=0.8), seed=7)
    S = init_matrix(800, 32, InitSpec(seed=1))
    T = init_matrix(1600, 32, InitSpec(seed=2))
    So, To = S.values.copy(), T.values.copy()
    losses = []
    configure(mode="hogwild", window=256)
    try:
        for e in range(25):
            losses.append(train_epoch(S, T, train, cfg, epoch=e).mean_loss)
    finally:
        configure(mode=None, window=0)
    assert np.isfinite(losses).all() and losses[-1] < losses[0]
    m_gpu = evaluate(S, T, train, test, cfg, k=20)
    for e in range(25):
        u, i = epoch_pairs(train, shuffle_seed(7, e))
        O.train_range(So, To, u, i, 0, len(u), O.derive_stream(7, 0x45504F43, e, 0),
                      n_neg=16, lr=0.05, mu=1.0, theta=0.8)
    rec_ref, _, _ = O.evaluate_ref(So, To, train.offsets, train.items, 800, test.offsets,
                                   test.items, 800, k=20)
    assert abs(m_gpu.recall_at_k - rec_ref) <= 0.01, (m_gpu.recall_at_k, rec_ref)


def test_eval_matches_reference_golden(torch_cuda):
    from paper_2304_07334_b200.dataset import InteractionSet
    from paper_2304_07334_b200.device import DeviceModel
    from paper_2304_07334_b200.evaluator import eval_users_device, evaluate
    from paper_2304_07334_b200.embeddings import EmbeddingMatrix
    from paper_2304_07334_b200.config import TrainingConfig
    z = np.load(os.path.join(GOLDEN, "eval.npz"))
    c1 = np.load(os.path.join(GOLDEN, "c1_epoch.npz"))
    S, T = EmbeddingMatrix(c1["S_e1"]), EmbeddingMatrix(c1["T_e1"])
    tr = InteractionSet(1000, 2000, z["tr_offsets"], z["tr_items"])
    te = InteractionSet(1000, 2000, z["te_offsets"], z["te_items"])
    for sim in ("cosine", "dot"):
        cfg = TrainingConfig(emb_dim=32, num_negatives=1, similarity=sim)
        for k in (20, 5):
            m = evaluate(S, T, tr, te, cfg, k=k)
            want = z[f"{sim}_k{k}"]
            assert m.users_evaluated == int(want[2])
            assert m.recall_at_k == pytest.approx(want[0], abs=1e-12)
            assert m.ndcg_at_k == pytest.approx(want[1], abs=1e-12)
        model = DeviceModel(S.values, T.values)
        users = z[f"{sim}_top20_users"].astype(np.int32)
        _, _, top = eval_users_device(model.S, model.T, users, tr, te, 20, sim == "cosine",
                                      want_topk=True)
        assert np.array_equal(top, z[f"{sim}_top20"])


def test_eval_c2_init_matches_reference(torch_cuda):
    from paper_2304_07334_b200 import InitSpec, init_matrix, TrainingConfig
    from paper_2304_07334_b200.evaluator import evaluate
    from workloads import make_dataset
    z = np.load(os.path.join(GOLDEN, "eval.npz"))
    tr, te, _ = make_dataset("c2")
    S = init_matrix(tr.num_users, 64, InitSpec(seed=0))
    T = init_matrix(tr.num_items, 64, InitSpec(seed=0))
    m = evaluate(S, T, tr, te, TrainingConfig(emb_dim=64, num_negatives=1), k=20)
    want = z["c2_init_k20"]
    assert m.users_evaluated == int(want[2])
    assert abs(m.recall_at_k - want[0]) <= 1e-9
    assert abs(m.ndcg_at_k - want[1]) <= 1e-9


def test_topk_items_reference_cases(torch_cuda):
    from paper_2304_07334_b200.embeddings import EmbeddingMatrix
    from paper_2304_07334_b200.evaluator import topk_items
    from oracle.oracle import topk_ref
    T3 = EmbeddingMatrix(np.array([[1, 0], [0, 1], [-1, 0]], dtype=np.float32))
    assert list(topk_items(np.array([1.0, 0.0]), T3, [], 2)) == [0, 1]
    assert list(topk_items(np.array([1.0, 0.0]), T3, [0], 2)) == [1, 2]
    assert list(topk_items(np.array([1.0, 0.0]), T3, [0], 10)) == [1, 2]
    Tt = EmbeddingMatrix(np.array([[1, 0], [1, 0], [1, 0], [0.5, 0.5]], dtype=np.float32))
    assert list(topk_items(np.array([1.0, 0.0]), Tt, [], 3)) == [0, 1, 2]
    rng = np.random.default_rng(1234)
    for _ in range(10):
        T = EmbeddingMatrix(rng.standard_normal((200, 8)).astype(np.float32))
        u = rng.standard_normal(8)
        excl = np.unique(rng.integers(0, 200, size=30))
        for sim in ("cosine", "dot"):
            got = topk_items(u, T, excl, 10, sim)
            t64 = T.values.astype(np.float64)
            sc = (t64 @ u) / (np.linalg.norm(t64, axis=1) * np.linalg.norm(u)) \
                if sim == "cosine" else t64 @ u
            assert list(got) == list(topk_ref(sc, excl, 10))
    with pytest.raises(ValueError):
        topk_items(np.array([1.0, 0.0]), T3, [], 0)


def test_eval_random_vs_oracle_many_ks(torch_cuda):
    from oracle import oracle as O
    from paper_2304_07334_b200 import TrainingConfig
    from paper_2304_07334_b200.dataset import from_user_lists
    from paper_2304_07334_b200.embeddings import EmbeddingMatrix
    from paper_2304_07334_b200.evaluator import evaluate
    rng = np.random.default_rng(5)
    for trial in range(6):
        nu, ni, K = int(rng.integers(5, 200)), int(rng.integers(30, 700)), int(rng.integers(1, 70))
        S = EmbeddingMatrix(rng.standard_normal((nu, K)).astype(np.float32))
        T = EmbeddingMatrix(rng.standard_normal((ni, K)).astype(np.float32))
        if trial == 1:
            S.values[0] = 0.0
            T.values[:5] = 0.0
        tr = from_user_lists({u: rng.integers(0, ni, int(rng.integers(0, 40)))
                              for u in range(nu)}, num_users=nu, num_items=ni)
        te = from_user_lists({u: rng.integers(0, ni, int(rng.integers(0, 6)))
                              for u in range(0, nu, 2)}, num_users=nu, num_items=ni)
        for sim in ("cosine", "dot"):
            for k in (1, 7, 20, 33, 100):
                m = evaluate(S, T, tr, te, TrainingConfig(emb_dim=K, num_negatives=1,
                                                          similarity=sim), k=k)
                rec, nd, n = O.evaluate_ref(S.values, T.values, tr.offsets, tr.items, nu,
                                            te.offsets, te.items, nu, k=k, similarity=sim)
                assert m.users_evaluated == n
                assert m.recall_at_k == pytest.approx(rec, abs=1e-12), (trial, sim, k)
                assert m.ndcg_at_k == pytest.approx(nd, abs=1e-12), (trial, sim, k)


def _rel_fro(a, b):
    return float(np.linalg.norm(a.astype(np.float64) - b) / np.linalg.norm(b.astype(np.float64)))


@pytest.mark.parametrize("fp64", [False, True])
@pytest.mark.parametrize("force_generic", [False, True])
def test_hogwild_window1_tracks_reference(torch_cuda, fp64, force_generic, monkeypatch):
    """window=1 -> one worker, pairs in order: the throughput kernel's math
    (fp32 or fp64 partial dots, fused update) must track the reference
    within the north_star tolerance (1e-4, norm-relative) over a c1 epoch."""
    from paper_2304_07334_b200 import _native as N
    from paper_2304_07334_b200.dataset import epoch_pairs
    from paper_2304_07334_b200.device import DeviceModel
    from paper_2304_07334_b200.embeddings import InitSpec, init_matrix
    from paper_2304_07334_b200.rng import epoch_stream, shuffle_seed
    from workloads import make_dataset
    if force_generic:
        monkeypatch.setenv("HEAT_FORCE_GENERIC", "1")
    z = np.load(os.path.join(GOLDEN, "c1_epoch.npz"))
    train, _, _ = make_dataset("c1")
    S = init_matrix(1000, 32, InitSpec(seed=0)).values
    T = init_matrix(2000, 32, InitSpec(seed=0)).values
    model = DeviceModel(S, T)
    u, i = epoch_pairs(train, shuffle_seed(0, 0))
    du, di = model.upload_pairs(u, i)
    p = model.params(n_neg=10, lr=1e-3, l2=0.0, mu=10.0, theta=0.5, cosine=True,
                     mode=N.MODE_HOGWILD, stream_base=epoch_stream(0, 0), window=1, fp64=fp64)
    model.counters.reset()
    model.train_range(du, di, 0, len(u), p)
    c = model.counters.read()
    model.download(S, T)
    assert c.pairs == len(u)
    assert abs(c.loss / len(u) - z["mean_loss"][0]) <= 1e-4 * abs(z["mean_loss"][0])
    assert _rel_fro(S, z["S_e0"]) <= 1e-4, _rel_fro(S, z["S_e0"])
    assert _rel_fro(T, z["T_e0"]) <= 1e-4, _rel_fro(T, z["T_e0"])


@pytest.mark.parametrize("K,N,cos,l2,theta", [(16, 7, True, 0.0, -0.5), (32, 33, False, 0.01, 0.3),
                                              (64, 100, True, 0.02, 0.2), (128, 300, True, 0.0, 0.1),
                                              (64, 5, True, 0.0, -1.0), (48, 20, True, 0.01, 0.0)])
def test_hogwild_window1_vs_oracle(torch_cuda, K, N, cos, l2, theta):
    """Branch coverage of the throughput kernels (fast K in {16,32,64,128},
    generic otherwise): sequential run vs the oracle, 1e-4 norm-relative."""
    from oracle import oracle as O
    from paper_2304_07334_b200 import _native as NN
    from paper_2304_07334_b200.device import DeviceModel
    rng = np.random.default_rng(K + N)
    nu, ni, P = 40, 250, 600
    S = (rng.standard_normal((nu, K)) * 0.1).astype(np.float32)
    T = (rng.standard_normal((ni, K)) * 0.1).astype(np.float32)
    S[3] = 0.0
    T[7] = 0.0
    u = rng.integers(0, nu, P).astype(np.int32)
    i = rng.integers(0, ni, P).astype(np.int32)
    s0 = 0x1234567890ABCDEF
    S2, T2 = S.copy(), T.copy()
    r = O.train_range(S2, T2, u, i, 0, P, s0, n_neg=N, lr=0.01, l2=l2, mu=2.0, theta=theta,
                      cosine=cos)
    model = DeviceModel(S, T)
    du, di = model.upload_pairs(u, i)
    p = model.params(n_neg=N, lr=0.01, l2=l2, mu=2.0, theta=theta, cosine=cos,
                     mode=NN.MODE_HOGWILD, stream_base=s0, window=1, fp64=True)
    model.counters.reset()
    model.train_range(du, di, 0, P, p)
    c = model.counters.read()
    model.download(S, T)
    assert c.degenerate == r.degenerate
    assert abs(c.active - r.active) <= max(2, r.active // 1000)
    assert abs(c.loss - r.loss) <= 1e-4 * abs(r.loss)
    assert _rel_fro(S, S2) <= 1e-4 and _rel_fro(T, T2) <= 1e-4


@pytest.mark.parametrize("G", [1, 2, 4])
def test_logical_shards_keep_item_replicas_identical(torch_cuda, G):
    """G logical ranks on one GPU through the sharded step
    code with a loopback exchange (concatenation in rank order = what the
    NCCL all-gather returns).  Item replicas must stay bit-identical, every
    pair is trained exactly once, and training tracks the 1-GPU run."""
    import torch
    from paper_2304_07334_b200 import _native as N
    from paper_2304_07334_b200.dataset import epoch_pairs
    from paper_2304_07334_b200.device import DeviceModel
    from paper_2304_07334_b200.embeddings import InitSpec, init_matrix
    from paper_2304_07334_b200.parallel import ShardedTrainer
    from paper_2304_07334_b200.rng import epoch_stream, shuffle_seed
    from workloads import make_dataset
    train, _, _ = make_dataset("c2", scale=0.05)
    S = init_matrix(train.num_users, 64, InitSpec(seed=0)).values
    T = init_matrix(train.num_items, 64, InitSpec(seed=0)).values
    ranks = [ShardedTrainer(DeviceModel(S, T), G, r) for r in range(G)]
    losses = []
    for e in range(2):
        u, i = epoch_pairs(train, shuffle_seed(0, e))
        for tr in ranks:
            p = tr.model.params(n_neg=100, lr=1e-3, l2=0.0, mu=150.0, theta=0.9, cosine=True,
                                mode=N.MODE_DELTA, stream_base=epoch_stream(0, e), window=256)
            tr.model.counters.reset()
            tr.prepare_epoch(u, i, p, 1024)
        for s in range(ranks[0].num_steps):
            logs = [tr.local_step(s) for tr in ranks]
            cmax = max(c for _, _, c in logs)
            if cmax == 0:
                continue
            all_ids = torch.cat([ids[:cmax] for ids, _, _ in logs])
            all_rows = torch.cat([rows[:cmax] for _, rows, _ in logs])
            valid = torch.cat([torch.arange(cmax, device="cuda") < c for _, _, c in logs])
            for tr in ranks:
                tr.apply_ordered(all_ids, all_rows, valid)
        cs = [tr.model.counters.read() for tr in ranks]
        assert sum(c.pairs for c in cs) == len(u)
        losses.append(sum(c.loss for c in cs) / len(u))
        T0 = ranks[0].model.T.cpu().numpy()
        for tr in ranks[1:]:
            assert tr.model.T.cpu().numpy().tobytes() == T0.tobytes()
    # user rows: each owned by exactly one rank
    Sg = np.zeros_like(S)
    for r, tr in enumerate(ranks):
        own = np.arange(train.num_users) % G == r
        Sg[own] = tr.model.S.cpu().numpy()[own]
    assert np.isfinite(Sg).all() and losses[1] < losses[0]
    # same workload through the 1-GPU hogwild path: loss within 2 %
    m = DeviceModel(init_matrix(train.num_users, 64, InitSpec(seed=0)).values,
                    init_matrix(train.num_items, 64, InitSpec(seed=0)).values)
    ref = []
    for e in range(2):
        u, i = epoch_pairs(train, shuffle_seed(0, e))
        du, di = m.upload_pairs(u, i)
        p = m.params(n_neg=100, lr=1e-3, l2=0.0, mu=150.0, theta=0.9, cosine=True,
                     mode=N.MODE_HOGWILD, stream_base=epoch_stream(0, e), window=256)
        m.counters.reset()
        m.train_range(du, di, 0, len(u), p)
        ref.append(m.counters.read().loss / len(u))
    assert abs(losses[1] - ref[1]) <= 0.02 * abs(ref[1]), (losses, ref)


def _agg_golden():
    z = np.load(os.path.join(GOLDEN, "agg_cases.npz"))
    for name in z["names"]:
        g = {k.split("/", 1)[1]: z[k] for k in z.files if k.startswith(f"{name}/")}
        yield str(name), g, z["offsets"], z["items"]


def test_exact_aggregator_bit_exact(torch_cuda):
    """SimpleX aggregation in EXACT mode == reference train_epoch(num_threads=1)
    with the aggregator on: S, T, W and mean loss bit for bit
    (trainer.py:148-173, 299-331)."""
    from paper_2304_07334_b200 import _native as N
    from paper_2304_07334_b200.config import AggregatorConfig
    from paper_2304_07334_b200.dataset import InteractionSet, epoch_pairs
    from paper_2304_07334_b200.device import DeviceAggregator, DeviceModel
    from paper_2304_07334_b200.rng import epoch_stream, shuffle_seed
    for name, g, offsets, items in _agg_golden():
        train = InteractionSet(60, 240, offsets, items)
        S, T = g["S0"].copy(), g["T0"].copy()
        model = DeviceModel(S, T)
        cfg_agg = AggregatorConfig(enabled=True, gamma=float(g["gamma"]),
                                   max_history=int(g["max_history"]),
                                   mini_batch_size=int(g["mb"]),
                                   history_grad=bool(g["hist_prop"]),
                                   learning_rate=float(g["agg_lr"]))
        agg = DeviceAggregator(g["W0"].copy(), train, cfg_agg, float(g["lr"]), model.device)
        for e in range(int(g["epochs"])):
            u, i = epoch_pairs(train, shuffle_seed(int(g["seed"]), e))
            du, di = model.upload_pairs(u, i)
            p = model.params(n_neg=int(g["N"]), lr=float(g["lr"]), l2=float(g["l2"]),
                             mu=float(g["mu"]), theta=float(g["theta"]), cosine=bool(g["cosine"]),
                             mode=N.MODE_EXACT, stream_base=epoch_stream(int(g["seed"]), e))
            model.counters.reset()
            agg.reset_epoch()
            for s in range(0, len(u), 37):  # arbitrary step split: state carried
                model.train_range(du, di, s, min(len(u), s + 37), p, agg=agg)
            c = model.counters.read()
            assert c.loss / len(u) == g["mean_loss"][e], name
        model.download(S, T)
        assert S.tobytes() == g["S"].tobytes(), name
        assert T.tobytes() == g["T"].tobytes(), name
        assert agg.W.cpu().numpy().tobytes() == g["W"].tobytes(), name


def test_train_epoch_api_with_aggregator(torch_cuda):
    from paper_2304_07334_b200 import LossParams, TrainingConfig
    from paper_2304_07334_b200.config import AggregatorConfig
    from paper_2304_07334_b200.dataset import InteractionSet
    from paper_2304_07334_b200.embeddings import EmbeddingMatrix
    from paper_2304_07334_b200.trainer import train_epoch
    name, g, offsets, items = next(_agg_golden())  # "basic"
    train = InteractionSet(60, 240, offsets, items)
    cfg = TrainingConfig(emb_dim=int(g["K"]), num_negatives=int(g["N"]), learning_rate=float(g["lr"]),
                         num_threads=1, loss=LossParams(mu=float(g["mu"]), theta=float(g["theta"])),
                         seed=int(g["seed"]),
                         aggregator=AggregatorConfig(enabled=True, gamma=float(g["gamma"]),
                                                     max_history=int(g["max_history"]),
                                                     mini_batch_size=int(g["mb"])))
    S, T, W = EmbeddingMatrix(g["S0"].copy()), EmbeddingMatrix(g["T0"].copy()), g["W0"].copy()
    for e in range(int(g["epochs"])):
        rep = train_epoch(S, T, train, cfg, W, epoch=e)
        assert rep.mean_loss == g["mean_loss"][e]
    assert S.values.tobytes() == g["S"].tobytes()
    assert T.values.tobytes() == g["T"].tobytes()
    assert W.tobytes() == g["W"].tobytes()  # updated in place, like the reference


def test_aggregated_evaluation_query(torch_cuda):
    """evaluator.py:91-110 + 113-179 with cfg.aggregator enabled."""
    from oracle import oracle as O
    from paper_2304_07334_b200 import TrainingConfig
    from paper_2304_07334_b200.config import AggregatorConfig
    from paper_2304_07334_b200.dataset import from_user_lists
    from paper_2304_07334_b200.embeddings import EmbeddingMatrix
    from paper_2304_07334_b200.evaluator import evaluate
    rng = np.random.default_rng(8)
    nu, ni, K = 40, 300, 16
    S = EmbeddingMatrix(rng.standard_normal((nu, K)).astype(np.float32))
    T = EmbeddingMatrix(rng.standard_normal((ni, K)).astype(np.float32))
    W = rng.standard_normal((K, K)).astype(np.float32)
    tr = from_user_lists({u: rng.integers(0, ni, int(rng.integers(0, 25))) for u in range(nu)},
                         num_users=nu, num_items=ni)
    te = from_user_lists({u: rng.integers(0, ni, 3) for u in range(nu)}, num_users=nu,
                         num_items=ni)
    for gamma, mh in ((0.0, 100), (0.4, 5), (1.0, 10)):
        cfg = TrainingConfig(emb_dim=K, num_negatives=1,
                             aggregator=AggregatorConfig(enabled=True, gamma=gamma,
                                                         max_history=mh))
        m = evaluate(S, T, tr, te, cfg, weights=W, k=10)
        pooled = np.zeros((nu, K))
        for u in range(nu):
            h = tr.slice(u)[:mh]
            if len(h):
                pooled[u] = T.values[h].astype(np.float64).mean(axis=0)
        q = gamma * S.values.astype(np.float64) + (1 - gamma) * (pooled @ W.astype(np.float64))
        rec, nd, n = O.evaluate_ref(q, T.values, tr.offsets, tr.items, nu, te.offsets, te.items,
                                    nu, k=10)
        assert m.users_evaluated == n
        assert m.recall_at_k == pytest.approx(rec, abs=1e-12)
        assert m.ndcg_at_k == pytest.approx(nd, abs=1e-12)


def _agg_case(rng, nu, ni, K):
    from paper_2304_07334_b200.dataset import from_user_lists
    tr = from_user_lists({u: rng.integers(0, ni, int(rng.integers(0, 30))) for u in range(nu)},
                         num_users=nu, num_items=ni)
    S = (rng.standard_normal((nu, K)) * 0.1).astype(np.float32)
    T = (rng.standard_normal((ni, K)) * 0.1).astype(np.float32)
    W = (rng.standard_normal((K, K)) / np.sqrt(K)).astype(np.float32)
    return tr, S, T, W


@pytest.mark.parametrize("K,N,gamma,hist,l2,cos,mh", [
    (16, 7, 0.5, False, 0.0, True, 100), (32, 20, 0.3, True, 0.01, True, 10),
    (64, 50, 0.0, True, 0.0, False, 100), (128, 64, 1.0, False, 0.0, True, 100),
    (128, 40, 0.2, True, 0.0, True, 5)])
def test_agg_hogwild_window1_vs_oracle(torch_cuda, K, N, gamma, hist, l2, cos, mh):
    """Throughput aggregator (csrc/heat_agg_hogwild.cu) with one pair per step
    and mini_batch 1: the reference flushes W after every pair too, so the
    sequence of reads and writes is the reference's (trainer.py:148-173,
    299-331); fp32 arithmetic tracks it within 1e-4 norm-relative."""
    from oracle import oracle as O
    from paper_2304_07334_b200 import _native as NN
    from paper_2304_07334_b200.config import AggregatorConfig
    from paper_2304_07334_b200.device import DeviceAggregator, DeviceModel
    rng = np.random.default_rng(K * 7 + N)
    nu, ni, P = 40, 250, 500
    tr, S, T, W = _agg_case(rng, nu, ni, K)
    u = rng.integers(0, nu, P).astype(np.int32)
    i = rng.integers(0, ni, P).astype(np.int32)
    s0 = 0x0DDC0FFEE0DDF00D
    S2, T2, W2 = S.copy(), T.copy(), W.copy()
    st = O.AggState(W=W2, tr_offsets=tr.offsets, tr_items=tr.items, gamma=gamma, lr=0.02,
                    mini_batch=1, max_history=mh, history_grad=hist)
    r = O.train_range(S2, T2, u, i, 0, P, s0, n_neg=N, lr=0.01, l2=l2, mu=2.0, theta=0.1,
                      cosine=cos, agg=st)
    model = DeviceModel(S, T)
    cfg_agg = AggregatorConfig(enabled=True, gamma=gamma, max_history=mh, mini_batch_size=1,
                               history_grad=hist, learning_rate=0.02)
    agg = DeviceAggregator(W.copy(), tr, cfg_agg, 0.01, model.device)
    du, di = model.upload_pairs(u, i)
    p = model.params(n_neg=N, lr=0.01, l2=l2, mu=2.0, theta=0.1, cosine=cos,
                     mode=NN.MODE_HOGWILD, stream_base=s0, window=1)
    model.counters.reset()
    model.train_range(du, di, 0, P, p, agg=agg)
    c = model.counters.read()
    model.download(S, T)
    Wg = agg.W.cpu().numpy()
    assert c.pairs == P
    assert abs(c.loss - r.loss) <= 1e-4 * abs(r.loss), (c.loss, r.loss)
    assert _rel_fro(S, S2) <= 1e-4, _rel_fro(S, S2)
    assert _rel_fro(T, T2) <= 1e-4, _rel_fro(T, T2)
    assert _rel_fro(Wg, W2) <= 1e-4, _rel_fro(Wg, W2)


def test_agg_hogwild_quality_matches_oracle(torch_cuda):
    """Throughput aggregator under concurrency (256-pair steps, W frozen per
    step): training descends and the aggregated-query recall@20 after 20
    epochs matches the oracle's single-thread run within 0.01, the
    reference's own thread-parity bound (test_trainer.py:199-208)."""
    from oracle import oracle as O
    from paper_2304_07334_b200 import LossParams, TrainingConfig, init_matrix, InitSpec
    from paper_2304_07334_b200.config import AggregatorConfig
    from paper_2304_07334_b200.dataset import epoch_pairs
    from paper_2304_07334_b200.evaluator import evaluate
    from paper_2304_07334_b200.rng import shuffle_seed
    from workloads import make_clustered
    from paper_2304_07334_b200.trainer import configure, train_epoch
    train, test = make_clustered(800, 1600, 16, 40, affinity=0.97, seed=11)
    K, E = 32, 20
    acfg = AggregatorConfig(enabled=True, gamma=0.5, max_history=20, mini_batch_size=32)
    cfg = TrainingConfig(emb_dim=K, num_negatives=16, learning_rate=0.05, num_threads=8,
                         loss=LossParams(mu=1.0, theta=0.8), seed=7, aggregator=acfg)
    S = init_matrix(800, K, InitSpec(seed=1))
    T = init_matrix(1600, K, InitSpec(seed=2))
    W = np.eye(K, dtype=np.float32)
    So, To, Wo = S.values.copy(), T.values.copy(), W.copy()
    losses = []
    configure(mode="hogwild", window=256)
    try:
        for e in range(E):
            losses.append(train_epoch(S, T, train, cfg, W, epoch=e).mean_loss)
    finally:
        configure(mode=None, window=0)
    assert np.isfinite(losses).all() and losses[-1] < losses[0], losses
    m_gpu = evaluate(S, T, train, test, cfg, weights=W, k=20)
    for e in range(E):
        u, i = epoch_pairs(train, shuffle_seed(7, e))
        st = O.AggState(W=Wo, tr_offsets=train.offsets, tr_items=train.items, gamma=0.5,
                        lr=0.05, mini_batch=32, max_history=20)
        O.train_range(So, To, u, i, 0, len(u), O.derive_stream(7, 0x45504F43, e, 0),
                      n_neg=16, lr=0.05, mu=1.0, theta=0.8, agg=st)
    pooled = np.zeros((800, K))
    for uu in range(800):
        h = train.slice(uu)[:20]
        if len(h):
            pooled[uu] = To[h].astype(np.float64).mean(axis=0)
    q = 0.5 * So.astype(np.float64) + 0.5 * (pooled @ Wo.astype(np.float64))
    rec_ref, _, _ = O.evaluate_ref(q, To, train.offsets, train.items, 800, test.offsets,
                                   test.items, 800, k=20)
    assert abs(m_gpu.recall_at_k - rec_ref) <= 0.01, (m_gpu.recall_at_k, rec_ref)


def test_fixed_point_apply_is_order_independent(torch_cuda):
    """heat_apply_row_deltas_fixed: the same gathered logs in any entry order
    give bit-identical rows (integer accumulation), equal to the exact sum
    within fp32 rounding; padding past each rank's count is ignored."""
    import ctypes
    import torch
    from paper_2304_07334_b200 import _native as N
    rng = np.random.default_rng(5)
    rows_t, K, world, stride = 50, 64, 3, 400
    counts = np.array([400, 123, 0], dtype=np.int64)
    ids = rng.integers(0, rows_t, world * stride).astype(np.int32)
    vals = (rng.standard_normal((world * stride, K)) * 1e-3).astype(np.float32)
    T0 = rng.standard_normal((rows_t, K)).astype(np.float32)
    valid = (np.arange(world * stride) % stride) < np.repeat(counts, stride)

    def apply(perm_within_rank):
        ii, vv = ids.copy(), vals.copy()
        for r in range(world):
            sl = slice(r * stride, r * stride + counts[r])
            p = perm_within_rank[r]
            ii[sl], vv[sl] = ii[sl][p], vv[sl][p]
        T = torch.from_numpy(T0.copy()).cuda()
        acc = torch.zeros(rows_t * K, dtype=torch.int64, device="cuda")
        flags = torch.zeros(rows_t, dtype=torch.int32, device="cuda")
        dc = torch.from_numpy(counts).cuda()
        di, dv = torch.from_numpy(ii).cuda(), torch.from_numpy(vv).cuda()
        P = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
        N.check(N.lib().heat_apply_row_deltas_fixed(P(T), rows_t, K, P(di), P(dv), P(dc), world,
                                                    stride, P(acc), P(flags), None))
        torch.cuda.synchronize()
        assert int(acc.abs().sum()) == 0 and int(flags.sum()) == 0  # left zero
        return T.cpu().numpy()

    a = apply([np.arange(c) for c in counts])
    b = apply([rng.permutation(c) for c in counts])
    assert a.tobytes() == b.tobytes()
    want = T0.astype(np.float64)
    np.add.at(want, ids[valid], vals[valid].astype(np.float64))
    assert np.abs(a - want).max() <= 1e-6


@pytest.mark.parametrize("G", [1, 2, 4])
def test_pipelined_shards_keep_replicas_identical(torch_cuda, G):
    """The pipelined multi-GPU step (exchange of step s overlapped with the
    kernel of step s+1, order-independent apply) driven for G logical ranks
    on one GPU: item replicas bit-identical, every pair trained once, loss
    within 3 % of the 1-GPU Hogwild run at the same staleness bound (two
    1024-pair steps of item updates in flight -> window 2048)."""
    from paper_2304_07334_b200 import _native as N
    from paper_2304_07334_b200.dataset import epoch_pairs
    from paper_2304_07334_b200.device import DeviceModel
    from paper_2304_07334_b200.embeddings import InitSpec, init_matrix
    from paper_2304_07334_b200.parallel import PipelinedShardTrainer, run_loopback
    from paper_2304_07334_b200.rng import epoch_stream, shuffle_seed
    from workloads import make_dataset
    train, _, _ = make_dataset("c2", scale=0.05)
    S = init_matrix(train.num_users, 64, InitSpec(seed=0)).values
    T = init_matrix(train.num_items, 64, InitSpec(seed=0)).values
    ranks = [PipelinedShardTrainer(DeviceModel(S, T), G, r) for r in range(G)]
    losses = []
    for e in range(2):
        u, i = epoch_pairs(train, shuffle_seed(0, e))
        gens = []
        for tr in ranks:
            p = tr.model.params(n_neg=100, lr=1e-3, l2=0.0, mu=150.0, theta=0.9, cosine=True,
                                mode=N.MODE_DELTA, stream_base=epoch_stream(0, e), window=256)
            tr.model.counters.reset()
            gens.append(tr.epoch_pipeline(u, i, p, 1024))
        if G == 1:
            for req in gens[0]:
                ranks[0].coll.run(req)
        else:
            run_loopback(gens)
        cs = [tr.model.counters.read() for tr in ranks]
        assert sum(c.pairs for c in cs) == len(u)
        assert sum(st.entries for st in ranks[0].stats) >= len(u)  # >= one row per pair
        losses.append(sum(c.loss for c in cs) / len(u))
        T0 = ranks[0].model.T.cpu().numpy()
        for tr in ranks[1:]:
            assert tr.model.T.cpu().numpy().tobytes() == T0.tobytes()
    assert losses[1] < losses[0]
    m = DeviceModel(init_matrix(train.num_users, 64, InitSpec(seed=0)).values,
                    init_matrix(train.num_items, 64, InitSpec(seed=0)).values)
    ref = []
    for e in range(2):
        u, i = epoch_pairs(train, shuffle_seed(0, e))
        du, di = m.upload_pairs(u, i)
        p = m.params(n_neg=100, lr=1e-3, l2=0.0, mu=150.0, theta=0.9, cosine=True,
                     mode=N.MODE_HOGWILD, stream_base=epoch_stream(0, e), window=2048)
        m.counters.reset()
        m.train_range(du, di, 0, len(u), p)
        ref.append(m.counters.read().loss / len(u))
    assert abs(losses[1] - ref[1]) <= 0.03 * abs(ref[1]), (losses, ref)


def test_native_shard_runtime_world1(torch_cuda):
    """csrc/heat_shard.cu (the production scheduler) at world 1: every pair
    trained once per epoch, one exchange per step, training tracks the 1-GPU
    Hogwild run at the same staleness bound (loss within 3 %)."""
    from paper_2304_07334_b200 import _native as N
    from paper_2304_07334_b200.dataset import epoch_pairs
    from paper_2304_07334_b200.device import DeviceModel
    from paper_2304_07334_b200.embeddings import InitSpec, init_matrix
    from paper_2304_07334_b200.parallel import NativeShardTrainer
    from paper_2304_07334_b200.rng import epoch_stream, shuffle_seed
    from workloads import make_dataset
    train, _, _ = make_dataset("c2", scale=0.05)
    mk = lambda: DeviceModel(init_matrix(train.num_users, 64, InitSpec(seed=0)).values,  # noqa: E731
                             init_matrix(train.num_items, 64, InitSpec(seed=0)).values)
    tr = NativeShardTrainer(mk(), 1, 0)
    m = mk()
    losses, ref = [], []
    for e in range(2):
        u, i = epoch_pairs(train, shuffle_seed(0, e))
        p = tr.model.params(n_neg=100, lr=1e-3, l2=0.0, mu=150.0, theta=0.9, cosine=True,
                            mode=N.MODE_DELTA, stream_base=epoch_stream(0, e), window=256)
        tr.model.counters.reset()
        st = tr.train_epoch(u, i, p, 1024)
        c = tr.model.counters.read()
        assert c.pairs == len(u) and st.steps == tr.num_steps
        assert st.entries >= len(u)
        losses.append(c.loss / len(u))
        du, di = m.upload_pairs(u, i)
        p = m.params(n_neg=100, lr=1e-3, l2=0.0, mu=150.0, theta=0.9, cosine=True,
                     mode=N.MODE_HOGWILD, stream_base=epoch_stream(0, e), window=2048)
        m.counters.reset()
        m.train_range(du, di, 0, len(u), p)
        ref.append(m.counters.read().loss / len(u))
    assert np.isfinite(tr.model.T.cpu().numpy()).all()
    assert abs(losses[1] - ref[1]) <= 0.03 * abs(ref[1]), (losses, ref)
    with pytest.raises(ValueError):  # EXACT/HOGWILD params are rejected: DELTA steps only
        p.mode = N.MODE_HOGWILD
        tr.params = p
        tr.train_epoch(u, i, p, 1024, prepared=True)
    tr.close()


@pytest.mark.parametrize("lag,graph,exchange", [("1", "1", "p2p"), ("3", "1", "p2p"),
                                                ("2", "0", "p2p"), ("2", "0", "gather")])
def test_native_shard_runtime_lag(torch_cuda, monkeypatch, lag, graph, exchange):
    """The native runtime with other staleness bounds (HEAT_SHARD_LAG: kernel(s)
    waits for the apply of step s - lag; lag + 1 log slots in rotation, two
    compute streams), with and without captured step graphs, and through the
    gather fallback: every pair trained once per epoch, every step exchanged,
    loss within 3 % of the 1-GPU Hogwild run."""
    from paper_2304_07334_b200 import _native as N
    from paper_2304_07334_b200.dataset import epoch_pairs
    from paper_2304_07334_b200.device import DeviceModel
    from paper_2304_07334_b200.embeddings import InitSpec, init_matrix
    from paper_2304_07334_b200.parallel import NativeShardTrainer
    from paper_2304_07334_b200.rng import epoch_stream, shuffle_seed
    from workloads import make_dataset
    monkeypatch.setenv("HEAT_SHARD_LAG", lag)
    monkeypatch.setenv("HEAT_SHARD_GRAPH", graph)  # captured step graphs / direct launches
    # gather: the fallback exchange (counts read on the host each step, the
    # log as its own gathered copy at world 1)
    monkeypatch.setenv("HEAT_SHARD_EXCHANGE", exchange)
    train, _, _ = make_dataset("c2", scale=0.05)
    mk = lambda: DeviceModel(init_matrix(train.num_users, 64, InitSpec(seed=0)).values,  # noqa: E731
                             init_matrix(train.num_items, 64, InitSpec(seed=0)).values)
    tr = NativeShardTrainer(mk(), 1, 0)
    m = mk()
    for e in range(3):  # epoch 0 launches step by step and captures; 1, 2 replay the graph
        u, i = epoch_pairs(train, shuffle_seed(0, e))
        p = tr.model.params(n_neg=100, lr=1e-3, l2=0.0, mu=150.0, theta=0.9, cosine=True,
                            mode=N.MODE_DELTA, stream_base=epoch_stream(0, e), window=512)
        tr.model.counters.reset()
        st = tr.train_epoch(u, i, p, 512)
        c = tr.model.counters.read()
        assert c.pairs == len(u) and st.steps == tr.num_steps and st.entries >= len(u)
        du, di = m.upload_pairs(u, i)
        p = m.params(n_neg=100, lr=1e-3, l2=0.0, mu=150.0, theta=0.9, cosine=True,
                     mode=N.MODE_HOGWILD, stream_base=epoch_stream(0, e), window=2048)
        m.counters.reset()
        m.train_range(du, di, 0, len(u), p)
    assert np.isfinite(tr.model.T.cpu().numpy()).all()
    ref = m.counters.read().loss
    assert abs(c.loss - ref) <= 0.03 * abs(ref), (c.loss, ref)
    tr.close()


def test_shard_graph_replay_equals_direct_launches(torch_cuda, monkeypatch):
    """The captured step graph (device-side step ranges and stream base,
    replayed from the second epoch of a shape on) trains the same pairs with
    the same negatives as step-by-step launches.  With one worker and lag 1
    the steps run strictly in order, so both runs agree up to the order of
    the per-warp user-gradient additions (fp32 rounding, ~1e-5 relative after
    five epochs); a wrong stream base changes the tables far more (the
    negative control below).  A changed shape (learning rate) recaptures."""
    from paper_2304_07334_b200 import _native as N
    from paper_2304_07334_b200.dataset import epoch_pairs
    from paper_2304_07334_b200.device import DeviceModel
    from paper_2304_07334_b200.embeddings import InitSpec, init_matrix
    from paper_2304_07334_b200.parallel import NativeShardTrainer
    from paper_2304_07334_b200.rng import epoch_stream, shuffle_seed
    from workloads import make_dataset
    train, _, _ = make_dataset("c2", scale=0.02)
    monkeypatch.setenv("HEAT_SHARD_LAG", "1")
    out = {}
    for graph in ("1", "0", "stale"):
        monkeypatch.setenv("HEAT_SHARD_GRAPH", "0" if graph == "stale" else graph)
        m = DeviceModel(init_matrix(train.num_users, 64, InitSpec(seed=0)).values,
                        init_matrix(train.num_items, 64, InitSpec(seed=0)).values)
        tr = NativeShardTrainer(m, 1, 0)
        for e, lr in ((0, 1e-2), (1, 1e-2), (2, 1e-2), (3, 5e-3), (4, 5e-3)):
            u, i = epoch_pairs(train, shuffle_seed(0, e))
            s0 = epoch_stream(0, 0 if graph == "stale" else e)  # stale: epoch 0's negatives
            p = m.params(n_neg=100, lr=lr, l2=0.0, mu=150.0, theta=0.9, cosine=True,
                         mode=N.MODE_DELTA, stream_base=s0, window=1)
            m.counters.reset()
            st = tr.train_epoch(u, i, p, 256)
            assert m.counters.read().pairs == len(u) and st.steps == tr.num_steps
        out[graph] = (m.S.cpu().numpy().astype(np.float64), m.T.cpu().numpy().astype(np.float64))
        tr.close()
    rel = lambda x, y: np.linalg.norm(x - y) / np.linalg.norm(y)  # noqa: E731
    for a, b, c in zip(out["1"], out["0"], out["stale"]):
        assert rel(a, b) <= 1e-4, rel(a, b)
        assert rel(c, b) > 20 * max(rel(a, b), 1e-6), (rel(c, b), rel(a, b))


@pytest.mark.parametrize("cfg", ["c4", "c5"])
def test_full_size_sharded_properties(torch_cuda, cfg):
    """The multi-GPU step code (native runtime, world 1) at BASELINE.json's
    full c4 / c5 table sizes with the config's B per step: every pair
    trained once per epoch, one exchange per step, the loss finite and
    falling, the tables finite."""
    import torch
    from paper_2304_07334_b200 import _native as N
    from paper_2304_07334_b200.dataset import epoch_pairs
    from paper_2304_07334_b200.device import DeviceModel
    from paper_2304_07334_b200.embeddings import InitSpec, init_matrix
    from paper_2304_07334_b200.parallel import NativeShardTrainer
    from paper_2304_07334_b200.rng import epoch_stream, shuffle_seed
    from workloads import make_dataset
    kw = {"sample_users": 0.02} if cfg == "c5" else {}
    tr, _, sp = make_dataset(cfg, **kw)
    m = DeviceModel(init_matrix(tr.num_users, sp.dim, InitSpec(seed=0)).values,
                    init_matrix(tr.num_items, sp.dim, InitSpec(seed=0)).values)
    sh = NativeShardTrainer(m, 1, 0)
    losses = []
    for e in range(2):
        u, i = epoch_pairs(tr, shuffle_seed(0, e))
        p = m.params(n_neg=sp.negatives, lr=sp.learning_rate, l2=0.0, mu=sp.mu, theta=sp.theta,
                     cosine=True, mode=N.MODE_DELTA, stream_base=epoch_stream(0, e),
                     window=sp.batch)
        m.counters.reset()
        st = sh.train_epoch(u, i, p, sp.batch)
        c = m.counters.read()
        assert c.pairs == tr.num_pairs and st.steps == sh.num_steps and np.isfinite(c.loss)
        losses.append(c.loss / c.pairs)
    sh.close()
    assert losses[1] < losses[0]
    assert bool(torch.isfinite(m.S).all()) and bool(torch.isfinite(m.T).all())


def test_train_device_resident_run_with_checkpoints(torch_cuda, tmp_path):
    """train() (trainer.py:480-533): tables stay on the device across epochs,
    yet the run equals the reference's epoch-by-epoch result bit for bit;
    evaluations at every interval plus the final one; best/final checkpoints
    in the HEATEMB1 bundle format hold the reported tables."""
    import dataclasses
    from oracle import oracle as O
    from paper_2304_07334_b200 import LossParams, TrainingConfig, init_matrix, InitSpec
    from paper_2304_07334_b200.dataset import from_user_lists
    from paper_2304_07334_b200.embeddings import load_model
    from workloads import make_dataset
    from paper_2304_07334_b200.trainer import train
    z = np.load(os.path.join(GOLDEN, "c1_epoch.npz"))
    tr, _, _ = make_dataset("c1")
    rng = np.random.default_rng(3)
    te = from_user_lists({u: rng.integers(0, 2000, 3) for u in range(0, 1000, 3)},
                         num_users=1000, num_items=2000)
    cfg = TrainingConfig(emb_dim=32, num_negatives=10, learning_rate=1e-3, num_threads=1,
                         loss=LossParams(mu=10.0, theta=0.5), seed=0)
    cfg = dataclasses.replace(cfg, epochs=2)
    S = init_matrix(1000, 32, InitSpec(seed=0))
    T = init_matrix(2000, 32, InitSpec(seed=0))
    seen = []
    res = train(S, T, tr, te, cfg, eval_interval=1, k=20, out_dir=str(tmp_path),
                on_epoch=lambda r: seen.append(r.epoch))
    assert seen == [0, 1]
    assert [r.mean_loss for r in res.reports] == list(z["mean_loss"][:2])
    assert S.values.tobytes() == z["S_e1"].tobytes()
    assert T.values.tobytes() == z["T_e1"].tobytes()
    assert [e for e, _ in res.evaluations] == [1, 2, 2]
    rec, nd, n = O.evaluate_ref(S.values, T.values, tr.offsets, tr.items, 1000, te.offsets,
                                te.items, 1000, k=20)
    assert res.final_metrics.recall_at_k == pytest.approx(rec, abs=1e-12)
    assert res.final_metrics.ndcg_at_k == pytest.approx(nd, abs=1e-12)
    assert res.best_recall == max(m.recall_at_k for _, m in res.evaluations)
    Sf, Tf, Wf = load_model(str(tmp_path / "final.ckpt"))
    assert Sf.values.tobytes() == S.values.tobytes() and Wf is None
    assert Tf.values.tobytes() == T.values.tobytes()
    Sb, Tb, _ = load_model(str(tmp_path / "best.ckpt"))
    assert Sb.values.shape == S.values.shape and Tb.values.shape == T.values.shape


@pytest.mark.parametrize("K,N,lpr,fp64,stages", [(64, 100, 1, False, 2), (64, 100, 2, False, 3),
                                                 (128, 300, 2, False, 2), (128, 300, 1, True, 4),
                                                 (128, 64, 2, True, 2), (64, 500, 2, True, 4),
                                                 (64, 60, 2, False, 4), (128, 300, 2, False, 1),
                                                 (64, 100, 1, False, 1)])
def test_staged_kernel_variants_window1_vs_oracle(torch_cuda, monkeypatch, K, N, lpr, fp64,
                                                  stages):
    """The staged throughput kernel in each row layout (one or two lanes per
    row), fp32 and fp64 dots, several ring depths: sequential run vs the
    oracle within 1e-4 norm-relative.  (Large-N cases use fp64 dots: with
    fp32 dots a margin decision |sim - theta| < ~1e-6 can flip, which is the
    fp32 mode's expected deviation, not a layout error.)"""
    from oracle import oracle as O
    from paper_2304_07334_b200 import _native as NN
    from paper_2304_07334_b200.device import DeviceModel
    monkeypatch.setenv("HEAT_HOGWILD_IMPL", "staged")
    monkeypatch.setenv("HEAT_LPR", str(lpr))
    monkeypatch.setenv("HEAT_STAGES", str(stages))
    rng = np.random.default_rng(K + N + lpr)
    nu, ni, P = 40, 250, 500
    S = (rng.standard_normal((nu, K)) * 0.1).astype(np.float32)
    T = (rng.standard_normal((ni, K)) * 0.1).astype(np.float32)
    S[3] = 0.0
    T[7] = 0.0
    u = rng.integers(0, nu, P).astype(np.int32)
    i = rng.integers(0, ni, P).astype(np.int32)
    s0 = 0x0F1E2D3C4B5A6978
    S2, T2 = S.copy(), T.copy()
    r = O.train_range(S2, T2, u, i, 0, P, s0, n_neg=N, lr=0.01, l2=0.0, mu=2.0, theta=0.1)
    model = DeviceModel(S, T)
    du, di = model.upload_pairs(u, i)
    p = model.params(n_neg=N, lr=0.01, l2=0.0, mu=2.0, theta=0.1, cosine=True,
                     mode=NN.MODE_HOGWILD, stream_base=s0, window=1, fp64=fp64)
    model.counters.reset()
    model.train_range(du, di, 0, P, p)
    c = model.counters.read()
    model.download(S, T)
    assert c.pairs == P and c.degenerate == r.degenerate
    assert abs(c.active - r.active) <= max(2, r.active // 1000)
    assert abs(c.loss - r.loss) <= 1e-4 * abs(r.loss)
    assert _rel_fro(S, S2) <= 1e-4 and _rel_fro(T, T2) <= 1e-4


@pytest.mark.parametrize("K,N,mode", [(512, 20, "hogwild"), (256, 255, "exact"), (64, 255, "hogwild"),
                                      (64, 255, "hogwild32"), (32, 63, "hogwild32"),
                                      (16, 1, "hogwild"), (1, 1, "exact"), (256, 8, "hogwild")])
def test_boundary_shapes_vs_oracle(torch_cuda, K, N, mode):
    """Size boundaries of every kernel family: the widest rows the ABI takes
    (dim 512, generic kernel), the largest resident pair (N+1 = 256 rows,
    eight 32-row stages), the largest speculative-exact row (dim 256), and
    the smallest shapes.  EXACT is bit-identical; HOGWILD at window 1 within
    1e-4 (fp64 dots; "hogwild32" = the fp32 resident kernel, with a margin
    that keeps sims away from theta so fp32 cannot flip a decision)."""
    from oracle import oracle as O
    from paper_2304_07334_b200 import _native as NN
    from paper_2304_07334_b200.device import DeviceModel
    rng = np.random.default_rng(K * 3 + N)
    nu, ni, P = 30, 400, 300
    S = (rng.standard_normal((nu, K)) * 0.1).astype(np.float32)
    T = (rng.standard_normal((ni, K)) * 0.1).astype(np.float32)
    u = rng.integers(0, nu, P).astype(np.int32)
    i = rng.integers(0, ni, P).astype(np.int32)
    s0 = 0x5EED5EED5EED5EED
    S2, T2 = S.copy(), T.copy()
    theta = 0.6 if mode == "hogwild32" else 0.05
    r = O.train_range(S2, T2, u, i, 0, P, s0, n_neg=N, lr=0.02, l2=0.0, mu=2.0, theta=theta)
    model = DeviceModel(S, T)
    du, di = model.upload_pairs(u, i)
    exact = mode == "exact"
    p = model.params(n_neg=N, lr=0.02, l2=0.0, mu=2.0, theta=theta, cosine=True,
                     mode=NN.MODE_EXACT if exact else NN.MODE_HOGWILD, stream_base=s0,
                     window=1, fp64=mode == "hogwild")
    model.counters.reset()
    model.train_range(du, di, 0, P, p)
    c = model.counters.read()
    model.download(S, T)
    assert c.pairs == P
    if exact:
        assert S.tobytes() == S2.tobytes() and T.tobytes() == T2.tobytes()
        assert c.loss == r.loss
    else:
        assert abs(c.loss - r.loss) <= 1e-4 * abs(r.loss)
        assert _rel_fro(S, S2) <= 1e-4 and _rel_fro(T, T2) <= 1e-4


@pytest.mark.parametrize("impl", ["resident", "staged", "generic", "multi"])
def test_hogwild_updates_are_sparse(torch_cuda, monkeypatch, impl):
    """Sparse updates (the reference's test_trainer.py:94-107): rows that no
    pair reads keep their exact initial bits, in every throughput kernel."""
    import torch
    from paper_2304_07334_b200 import _native as N
    from paper_2304_07334_b200.device import DeviceModel
    monkeypatch.setenv("HEAT_HOGWILD_IMPL", impl)
    rng = np.random.default_rng(17)
    nu, ni, K, NN, P = 500, 20000, 64, 40, 800
    S = (rng.standard_normal((nu, K)) * 0.1).astype(np.float32)
    T = (rng.standard_normal((ni, K)) * 0.1).astype(np.float32)
    u = rng.integers(0, nu // 2, P).astype(np.int32)  # upper half of the users never trains
    i = rng.integers(0, ni, P).astype(np.int32)
    s0 = 0xABCDEF0123456789
    m = DeviceModel(S.copy(), T.copy())
    du, di = m.upload_pairs(u, i)
    p = m.params(n_neg=NN, lr=0.05, l2=0.0, mu=2.0, theta=0.0, cosine=True,
                 mode=N.MODE_HOGWILD, stream_base=s0, window=64)
    m.counters.reset()
    m.train_range(du, di, 0, P, p)
    negs = torch.empty(P * NN, dtype=torch.int32, device="cuda")
    N.check(N.lib().heat_sample_negatives(s0, 0, P, NN, ni, ctypes_ptr(negs), None))
    read = np.zeros(ni, bool)
    read[i] = True
    read[negs.cpu().numpy()] = True
    S2, T2 = m.S.cpu().numpy(), m.T.cpu().numpy()
    assert S2[nu // 2:].tobytes() == S[nu // 2:].tobytes()
    assert T2[~read].tobytes() == T[~read].tobytes()
    assert (~read).sum() > 1000 and not np.array_equal(T2[read], T[read])


def ctypes_ptr(t):
    import ctypes
    return ctypes.c_void_p(t.data_ptr())


def test_c2_recall_parity_throughput_vs_deterministic(torch_cuda):
    """north_star: final recall@20 within 0.5 % absolute.  Full config 2, a
    few epochs: the throughput kernel (B = 1024 in flight) against the
    deterministic kernel, which is bit-identical to the reference's single
    thread.  (20 epochs: 0.1650 vs 0.1654, profiles/r01_quality_c2.json.)"""
    from paper_2304_07334_b200 import _native as N
    from paper_2304_07334_b200 import LossParams, TrainingConfig
    from paper_2304_07334_b200.dataset import epoch_pairs
    from paper_2304_07334_b200.device import DeviceModel
    from paper_2304_07334_b200.embeddings import InitSpec, init_matrix
    from paper_2304_07334_b200.evaluator import evaluate_device
    from paper_2304_07334_b200.rng import epoch_stream, shuffle_seed
    from workloads import make_dataset
    tr, te, sp = make_dataset("c2")
    rec = {}
    for mode in (N.MODE_HOGWILD, N.MODE_EXACT):
        S = init_matrix(tr.num_users, sp.dim, InitSpec(seed=0))
        T = init_matrix(tr.num_items, sp.dim, InitSpec(seed=0))
        m = DeviceModel(S.values, T.values)
        for e in range(4):
            u, i = epoch_pairs(tr, shuffle_seed(0, e))
            du, di = m.upload_pairs(u, i)
            p = m.params(n_neg=sp.negatives, lr=sp.learning_rate, l2=0.0, mu=sp.mu,
                         theta=sp.theta, cosine=True, mode=mode,
                         stream_base=epoch_stream(0, e), window=sp.batch)
            m.counters.reset()
            m.train_range(du, di, 0, len(u), p)
        cfg = TrainingConfig(emb_dim=sp.dim, num_negatives=sp.negatives,
                             loss=LossParams(mu=sp.mu, theta=sp.theta))
        rec[mode] = evaluate_device(m, S, T, tr, te, cfg, k=20).recall_at_k
    assert rec[N.MODE_EXACT] > 0.05  # training moved far from the init (0.0005)
    assert abs(rec[N.MODE_HOGWILD] - rec[N.MODE_EXACT]) <= 0.005, rec


@pytest.mark.parametrize("K,N,window", [(64, 500, 1), (32, 300, 1), (64, 100, 1), (64, 500, 64),
                                        (128, 300, 1), (128, 64, 1), (128, 500, 64)])
def test_multi_warp_kernel_vs_oracle(torch_cuda, monkeypatch, K, N, window):
    """The several-warps-per-pair kernel (csrc/heat_hogwild_multi.cu, the
    default for K <= 64 with N + 1 > 256): window 1 tracks the oracle within
    1e-4 (theta keeps fp32 away from margin flips); with 64 pairs in flight
    the loss stays within 2 % of the sequential run."""
    from oracle import oracle as O
    from paper_2304_07334_b200 import _native as NN
    from paper_2304_07334_b200.device import DeviceModel
    monkeypatch.setenv("HEAT_HOGWILD_IMPL", "multi")
    rng = np.random.default_rng(K + N + window)
    nu, ni, P = 40, 3000, 400
    S = (rng.standard_normal((nu, K)) * 0.1).astype(np.float32)
    T = (rng.standard_normal((ni, K)) * 0.1).astype(np.float32)
    S[3] = 0.0
    u = rng.integers(0, nu, P).astype(np.int32)
    i = rng.integers(0, ni, P).astype(np.int32)
    s0 = 0x1122334455667788
    S2, T2 = S.copy(), T.copy()
    r = O.train_range(S2, T2, u, i, 0, P, s0, n_neg=N, lr=0.02, l2=0.0, mu=2.0, theta=0.5)
    model = DeviceModel(S, T)
    du, di = model.upload_pairs(u, i)
    p = model.params(n_neg=N, lr=0.02, l2=0.0, mu=2.0, theta=0.5, cosine=True,
                     mode=NN.MODE_HOGWILD, stream_base=s0, window=window)
    model.counters.reset()
    model.train_range(du, di, 0, P, p)
    c = model.counters.read()
    model.download(S, T)
    assert c.pairs == P and c.degenerate == r.degenerate
    if window == 1:
        assert abs(c.loss - r.loss) <= 1e-4 * abs(r.loss)
        assert _rel_fro(S, S2) <= 1e-4 and _rel_fro(T, T2) <= 1e-4
    else:
        assert abs(c.loss - r.loss) <= 0.02 * abs(r.loss)


@pytest.mark.parametrize("K,N", [(64, 300), (128, 300), (32, 40)])
def test_delta_mode_every_kernel_family(torch_cuda, K, N):
    """DELTA mode (the multi-GPU step) through each throughput kernel family
    the dispatcher picks (multi-warp for K 64 / N 300, staged for K 128,
    resident for K 32 / N 40): two logical ranks on one GPU through the
    pipelined driver keep bit-identical item replicas and train every pair."""
    import torch
    from paper_2304_07334_b200 import _native as NN
    from paper_2304_07334_b200.dataset import epoch_pairs
    from paper_2304_07334_b200.device import DeviceModel
    from paper_2304_07334_b200.embeddings import InitSpec, init_matrix
    from paper_2304_07334_b200.parallel import PipelinedShardTrainer, run_loopback
    from paper_2304_07334_b200.rng import epoch_stream, shuffle_seed
    from workloads import make_clustered
    train, _ = make_clustered(600, 3000, 8, 30, seed=5)
    S = init_matrix(600, K, InitSpec(seed=1)).values
    T = init_matrix(3000, K, InitSpec(seed=2)).values
    ranks = [PipelinedShardTrainer(DeviceModel(S, T), 2, r) for r in range(2)]
    u, i = epoch_pairs(train, shuffle_seed(0, 0))
    gens = []
    for tr in ranks:
        p = tr.model.params(n_neg=N, lr=0.05, l2=0.0, mu=1.0, theta=0.3, cosine=True,
                            mode=NN.MODE_DELTA, stream_base=epoch_stream(0, 0), window=128)
        tr.model.counters.reset()
        gens.append(tr.epoch_pipeline(u, i, p, 512))
    run_loopback(gens)
    torch.cuda.synchronize()
    cs = [tr.model.counters.read() for tr in ranks]
    assert sum(c.pairs for c in cs) == len(u)
    assert sum(st.entries for st in ranks[0].stats) >= len(u)
    T0 = ranks[0].model.T.cpu().numpy()
    assert ranks[1].model.T.cpu().numpy().tobytes() == T0.tobytes()
    assert np.isfinite(T0).all() and not np.array_equal(T0, T)


@pytest.mark.parametrize("cfg", ["c1", "c2", "c3", "c4", "c5"])
def test_full_size_properties(torch_cuda, cfg):
    """BASELINE.json's full sizes (c1-c3; c4 53 k x 92 k x 128, N 1000; c5 10 M x 2 M
    x 128 tables with a 2 % user sample), through size-independent
    properties: every pair trained exactly once per epoch, the loss finite and
    falling, the tables finite, and user rows that own no pair bit-identical
    to their initial values (sparse updates, test_trainer.py:94-107)."""
    import torch
    from paper_2304_07334_b200 import _native as N
    from paper_2304_07334_b200.dataset import epoch_pairs
    from paper_2304_07334_b200.device import DeviceModel
    from paper_2304_07334_b200.embeddings import InitSpec, init_matrix
    from paper_2304_07334_b200.rng import epoch_stream, shuffle_seed
    from workloads import make_dataset
    kw = {"sample_users": 0.02} if cfg == "c5" else {}
    tr, _, sp = make_dataset(cfg, **kw)
    S = init_matrix(tr.num_users, sp.dim, InitSpec(seed=0)).values
    T = init_matrix(tr.num_items, sp.dim, InitSpec(seed=0)).values
    m = DeviceModel(S, T)
    losses = []
    for e in range(2):
        u, i = epoch_pairs(tr, shuffle_seed(0, e))
        du, di = m.upload_pairs(u, i)
        p = m.params(n_neg=sp.negatives, lr=sp.learning_rate, l2=0.0, mu=sp.mu, theta=sp.theta,
                     cosine=True, mode=N.MODE_HOGWILD, stream_base=epoch_stream(0, e),
                     window=sp.batch)
        m.counters.reset()
        m.train_range(du, di, 0, len(u), p)
        c = m.counters.read()
        assert c.pairs == tr.num_pairs and np.isfinite(c.loss)
        losses.append(c.loss / c.pairs)
    assert losses[1] < losses[0]
    idle = np.flatnonzero(np.diff(tr.offsets) == 0)  # users without a pair
    S2 = m.S[torch.from_numpy(idle).cuda()].cpu().numpy() if len(idle) else None
    if S2 is not None:
        assert S2.tobytes() == S[idle].tobytes()
    assert bool(torch.isfinite(m.S).all()) and bool(torch.isfinite(m.T).all())
