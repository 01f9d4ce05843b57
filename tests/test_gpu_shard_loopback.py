"""The native multi-GPU runtime (csrc/heat_shard.cu) at world > 1, as
`world` ranks of one process on one GPU (heat_shard_epoch_loopback; the
B200 box of this build has one GPU, and ranks whose kernels wait on one
another must not share a GPU — here nothing spins: every cross-rank
dependency is an event wait).

Exercised: the rank-local DELTA steps, the count "collective" as the
cross-rank fence, the fused gather+apply reading the peers' logs through
device pointers, the gather fallback, the log-slot rotation under each lag,
the exact-capacity logs, and replica bit-identity.  Not exercised here: the
CUDA IPC mapping (tests/test_gpu_shard_ipc.py runs two processes for that)
and the NCCL calls themselves (they need two GPUs).

Determinism argument used by the first test: with one pair in flight per
rank (one warp per pair) and lag 1, step s of every rank reads T as left by the apply of step
s-1, users are disjoint between ranks and the fixed-point apply is
order-free, so the sharded epoch does not depend on the number of ranks —
the world-G tables equal the world-1 tables bit for bit.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    assert torch.cuda.is_available()
    from paper_2304_07334_b200 import _native
    _native.lib()
    return torch


def _setup(K, scale=0.02):
    from paper_2304_07334_b200.embeddings import InitSpec, init_matrix
    from workloads import make_dataset
    train, _, _ = make_dataset("c2", scale=scale)
    S = init_matrix(train.num_users, K, InitSpec(seed=0)).values
    T = init_matrix(train.num_items, K, InitSpec(seed=0)).values
    return train, S, T


def _params(m, e, window, N=100, theta=0.3):
    from paper_2304_07334_b200 import _native as NN
    from paper_2304_07334_b200.rng import epoch_stream
    return m.params(n_neg=N, lr=0.01, l2=0.0, mu=20.0, theta=theta, cosine=True,
                    mode=NN.MODE_DELTA, stream_base=epoch_stream(0, e), window=window)


@pytest.mark.parametrize("G,K", [(2, 64), (3, 128)])
def test_world_g_equals_world_1_bit_exact(torch_cuda, monkeypatch, G, K):
    from paper_2304_07334_b200.dataset import epoch_pairs
    from paper_2304_07334_b200.device import DeviceModel
    from paper_2304_07334_b200.parallel import LoopbackShardGroup, NativeShardTrainer
    from paper_2304_07334_b200.rng import shuffle_seed
    monkeypatch.setenv("HEAT_SHARD_LAG", "1")
    monkeypatch.setenv("HEAT_SHARD_GRAPH", "0")
    # one warp per pair (the register-streamed kernel): with one pair in
    # flight its user-row update is a single add per element, so a run is
    # deterministic (the pair-per-CTA kernel adds four warps' shares in
    # arrival order)
    monkeypatch.setenv("HEAT_HOGWILD_IMPL", "wide")
    train, S, T = _setup(K)
    ref = DeviceModel(S, T)
    one = NativeShardTrainer(ref, 1, 0)
    grp = LoopbackShardGroup([DeviceModel(S, T) for _ in range(G)])
    for e in range(2):
        u, i = epoch_pairs(train, shuffle_seed(0, e))
        ref.counters.reset()
        one.train_epoch(u, i, _params(ref, e, 1), 256)
        for m in grp.models:
            m.counters.reset()
        st = grp.train_epoch(u, i, _params(grp.models[0], e, 1), 256)
        assert sum(m.counters.read().pairs for m in grp.models) == len(u)
        assert all(s.steps == st[0].steps for s in st) and st[0].entries >= len(u)
        assert st[0].exchanged_bytes > 0
        T0 = grp.models[0].T.cpu().numpy()
        for m in grp.models[1:]:
            assert m.T.cpu().numpy().tobytes() == T0.tobytes()  # replicas identical
        assert T0.tobytes() == ref.T.cpu().numpy().tobytes()  # = the world-1 epoch
        S_ref = ref.S.cpu().numpy()
        for r, m in enumerate(grp.models):  # each rank owns users u % G
            mine = np.arange(train.num_users) % G == r
            assert m.S.cpu().numpy()[mine].tobytes() == S_ref[mine].tobytes()
        loss = sum(m.counters.read().loss for m in grp.models)
        assert abs(loss - ref.counters.read().loss) <= 1e-9 * abs(loss)
    grp.close()
    one.close()


@pytest.mark.parametrize("lag,exchange", [("2", "p2p"), ("3", "p2p"), ("1", "gather"),
                                          ("2", "gather")])
def test_world_2_concurrent_steps_keep_replicas_identical(torch_cuda, monkeypatch, lag, exchange):
    """Many pairs in flight, every staleness bound, both exchanges (the
    gather fallback runs lag >= 2 whatever HEAT_SHARD_LAG says): every pair
    trained once, replicas bit-identical, loss within 3 % of the world-1
    runtime at the same settings."""
    from paper_2304_07334_b200.dataset import epoch_pairs
    from paper_2304_07334_b200.device import DeviceModel
    from paper_2304_07334_b200.parallel import LoopbackShardGroup, NativeShardTrainer
    from paper_2304_07334_b200.rng import shuffle_seed
    monkeypatch.setenv("HEAT_SHARD_LAG", lag)
    monkeypatch.setenv("HEAT_SHARD_EXCHANGE", exchange)
    train, S, T = _setup(64, scale=0.05)
    grp = LoopbackShardGroup([DeviceModel(S, T) for _ in range(2)])
    ref = DeviceModel(S, T)
    one = NativeShardTrainer(ref, 1, 0)
    for e in range(3):
        u, i = epoch_pairs(train, shuffle_seed(0, e))
        for m in grp.models:
            m.counters.reset()
        grp.train_epoch(u, i, _params(grp.models[0], e, 256), 1024)
        ref.counters.reset()
        one.train_epoch(u, i, _params(ref, e, 256), 1024)
        assert sum(m.counters.read().pairs for m in grp.models) == len(u)
        assert (grp.models[0].T.cpu().numpy().tobytes() ==
                grp.models[1].T.cpu().numpy().tobytes())
    loss = sum(m.counters.read().loss for m in grp.models)
    want = ref.counters.read().loss
    assert np.isfinite(loss) and abs(loss - want) <= 0.03 * abs(want), (loss, want)
    grp.close()
    one.close()


def test_theta_below_zero_fills_the_log_without_loss(torch_cuda):
    """theta -1 makes every negative active: each pair logs N + 1 entries, the
    exact worst case the capacity is sized for.  Nothing is dropped (the
    applied entry count is exactly pairs x (N + 1)) and the replicas agree."""
    from paper_2304_07334_b200.dataset import epoch_pairs
    from paper_2304_07334_b200.device import DeviceModel
    from paper_2304_07334_b200.parallel import LoopbackShardGroup
    from paper_2304_07334_b200.rng import shuffle_seed
    train, S, T = _setup(64)
    grp = LoopbackShardGroup([DeviceModel(S, T) for _ in range(2)])
    u, i = epoch_pairs(train, shuffle_seed(0, 0))
    st = grp.train_epoch(u, i, _params(grp.models[0], 0, 128, N=40, theta=-1.0), 512)
    assert st[0].entries == len(u) * 41
    assert st[0].max_entries <= 512 * 41
    assert (grp.models[0].T.cpu().numpy().tobytes() == grp.models[1].T.cpu().numpy().tobytes())
    grp.close()


@pytest.mark.parametrize("G,K", [(1, 128), (2, 64), (2, 128)])
def test_persistent_epoch_equals_stream_ordered_steps(torch_cuda, monkeypatch, G, K):
    """The persistent epoch (one launch, steps gated on the device, applies
    done by the workers between pairs) against the stream-ordered step
    runtime (HEAT_SHARD_PERSIST=0): with one pair in flight per rank and lag
    1 both train step s against T as left by the apply of step s-1, so the
    tables, the user rows and the loss agree bit for bit."""
    from paper_2304_07334_b200.dataset import epoch_pairs
    from paper_2304_07334_b200.device import DeviceModel
    from paper_2304_07334_b200.parallel import LoopbackShardGroup, NativeShardTrainer
    from paper_2304_07334_b200.rng import shuffle_seed
    monkeypatch.setenv("HEAT_SHARD_LAG", "1")
    monkeypatch.setenv("HEAT_SHARD_GRAPH", "0")
    monkeypatch.setenv("HEAT_HOGWILD_IMPL", "wide")
    train, S, T = _setup(K)

    def run(persist):
        monkeypatch.setenv("HEAT_SHARD_PERSIST", persist)
        if G == 1:
            ms = [DeviceModel(S, T)]
            tr = NativeShardTrainer(ms[0], 1, 0)
        else:
            tr = LoopbackShardGroup([DeviceModel(S, T) for _ in range(G)])
            ms = tr.models
        stats = []
        for e in range(2):
            u, i = epoch_pairs(train, shuffle_seed(0, e))
            for m in ms:
                m.counters.reset()
            st = tr.train_epoch(u, i, _params(ms[0], e, 1), 256)
            stats.append(st)
            assert sum(m.counters.read().pairs for m in ms) == len(u)
        out = ([m.T.cpu().numpy().copy() for m in ms], [m.S.cpu().numpy().copy() for m in ms],
               sum(m.counters.read().loss for m in ms), stats)
        tr.close()
        return out

    Tp, Sp, lp, sp = run("2")  # (2: also at K = 64, where the default is stream-ordered)
    Ts, Ss, ls, ss = run("0")
    for a, b in zip(Tp + Sp, Ts + Ss):
        assert a.tobytes() == b.tobytes()
    assert abs(lp - ls) <= 1e-12 * abs(ls)  # (fp64 sums grouped per launch)
    a = sp[-1] if G > 1 else [sp[-1]]
    b = ss[-1] if G > 1 else [ss[-1]]
    assert [(x.steps, x.entries, x.max_entries) for x in a] == \
        [(x.steps, x.entries, x.max_entries) for x in b]


@pytest.mark.parametrize("G,K,lag", [(1, 128, "2"), (1, 64, "3"), (2, 128, "2"), (4, 64, "2")])
def test_persistent_epoch_full_occupancy(torch_cuda, monkeypatch, G, K, lag):
    """Every resident worker in flight (no window), several epochs back to
    back (the global step count and the mailbox epoch tags carry over):
    every pair trained once, nothing dropped from the logs, replicas
    bit-identical, loss within 3 % of the stream-ordered runtime."""
    from paper_2304_07334_b200.dataset import epoch_pairs
    from paper_2304_07334_b200.device import DeviceModel
    from paper_2304_07334_b200.parallel import LoopbackShardGroup, NativeShardTrainer
    from paper_2304_07334_b200.rng import shuffle_seed
    monkeypatch.setenv("HEAT_SHARD_LAG", lag)
    train, S, T = _setup(K, scale=0.05)

    def run(persist):
        monkeypatch.setenv("HEAT_SHARD_PERSIST", persist)
        if G == 1:
            ms = [DeviceModel(S, T)]
            tr = NativeShardTrainer(ms[0], 1, 0)
        else:
            tr = LoopbackShardGroup([DeviceModel(S, T) for _ in range(G)])
            ms = tr.models
        for e in range(3):
            u, i = epoch_pairs(train, shuffle_seed(0, e))
            for m in ms:
                m.counters.reset()
            tr.train_epoch(u, i, _params(ms[0], e, 0), 512)
            assert sum(m.counters.read().pairs for m in ms) == len(u)
            T0 = ms[0].T.cpu().numpy()
            for m in ms[1:]:
                assert m.T.cpu().numpy().tobytes() == T0.tobytes()
        loss = sum(m.counters.read().loss for m in ms)
        tr.close()
        return loss

    lp = run("2")
    ls = run("0")
    assert np.isfinite(lp) and abs(lp - ls) <= 0.03 * abs(ls), (lp, ls)


@pytest.mark.parametrize("K,launches_one", [(128, True), (64, False)])
def test_default_mode_by_dim(torch_cuda, monkeypatch, K, launches_one):
    """The runtime's default: the persistent epoch (one launch) at K = 128,
    the stream-ordered steps (a DELTA kernel and two apply kernels per step)
    at K = 64; both train every pair once."""
    from paper_2304_07334_b200.dataset import epoch_pairs
    from paper_2304_07334_b200.device import DeviceModel
    from paper_2304_07334_b200.parallel import NativeShardTrainer
    from paper_2304_07334_b200.rng import shuffle_seed
    for v in ("HEAT_SHARD_PERSIST", "HEAT_SHARD_LAG", "HEAT_SHARD_GRAPH", "HEAT_HOGWILD_IMPL"):
        monkeypatch.delenv(v, raising=False)
    train, S, T = _setup(K)
    m = DeviceModel(S, T)
    tr = NativeShardTrainer(m, 1, 0)
    u, i = epoch_pairs(train, shuffle_seed(0, 0))
    m.counters.reset()
    st = tr.train_epoch(u, i, _params(m, 0, 0), 512)
    assert m.counters.read().pairs == len(u)
    assert st.steps > 1
    assert (st.launches == 1) == launches_one, (st.launches, st.steps)
    if not launches_one:
        assert st.launches == 3 * st.steps
    tr.close()


@pytest.mark.parametrize("lag", ["1", "3"])
def test_persistent_epoch_with_empty_steps(torch_cuda, monkeypatch, lag):
    """Steps in which a rank has no pairs at all (its log is published empty
    at kernel start) and steps with nothing to apply: the first half of the
    epoch only holds rank 0's users.  Every pair is trained once, the
    replicas agree bit for bit, and at one pair in flight with lag 1 the
    world-2 epoch equals the world-1 epoch bit for bit."""
    from paper_2304_07334_b200.dataset import epoch_pairs
    from paper_2304_07334_b200.device import DeviceModel
    from paper_2304_07334_b200.parallel import LoopbackShardGroup, NativeShardTrainer
    from paper_2304_07334_b200.rng import shuffle_seed
    monkeypatch.setenv("HEAT_SHARD_LAG", lag)
    monkeypatch.setenv("HEAT_SHARD_GRAPH", "0")
    train, S, T = _setup(128)
    u, i = epoch_pairs(train, shuffle_seed(0, 0))
    order = np.argsort(u % 2, kind="stable")  # rank 0's users (even) first
    u, i = u[order][:4000], i[order][:4000]
    window = 1 if lag == "1" else 0
    grp = LoopbackShardGroup([DeviceModel(S, T) for _ in range(2)])
    for m in grp.models:
        m.counters.reset()
    st = grp.train_epoch(u, i, _params(grp.models[0], 0, window), 256)
    assert sum(m.counters.read().pairs for m in grp.models) == len(u)
    assert st[0].launches == 1 and st[0].steps > 4
    T0 = grp.models[0].T.cpu().numpy()
    assert grp.models[1].T.cpu().numpy().tobytes() == T0.tobytes()
    if lag == "1":
        ref = DeviceModel(S, T)
        one = NativeShardTrainer(ref, 1, 0)
        ref.counters.reset()
        one.train_epoch(u, i, _params(ref, 0, 1), 256)
        assert T0.tobytes() == ref.T.cpu().numpy().tobytes()
        one.close()
    grp.close()
