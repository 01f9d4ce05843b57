"""Phase profile of train_epoch(collect_phases=True) on the device.

The reference accumulates cycle counts per phase (read_emb, similarity, loss,
gradient, update, aggregate) inside its numba loop and reports seconds
averaged over its threads (trainer.py:120-331, 452-457; timing.py:20-53).
Here the phase-instrumented kernels (heat_phase_collect / heat_phase_read)
do the same with clock64: the serial EXACT kernel (the reference's phases one
pair at a time), the register-streamed Hogwild kernel at dim 64/128 and the
generic Hogwild kernel at other dims.  Checked: every phase the path runs is
positive, the others are zero, the phases fit in the wall time, and turning
the profile on changes no result in EXACT mode.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu



@pytest.fixture(scope="module")
def torch_cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2304_07334_b200.trainer import configure
    configure(mode=None, window=0, fp64=False)  # the reference's thread-count mapping
    return torch


PHASES = ("read_emb", "similarity", "loss", "gradient", "update", "aggregate")


def _data(dim, users=300, items=900, seed=5):
    from paper_2304_07334_b200 import InitSpec, init_matrix
    from workloads import make_clustered
    train, _ = make_clustered(users, items, 6, 20, seed=seed)
    S = init_matrix(train.num_users, dim, InitSpec(seed=1))
    T = init_matrix(train.num_items, dim, InitSpec(seed=2))
    return train, S, T


def _cfg(dim, threads, n_neg=50, theta=0.2, **kw):
    from paper_2304_07334_b200 import LossParams, TrainingConfig
    return TrainingConfig(emb_dim=dim, num_negatives=n_neg, learning_rate=0.05,
                          num_threads=threads, loss=LossParams(mu=5.0, theta=theta), seed=3, **kw)


@pytest.mark.parametrize("dim,threads", [(128, 8), (64, 8), (16, 8), (32, 1), (128, 1)])
def test_phases_measured(torch_cuda, dim, threads):
    from paper_2304_07334_b200.trainer import train_epoch
    train, S, T = _data(dim)
    rep = train_epoch(S, T, train, _cfg(dim, threads), epoch=0, collect_phases=True)
    assert set(rep.phase_times) == set(PHASES)
    for name in PHASES[:5]:
        assert rep.phase_times[name] > 0, (name, rep.phase_times)
    assert rep.phase_times["aggregate"] == 0
    assert sum(rep.phase_times.values()) <= rep.wall_time
    # no phases are left on: the next epoch without the profile reports zeros
    rep2 = train_epoch(S, T, train, _cfg(dim, threads), epoch=1)
    assert all(v == 0 for v in rep2.phase_times.values())


def test_exact_profile_changes_no_bits(torch_cuda):
    """EXACT with the profile on runs the serial kernel; its tables, losses and
    counters equal the default (speculative) kernel's bit for bit."""
    from paper_2304_07334_b200.trainer import train_epoch
    out = []
    for phases in (False, True):
        train, S, T = _data(64, seed=9)
        cfg = _cfg(64, 1, n_neg=40, theta=0.1)
        reps = [train_epoch(S, T, train, cfg, epoch=e, collect_phases=phases) for e in range(2)]
        out.append((S.values.tobytes(), T.values.tobytes(),
                    [(r.mean_loss, r.degenerate_count, r.active_negatives) for r in reps]))
    assert out[0] == out[1]


def test_exact_aggregator_phase(torch_cuda):
    from paper_2304_07334_b200 import AggregatorConfig, InitSpec, init_matrix
    from paper_2304_07334_b200.trainer import train_epoch
    train, S, T = _data(16, users=120, items=400)
    W = init_matrix(16, 16, InitSpec(kind="xavier", seed=9)).values
    cfg = _cfg(16, 1, n_neg=8, aggregator=AggregatorConfig(enabled=True, max_history=20))
    rep = train_epoch(S, T, train, cfg, W, epoch=0, collect_phases=True)
    for name in PHASES:
        assert rep.phase_times[name] > 0, (name, rep.phase_times)
    assert sum(rep.phase_times.values()) <= rep.wall_time


def test_phase_read_counts_workers(torch_cuda):
    """heat_phase_read: workers and pairs of the launches since the last reset."""
    import ctypes
    from paper_2304_07334_b200 import _native as N
    from paper_2304_07334_b200.trainer import train_epoch, _phase_begin
    train, S, T = _data(128)
    _phase_begin()
    try:
        train_epoch(S, T, train, _cfg(128, 8), epoch=0)
        L = N.lib()
        sec = (ctypes.c_double * 6)()
        w, p = ctypes.c_int64(0), ctypes.c_int64(0)
        N.check(L.heat_phase_read(sec, ctypes.byref(w), ctypes.byref(p), 1))
    finally:
        N.check(N.lib().heat_phase_collect(0))
    assert p.value == train.num_pairs
    assert 1 <= w.value <= train.num_pairs
    assert all(np.isfinite(list(sec)))
