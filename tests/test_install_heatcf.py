"""install() against the real reference package, when it is importable
(build container only: /root/reference is absent on the GPU box).  Checks the
rebinding itself on CPU; the GPU run of heatcf.train through the patched
entry points is exercised where both exist."""

import importlib
import os
import sys

import pytest

REF = "/root/reference/pkg/src"


@pytest.fixture
def heatcf_mod(monkeypatch):
    if not os.path.isdir(REF):
        pytest.skip("reference not present")
    monkeypatch.setenv("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    monkeypatch.setenv("PYTHONDONTWRITEBYTECODE", "1")
    sys.dont_write_bytecode = True
    monkeypatch.syspath_prepend(REF)
    try:
        return importlib.import_module("heatcf")
    except Exception as exc:  # pragma: no cover
        pytest.skip(f"heatcf not importable: {exc}")


def test_install_rebinds_and_uninstall_restores(heatcf_mod):
    import heatcf.evaluator
    import heatcf.trainer
    from paper_2304_07334_b200 import evaluator, trainer
    from paper_2304_07334_b200.install import install, uninstall
    orig_te, orig_ev = heatcf.trainer.train_epoch, heatcf.evaluator.evaluate
    install(heatcf_mod)
    try:
        assert heatcf.trainer.train_epoch is trainer.train_epoch
        assert heatcf.evaluator.evaluate is evaluator.evaluate
        assert heatcf_mod.train_epoch is trainer.train_epoch
    finally:
        uninstall()
    assert heatcf.trainer.train_epoch is orig_te
    assert heatcf.evaluator.evaluate is orig_ev


def test_reference_objects_flow_through_validation(heatcf_mod):
    """heatcf's own dataclasses are accepted (duck typing) and validated in
    the reference's order before any device work."""
    from paper_2304_07334_b200.trainer import train_epoch
    train = heatcf_mod.dataset.from_user_lists({0: [1]}, num_users=2, num_items=3)
    S = heatcf_mod.init_matrix(2, 8, heatcf_mod.InitSpec(seed=1))
    T = heatcf_mod.init_matrix(3, 8, heatcf_mod.InitSpec(seed=2))
    with pytest.raises(ValueError):
        train_epoch(S, T, train, heatcf_mod.TrainingConfig(emb_dim=4, num_negatives=1))
    with pytest.raises(ValueError):
        train_epoch(S, T, train, heatcf_mod.TrainingConfig(
            emb_dim=8, num_negatives=1,
            sampler=heatcf_mod.SamplerConfig(kind="tiling", tile_size=2, refresh_interval=2)))


def test_installed_bench_skips_the_tiling_sampler():
    """Both shipped configs bench `uniform,tiling`; the tiling sampler is not
    on the B200 path, so the installed run_bench drops those variants up front
    and says so in its warnings (rather than stopping at the first tiling row)."""
    import dataclasses
    from paper_2304_07334_b200.install import _bench_without_tiling
    seen = []

    @dataclasses.dataclass(frozen=True)
    class Cfg:
        bench_samplers: tuple = ("uniform", "tiling")

    def fake_run_bench(train, cfg, log=None):
        seen.append(cfg.bench_samplers)
        return [{"variant": "uniform"}], ["w"]

    logs = []
    rows, warnings = _bench_without_tiling(fake_run_bench)(None, Cfg(), log=logs.append)
    assert seen == [("uniform",)] and rows == [{"variant": "uniform"}]
    assert "tiling" in warnings[0] and warnings[1:] == ["w"] and "tiling" in logs[0]
    rows, warnings = _bench_without_tiling(fake_run_bench)(None, Cfg(("uniform",)))
    assert seen[-1] == ("uniform",) and warnings == ["w"]


def test_kernels_spec_restatement_matches_reference(heatcf_mod):
    """oracle/kernels_spec.py (the A13 checker used by tests/test_gpu_math_spec.py)
    against heatcf.kernels itself: identical cosine reductions, loss and
    gradients on random inputs, and the same degenerate handling."""
    import numpy as np
    import heatcf.kernels as RK
    from oracle import kernels_spec as KS
    rng = np.random.default_rng(7)
    for dim in (2, 33, 128):
        for _ in range(20):
            u = rng.standard_normal(dim)
            v = rng.standard_normal(dim)
            c = RK.cosine_forward(u, v)
            assert KS.cosine_forward(u, v) == (c.ss, c.tt, c.st, c.sim, c.degenerate)
            assert np.array_equal(KS.cosine_grad_user(u, v), RK.cosine_grad_user(u, v, c))
            assert np.array_equal(KS.cosine_grad_item(u, v), RK.cosine_grad_item(u, v, c))
            mu, theta = float(rng.uniform(0, 3)), float(rng.uniform(-0.9, 0.9))
            negs = rng.uniform(-1, 1, int(rng.integers(1, 9)))
            p = RK.LossParams(mu=mu, theta=theta)
            assert KS.ccl_loss(0.3, negs, mu, theta) == RK.ccl_loss(0.3, negs, p)
            dp, dn = KS.ccl_loss_grad(0.3, negs, mu, theta)
            rdp, rdn = RK.ccl_loss_grad(0.3, negs, p)
            assert dp == rdp and np.array_equal(dn, rdn)
    z = np.zeros(4)
    assert KS.cosine_forward(z, np.ones(4))[3:] == (0.0, True)
    assert not KS.cosine_grad_user(z, np.ones(4)).any()


def test_reference_arm_sample_is_a_valid_subset(heatcf_mod):
    """bench.py --impl reference times heatcf itself on a bounded sample: the
    sample is a well-formed heatcf InteractionSet over the full universe whose
    pairs are a subset of the workload's, and one heatcf epoch over it runs."""
    import numpy as np

    import bench
    import heatcf.embeddings
    import heatcf.trainer
    train, _, spec, S, T = bench.build_workload("c1")
    sub = bench.heatcf_sample(heatcf_mod, spec, train, 5000)
    assert (sub.num_users, sub.num_items, sub.num_pairs) == (train.num_users, train.num_items, 5000)
    full = {(u, int(i)) for u in range(train.num_users)
            for i in train.items[train.offsets[u]:train.offsets[u + 1]]}
    for u in range(sub.num_users):
        sl = sub.slice(u)
        assert np.all(np.diff(sl) > 0)  # ascending, no duplicates
        assert all((u, int(i)) in full for i in sl)
    cfg = heatcf.trainer.TrainingConfig(emb_dim=spec.dim, num_negatives=spec.negatives,
                                        learning_rate=spec.learning_rate, num_threads=2,
                                        loss=heatcf.trainer.LossParams(mu=spec.mu, theta=spec.theta))
    r = heatcf.trainer.train_epoch(heatcf.embeddings.EmbeddingMatrix(S.copy()),
                                   heatcf.embeddings.EmbeddingMatrix(T.copy()), sub, cfg)
    assert r.num_pairs == 5000 and np.isfinite(r.mean_loss) and r.wall_time > 0
