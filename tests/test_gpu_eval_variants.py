"""The three recall/NDCG kernels of csrc/heat_eval.cu agree with one another
and with the oracle evaluator (evaluator.py:113-179 restated) — top-k lists
included — on data built to hit the merge's corners: duplicated item rows
(exact score ties, which the reference breaks towards the lower id,
evaluator.py:61-73), zero user and item vectors (cosine 0 by definition),
k below / at / above the 32-entry lane-resident list, and the catalog cut into
item ranges whose lists eval_finish_kernel merges."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

VARIANTS = {
    "fragment-resident": {},
    "fragment-resident, 2 item ranges": {"HEAT_EVAL_SPLIT": "2"},
    "register-blocked": {"HEAT_EVAL_RB": "1"},
    "plain": {"HEAT_EVAL_PLAIN": "1"},
}


def _data(K, seed):
    from paper_2304_07334_b200.dataset import from_user_lists
    rng = np.random.default_rng(seed)
    nu, ni = 150, 3000
    S = rng.standard_normal((nu, K)).astype(np.float32)
    T = rng.standard_normal((ni, K)).astype(np.float32)
    T[rng.integers(0, ni, 400)] = T[rng.integers(0, ni, 400)]  # exact ties, far apart in id
    T[ni // 2 - 3:ni // 2 + 3] = T[7]                           # ... and across the range cut
    T[:4] = 0.0
    S[3] = 0.0
    tr = from_user_lists({u: rng.integers(0, ni, int(rng.integers(0, 60))) for u in range(nu)},
                         num_users=nu, num_items=ni)
    te = from_user_lists({u: rng.integers(0, ni, int(rng.integers(1, 8)))
                          for u in range(0, nu, 2)}, num_users=nu, num_items=ni)
    return S, T, tr, te


@pytest.mark.parametrize("K", [16, 64, 128])
@pytest.mark.parametrize("sim", ["cosine", "dot"])
def test_eval_kernels_agree(monkeypatch, K, sim):
    import torch

    from oracle import oracle as O
    from paper_2304_07334_b200.evaluator import eval_users_device
    assert torch.cuda.is_available()
    S, T, tr, te = _data(K, seed=K)
    users = np.flatnonzero(np.diff(te.offsets) > 0).astype(np.int32)
    Sd, Td = torch.from_numpy(S).cuda(), torch.from_numpy(T).cuda()
    for k in (5, 20, 40):
        want = O.evaluate_ref(S, T, tr.offsets, tr.items, tr.num_users, te.offsets, te.items,
                              te.num_users, k=k, similarity=sim)
        first = None
        for name, env in VARIANTS.items():
            for var in ("HEAT_EVAL_SPLIT", "HEAT_EVAL_RB", "HEAT_EVAL_PLAIN"):
                monkeypatch.delenv(var, raising=False)
            for var, val in env.items():
                monkeypatch.setenv(var, val)
            rec, nd, top = eval_users_device(Sd, Td, users, tr, te, k, sim == "cosine",
                                             want_topk=True)
            assert abs(float(np.mean(rec)) - want[0]) <= 1e-12, (name, k)
            assert abs(float(np.mean(nd)) - want[1]) <= 1e-12, (name, k)
            if first is None:
                first = (rec, nd, top)
            else:  # the same lists, entry for entry (ties included)
                assert np.array_equal(top, first[2]), (name, k)
                assert np.array_equal(rec, first[0]) and np.array_equal(nd, first[1]), (name, k)


def test_small_user_set_is_split_over_item_ranges(monkeypatch):
    """A handful of users against a long catalog: the launcher cuts the catalog
    into item ranges on its own (one CTA per range) and the merged lists equal
    the unsplit kernel's."""
    import torch

    from paper_2304_07334_b200.dataset import from_user_lists
    from paper_2304_07334_b200.evaluator import eval_users_device
    rng = np.random.default_rng(11)
    nu, ni, K = 40, 40000, 64
    S = rng.standard_normal((nu, K)).astype(np.float32)
    T = rng.standard_normal((ni, K)).astype(np.float32)
    tr = from_user_lists({u: rng.integers(0, ni, 30) for u in range(nu)}, num_users=nu,
                         num_items=ni)
    te = from_user_lists({u: rng.integers(0, ni, 5) for u in range(nu)}, num_users=nu,
                         num_items=ni)
    users = np.arange(nu, dtype=np.int32)
    Sd, Td = torch.from_numpy(S).cuda(), torch.from_numpy(T).cuda()
    for var in ("HEAT_EVAL_SPLIT", "HEAT_EVAL_RB", "HEAT_EVAL_PLAIN"):
        monkeypatch.delenv(var, raising=False)
    auto = eval_users_device(Sd, Td, users, tr, te, 20, True, want_topk=True)
    monkeypatch.setenv("HEAT_EVAL_SPLIT", "1")
    one = eval_users_device(Sd, Td, users, tr, te, 20, True, want_topk=True)
    for a, b in zip(auto, one):
        assert np.array_equal(a, b)
