"""CPU oracle for the SimpleX-MF-CCL hot path — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this module, and only as the checker or
as the timed CPU baseline.  The product package (paper_2304_07334_b200)
never imports it.

Contents
- ctypes bindings to libheat_oracle.so (heat_oracle.c): a binary64
  restatement of trainer.py:103-331 (uniform sampler, no aggregator, cosine
  and dot), the SplitMix64 stream of rng.py, and the threaded epoch driver of
  trainer.py:385-466.
- ``evaluate_ref``: a numpy restatement of evaluator.py:113-179 (recall@K /
  NDCG@K with train positives masked and ties toward the lower id).

Pinning: tests/test_oracle_golden.py checks both against vectors written by
the reference itself (tests/golden/make_golden.py, run against
/root/reference in the build container).
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libheat_oracle.so")

_EPOCH_SALT = 0x45504F43
_SHUFFLE_SALT = 0x53485546

_lib = None


def build(force: bool = False) -> str:
    """Compile the oracle with its Makefile (gcc, no FMA contraction)."""
    if force or not os.path.exists(LIB_PATH) or (
        os.path.getmtime(LIB_PATH) < os.path.getmtime(os.path.join(HERE, "heat_oracle.c"))
    ):
        subprocess.run(["make", "-s", "-C", HERE] + (["-B"] if force else []), check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(LIB_PATH)
        P = ctypes.c_void_p
        i64, u64, i32, f64 = ctypes.c_int64, ctypes.c_uint64, ctypes.c_int, ctypes.c_double
        L.ho_mix64.restype = u64
        L.ho_mix64.argtypes = [u64]
        L.ho_derive_stream.restype = u64
        L.ho_derive_stream.argtypes = [u64, P, i32]
        L.ho_sample_negatives.restype = None
        L.ho_sample_negatives.argtypes = [P, i64, i32, i64, P]
        L.ho_train_range.restype = i32
        L.ho_train_range.argtypes = [P, P, i64, i32, P, P, i64, i64, P, i32, i32,
                                     f64, f64, f64, f64, P, P, P, P,
                                     P, P, P, f64, f64, i64, i64, i32, P, P]
        L.ho_train_epoch_threads.restype = i32
        L.ho_train_epoch_threads.argtypes = [P, P, i64, i32, P, P, i64, u64, i64, i32, i64,
                                             i32, i32, f64, f64, f64, f64, P, P, P]
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def mix64(x: int) -> int:
    return int(lib().ho_mix64(x & 0xFFFFFFFFFFFFFFFF))


def derive_stream(seed: int, *words: int) -> int:
    w = np.array([x & 0xFFFFFFFFFFFFFFFF for x in words], dtype=np.uint64)
    return int(lib().ho_derive_stream(seed & 0xFFFFFFFFFFFFFFFF, _ptr(w) if len(w) else None, len(w)))


def sample_negatives(state: int, npairs: int, n_neg: int, num_items: int):
    """Negatives of npairs consecutive pairs from stream state; returns (ids, new_state)."""
    st = np.array([state], dtype=np.uint64)
    out = np.empty(npairs * n_neg, dtype=np.int32)
    lib().ho_sample_negatives(_ptr(st), npairs, n_neg, num_items, _ptr(out))
    return out.reshape(npairs, n_neg), int(st[0])


@dataclass
class RangeResult:
    loss: float
    degenerate: int
    active: int
    state: int
    last_neg_ids: np.ndarray


@dataclass
class AggState:
    """Aggregator inputs + the per-thread state of trainer.py:348-349
    (accumulator, flush counter), carried across calls within an epoch."""
    W: np.ndarray                 # K x K float32, updated in place
    tr_offsets: np.ndarray
    tr_items: np.ndarray
    gamma: float = 0.5
    lr: float = 0.05
    mini_batch: int = 32
    max_history: int = 100
    history_grad: bool = False
    accu: np.ndarray | None = None
    counter: np.ndarray | None = None

    def __post_init__(self):
        K = self.W.shape[0]
        self.tr_offsets = np.ascontiguousarray(self.tr_offsets, dtype=np.int64)
        self.tr_items = np.ascontiguousarray(self.tr_items, dtype=np.int32)
        if self.accu is None:
            self.accu = np.zeros((K, K), dtype=np.float64)
        if self.counter is None:
            self.counter = np.zeros(1, dtype=np.int64)


def train_range(S: np.ndarray, T: np.ndarray, ep_users, ep_items, start: int, stop: int,
                state: int, *, n_neg: int, lr: float, l2: float = 0.0, mu: float = 1.0,
                theta: float = 0.8, cosine: bool = True, loss0: float = 0.0,
                agg: AggState | None = None) -> RangeResult:
    """Sequential pairs [start, stop) in place on S, T (trainer.py:114-297).

    ``loss0`` seeds the running loss accumulator so a sequence of calls
    reproduces the reference's per-thread ``loss_out`` bit for bit.
    """
    assert S.dtype == np.float32 and T.dtype == np.float32
    assert S.flags.c_contiguous and T.flags.c_contiguous
    ep_users = np.ascontiguousarray(ep_users, dtype=np.int32)
    ep_items = np.ascontiguousarray(ep_items, dtype=np.int32)
    st = np.array([state], dtype=np.uint64)
    loss = np.array([loss0], dtype=np.float64)
    degen = np.zeros(1, dtype=np.int64)
    active = np.zeros(1, dtype=np.int64)
    last = np.zeros(n_neg, dtype=np.int32)
    if agg is not None:
        assert agg.W.dtype == np.float32 and agg.W.flags.c_contiguous
        ag = (_ptr(agg.W), _ptr(agg.tr_offsets), _ptr(agg.tr_items), agg.gamma, agg.lr,
              agg.mini_batch, agg.max_history, int(bool(agg.history_grad)), _ptr(agg.accu),
              _ptr(agg.counter))
    else:
        ag = (None, None, None, 0.0, 0.0, 1, 0, 0, None, None)
    rc = lib().ho_train_range(_ptr(S), _ptr(T), T.shape[0], S.shape[1], _ptr(ep_users),
                              _ptr(ep_items), start, stop, _ptr(st), int(bool(cosine)), n_neg,
                              lr, l2, mu, theta, _ptr(loss), _ptr(degen), _ptr(active),
                              _ptr(last), *ag)
    if rc != 0:
        raise MemoryError("oracle scratch allocation failed")
    return RangeResult(float(loss[0]), int(degen[0]), int(active[0]), int(st[0]), last)


def epoch_pairs(offsets: np.ndarray, items: np.ndarray, num_users: int, seed: int):
    """dataset.py:146-158 restated (same numpy PCG64 permutation)."""
    counts = np.diff(offsets)
    users = np.repeat(np.arange(num_users, dtype=np.int32), counts)
    perm = np.random.Generator(np.random.PCG64(seed)).permutation(len(items))
    return users[perm], np.asarray(items)[perm].astype(np.int32)


def shuffle_seed(seed: int, epoch: int) -> int:
    return derive_stream(seed, _SHUFFLE_SALT, epoch) >> 1


def train_epoch_threads(S: np.ndarray, T: np.ndarray, ep_users, ep_items, *, seed: int,
                        epoch: int, num_threads: int, n_neg: int, lr: float, l2: float = 0.0,
                        mu: float = 1.0, theta: float = 0.8, cosine: bool = True,
                        chunk_pairs: int = 2048, npairs: int | None = None):
    """trainer.py:385-466 restated with pthreads (Hogwild for num_threads > 1).

    Returns (sum of per-thread losses, degenerate count, active negatives)."""
    ep_users = np.ascontiguousarray(ep_users, dtype=np.int32)
    ep_items = np.ascontiguousarray(ep_items, dtype=np.int32)
    n = len(ep_users) if npairs is None else npairs
    loss = np.zeros(1, dtype=np.float64)
    degen = np.zeros(1, dtype=np.int64)
    active = np.zeros(1, dtype=np.int64)
    rc = lib().ho_train_epoch_threads(_ptr(S), _ptr(T), T.shape[0], S.shape[1], _ptr(ep_users),
                                      _ptr(ep_items), n, seed, epoch, num_threads, chunk_pairs,
                                      int(bool(cosine)), n_neg, lr, l2, mu, theta, _ptr(loss),
                                      _ptr(degen), _ptr(active))
    if rc != 0:
        raise RuntimeError(f"oracle epoch failed ({rc})")
    return float(loss[0]), int(degen[0]), int(active[0])


# ---------------------------------------------------------------------------
# evaluator.py:113-179 restated in numpy
# ---------------------------------------------------------------------------

def topk_ref(scores: np.ndarray, exclude: np.ndarray, k: int) -> np.ndarray:
    """evaluator.py:61-73: mask, partition, lexsort (-score, id)."""
    scores = scores.copy()
    if len(exclude):
        scores[exclude] = -np.inf
    n_cand = len(scores) - len(exclude)
    kk = min(k, n_cand)
    if kk <= 0:
        return np.empty(0, dtype=np.int64)
    thresh = np.partition(scores, len(scores) - kk)[len(scores) - kk]
    cand = np.flatnonzero(scores >= thresh)
    order = np.lexsort((cand, -scores[cand]))
    return cand[order][:kk]


def evaluate_ref(S: np.ndarray, T: np.ndarray, train_offsets, train_items, train_num_users,
                 test_offsets, test_items, test_num_users, k: int = 20,
                 similarity: str = "cosine", block_users: int = 512,
                 return_per_user: bool = False):
    """(recall@k, ndcg@k, users) with the reference's arithmetic.

    With return_per_user, also returns {user: top-k ids} for checked users."""
    users_mat = S.astype(np.float64)
    item64 = T.astype(np.float64)
    item_norms = np.sqrt(np.einsum("ij,ij->i", item64, item64))
    tcounts = np.diff(test_offsets)
    eval_users = [u for u in range(test_num_users) if tcounts[u] > 0]
    if not eval_users:
        raise ValueError("no user has a test item")
    idcg = []
    acc = 0.0
    for r in range(1, k + 1):
        acc += 1.0 / math.log2(r + 1)
        idcg.append(acc)
    recall_sum = 0.0
    ndcg_sum = 0.0
    tops = {}
    for b in range(0, len(eval_users), block_users):
        block = eval_users[b:b + block_users]
        sub = users_mat[block]
        scores = sub @ item64.T
        if similarity == "cosine":
            unorms = np.sqrt(np.einsum("ij,ij->i", sub, sub))
            with np.errstate(invalid="ignore", divide="ignore"):
                scores = scores / (unorms[:, None] * item_norms[None, :])
            scores[unorms == 0.0, :] = 0.0
            scores[:, item_norms == 0.0] = 0.0
        for row, u in enumerate(block):
            if u < train_num_users:
                exclude = np.asarray(train_items[train_offsets[u]:train_offsets[u + 1]], np.int64)
            else:
                exclude = np.empty(0, np.int64)
            top = topk_ref(scores[row], exclude, k)
            if return_per_user:
                tops[u] = top
            test_set = set(int(i) for i in test_items[test_offsets[u]:test_offsets[u + 1]])
            dcg = 0.0
            hits = 0
            for rank, item in enumerate(top, start=1):
                if int(item) in test_set:
                    hits += 1
                    dcg += 1.0 / math.log2(rank + 1)
            recall_sum += hits / len(test_set)
            ndcg_sum += dcg / idcg[min(k, len(test_set)) - 1]
    n = len(eval_users)
    out = (recall_sum / n, ndcg_sum / n, n)
    return (out, tops) if return_per_user else out
