"""Recall@K / NDCG@K on the B200 — drop-in for heatcf.evaluator.

``evaluate`` follows /root/reference/pkg/src/heatcf/evaluator.py:113-179:
same validation and errors, users with an empty test slice left out, train
positives masked, ties toward the lower item id.  Scoring, top-k selection
and the per-user hit / DCG computation run in csrc/heat_eval.cu; the host
only builds the 1/log2(r+1) and IDCG tables with the reference's arithmetic
(evaluator.py:144-148) and sums the per-user values in user order, the same
floating-point order as evaluator.py:171-178.
"""

from __future__ import annotations

import ctypes
import json
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from .device import DeviceModel, _p, _stream, require_cuda


class EmptyTestSetError(ValueError):
    """No user has any test item; metrics are undefined."""


@dataclass(frozen=True)
class MetricsReport:
    recall_at_k: float
    ndcg_at_k: float
    k: int
    users_evaluated: int


def metrics_json(epoch: int, m: MetricsReport) -> str:
    return json.dumps({"epoch": epoch, f"recall@{m.k}": m.recall_at_k,
                       f"ndcg@{m.k}": m.ndcg_at_k, "users": m.users_evaluated})


def _weight_tables(k: int):
    w, idcg = [], []
    acc = 0.0
    for r in range(1, k + 1):
        x = 1.0 / math.log2(r + 1)
        w.append(x)
        acc += x
        idcg.append(acc)
    return np.array(w, dtype=np.float64), np.array(idcg, dtype=np.float64)


def _validate(S, T, train, test, cfg, weights):
    if test.num_users > S.rows:
        raise ValueError(f"test has {test.num_users} users but matrix {S.rows} rows")
    if max(train.num_items, test.num_items) > T.rows:
        raise ValueError("item universe exceeds item matrix rows")
    if test.num_pairs == 0:
        raise EmptyTestSetError("no user has a test item")
    agg = getattr(cfg, "aggregator", None)
    if agg is not None and agg.enabled and weights is None:
        raise ValueError("aggregator enabled but no weight matrix given")


def eval_users_device(Sdev: torch.Tensor, Tdev: torch.Tensor, users: np.ndarray, train,
                      test, k: int, cosine: bool, want_topk: bool = False):
    """Per-user (recall, ndcg[, topk]) for `users` (host int array)."""
    dev = Tdev.device
    K = int(Tdev.shape[1])
    n = len(users)
    du = torch.from_numpy(np.ascontiguousarray(users, dtype=np.int32)).to(dev)
    tr_off = torch.from_numpy(np.ascontiguousarray(train.offsets, np.int64)).to(dev)
    tr_it = torch.from_numpy(np.ascontiguousarray(train.items, np.int32)).to(dev) \
        if len(train.items) else torch.zeros(1, dtype=torch.int32, device=dev)
    te_off = torch.from_numpy(np.ascontiguousarray(test.offsets, np.int64)).to(dev)
    te_it = torch.from_numpy(np.ascontiguousarray(test.items, np.int32)).to(dev) \
        if len(test.items) else torch.zeros(1, dtype=torch.int32, device=dev)
    w, idcg = _weight_tables(k)
    dw = torch.from_numpy(w).to(dev)
    di = torch.from_numpy(idcg).to(dev)
    rec = torch.empty(n, dtype=torch.float64, device=dev)
    ndcg = torch.empty(n, dtype=torch.float64, device=dev)
    topk = torch.empty((n, k), dtype=torch.int32, device=dev) if want_topk else None
    s_f64 = 1 if Sdev.dtype == torch.float64 else 0
    rc = N.lib().heat_eval_users(_p(Sdev), s_f64, _p(Tdev), Tdev.shape[0], K, _p(du), n,
                                 _p(tr_off), _p(tr_it), train.num_users, _p(te_off), _p(te_it),
                                 k, int(bool(cosine)), _p(dw), _p(di), _p(topk), _p(rec),
                                 _p(ndcg), _stream(dev))
    N.check(rc)
    out = (rec.cpu().numpy(), ndcg.cpu().numpy())
    if want_topk:
        out = out + (topk.cpu().numpy(),)
    return out


def aggregated_queries(model: DeviceModel, train, weights, gamma: float,
                       max_history: int) -> torch.Tensor:
    """binary64 aggregated user vectors on the device (evaluator.py:91-110)."""
    dev = model.device
    W = weights if torch.is_tensor(weights) else torch.from_numpy(
        np.ascontiguousarray(weights, dtype=np.float32))
    W = W.to(dev, dtype=torch.float32).contiguous()
    tr_off = torch.from_numpy(np.ascontiguousarray(train.offsets, np.int64)).to(dev)
    items = np.ascontiguousarray(train.items, np.int32)
    tr_it = torch.from_numpy(items if len(items) else np.zeros(1, np.int32)).to(dev)
    out = torch.empty(model.S.shape, dtype=torch.float64, device=dev)
    rc = N.lib().heat_aggregate_users(_p(model.S), model.S.shape[0], _p(model.T), _p(W),
                                      model.dim, _p(tr_off), _p(tr_it), train.num_users,
                                      float(gamma), int(max_history), _p(out), _stream(dev))
    N.check(rc)
    return out


def _mean_in_order(values: np.ndarray) -> float:
    """Left-to-right binary64 sum (the reference's running `+=`,
    evaluator.py:171-178): np.cumsum accumulates sequentially, unlike
    np.sum's pairwise reduction, so the last prefix is the same float."""
    if len(values) == 0:
        return 0.0
    return float(np.cumsum(np.asarray(values, dtype=np.float64))[-1])


def evaluate_device(model: DeviceModel, S, T, train, test, cfg, weights=None, k: int = 20,
                    block_users: int = 512) -> MetricsReport:
    _validate(S, T, train, test, cfg, weights)
    if k < 1:
        raise ValueError(f"k must be >= 1, got {k}")
    similarity = getattr(cfg, "similarity", "cosine")
    counts = np.diff(test.offsets)
    users = np.flatnonzero(counts > 0).astype(np.int32)
    query = model.S
    agg = getattr(cfg, "aggregator", None)
    if agg is not None and agg.enabled:
        query = aggregated_queries(model, train, weights, agg.gamma, agg.max_history)
    rec, nd = eval_users_device(query, model.T, users, train, test, k,
                                similarity == "cosine")
    n = len(users)
    return MetricsReport(recall_at_k=_mean_in_order(rec) / n, ndcg_at_k=_mean_in_order(nd) / n,
                         k=k, users_evaluated=n)


def evaluate(S, T, train, test, cfg, weights=None, k: int = 20,
             block_users: int = 512) -> MetricsReport:
    """Drop-in for heatcf.evaluator.evaluate (evaluator.py:113-179)."""
    _validate(S, T, train, test, cfg, weights)
    model = DeviceModel(S.values, T.values)
    return evaluate_device(model, S, T, train, test, cfg, weights, k, block_users)


def topk_items(user_vec, T, exclude, k: int, similarity: str = "cosine") -> np.ndarray:
    """evaluator.py:76-88: the k items most similar to user_vec."""
    if k < 1:
        raise ValueError(f"k must be >= 1, got {k}")
    dev = require_cuda()
    u = np.asarray(user_vec, dtype=np.float64).reshape(1, -1)
    excl = np.asarray(exclude, dtype=np.int64).ravel()
    kk = min(k, T.rows - len(excl))  # evaluator.py:66-67 counts duplicates too
    if kk <= 0:
        return np.empty(0, dtype=np.int64)
    uniq = np.unique(excl).astype(np.int32)
    from .dataset import InteractionSet
    tr = InteractionSet(1, T.rows, np.array([0, len(uniq)], np.int64), uniq)
    te = InteractionSet(1, T.rows, np.array([0, 1], np.int64), np.zeros(1, np.int32))
    Sdev = torch.from_numpy(u).to(dev)
    Tdev = torch.from_numpy(np.ascontiguousarray(T.values, dtype=np.float32)).to(dev)
    _, _, top = eval_users_device(Sdev, Tdev, np.zeros(1, np.int32), tr, te, k,
                                  similarity == "cosine", want_topk=True)
    top = top[0]
    return top[top >= 0][:kk].astype(np.int64)
