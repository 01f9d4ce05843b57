"""Interaction sets (CSR per-user adjacency) and the epoch shuffle.

Same layout and semantics as /root/reference/pkg/src/heatcf/dataset.py:
``items[offsets[u]:offsets[u+1]]`` is user u's sorted, deduplicated positive
list (dataset.py:29-52).  ``epoch_pairs`` must produce exactly the
reference's order because the training trajectory depends on it
(dataset.py:146-158): it uses the same numpy Generator(PCG64) permutation.
Text parsing and serialisation are out of scope (host plumbing unchanged in
the reference).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class InteractionSet:
    """Compressed per-user adjacency of positive items (dataset.py:29-52)."""

    num_users: int
    num_items: int
    offsets: np.ndarray  # int64[num_users + 1]
    items: np.ndarray    # int32, sorted within each user slice

    def __post_init__(self):
        self.offsets = np.ascontiguousarray(self.offsets, dtype=np.int64)
        self.items = np.ascontiguousarray(self.items, dtype=np.int32)
        if len(self.offsets) != self.num_users + 1:
            raise ValueError("offsets length must be num_users + 1")
        if self.offsets[-1] != len(self.items):
            raise ValueError("offsets[-1] must equal len(items)")

    def slice(self, user: int) -> np.ndarray:
        return self.items[self.offsets[user]:self.offsets[user + 1]]

    @property
    def num_pairs(self) -> int:
        return int(len(self.items))


def from_user_lists(lists, num_users: int | None = None,
                    num_items: int | None = None) -> InteractionSet:
    """{user: item ids} -> InteractionSet; dedupes and sorts (dataset.py:55-78)."""
    max_user = max(lists.keys(), default=-1)
    n_users = num_users if num_users is not None else max_user + 1
    if max_user >= n_users:
        raise ValueError(f"user id {max_user} out of range for num_users={n_users}")
    if not lists:
        n_items = num_items if num_items is not None else 0
        return InteractionSet(n_users, n_items, np.zeros(n_users + 1, np.int64),
                              np.empty(0, np.int32))
    users = np.fromiter(lists.keys(), dtype=np.int64, count=len(lists))
    chunks = [np.asarray(lists[int(u)], dtype=np.int64).ravel() for u in users]
    lens = np.array([len(c) for c in chunks], dtype=np.int64)
    flat_items = np.concatenate(chunks) if chunks else np.empty(0, np.int64)
    flat_users = np.repeat(users, lens)
    return from_pairs(flat_users, flat_items, n_users, num_items)


def from_pairs(users: np.ndarray, items: np.ndarray, num_users: int,
               num_items: int | None = None) -> InteractionSet:
    """Vectorised CSR build from parallel (user, item) arrays; dedupes."""
    users = np.asarray(users, dtype=np.int64)
    items = np.asarray(items, dtype=np.int64)
    if len(items) and items.min() < 0:
        bad = int(users[np.argmin(items)])
        raise ValueError(f"negative item id for user {bad}")
    if len(users) and (users.min() < 0 or users.max() >= num_users):
        raise ValueError("user id out of range")
    max_item = int(items.max()) if len(items) else -1
    n_items = num_items if num_items is not None else max_item + 1
    if max_item >= n_items:
        raise ValueError(f"item id {max_item} out of range for num_items={n_items}")
    key = np.unique(users * (max(n_items, 1)) + items)
    u = key // max(n_items, 1)
    it = (key % max(n_items, 1)).astype(np.int32)
    counts = np.bincount(u, minlength=num_users).astype(np.int64)
    offsets = np.zeros(num_users + 1, dtype=np.int64)
    np.cumsum(counts, out=offsets[1:])
    return InteractionSet(num_users, n_items, offsets, it)


def with_universe(s: InteractionSet, num_users: int, num_items: int) -> InteractionSet:
    """Re-frame into a larger universe (dataset.py:124-131)."""
    if num_users < s.num_users or num_items < s.num_items:
        raise ValueError("universe must not shrink")
    offsets = np.zeros(num_users + 1, dtype=np.int64)
    offsets[: s.num_users + 1] = s.offsets
    offsets[s.num_users + 1:] = s.offsets[-1]
    return InteractionSet(num_users, num_items, offsets, s.items)


def epoch_pairs(train, seed: int, out=None) -> tuple[np.ndarray, np.ndarray]:
    """One epoch's (user, positive) pairs in seed order (dataset.py:146-158).

    The order is numpy's Generator(PCG64(seed)).permutation of the CSR pairs.
    With the native library present the shuffle runs in C++
    (csrc/heat_host.cpp: the same PCG64 stream and Fisher-Yates swaps, applied
    to the packed pairs; bit-identical, GIL released); `out` may supply the
    two int32 output arrays (e.g. pinned host buffers).
    """
    if train.num_pairs == 0:
        raise ValueError("training set has no pairs")
    lib = _native_lib()
    if lib is not None:
        import ctypes
        st = np.random.PCG64(seed).state
        s, inc = int(st["state"]["state"]), int(st["state"]["inc"])
        P = int(train.num_pairs)
        offsets = np.ascontiguousarray(train.offsets, dtype=np.int64)
        items = np.ascontiguousarray(train.items, dtype=np.int32)
        if out is None:
            out = (np.empty(P, dtype=np.int32), np.empty(P, dtype=np.int32))
        ou, oi = out
        m64 = (1 << 64) - 1
        rc = lib.heat_epoch_pairs(offsets.ctypes.data, int(train.num_users), items.ctypes.data, P,
                                  s >> 64, s & m64, inc >> 64, inc & m64,
                                  int(st["has_uint32"]), int(st["uinteger"]),
                                  ou.ctypes.data, oi.ctypes.data)
        if rc != 0:
            raise ValueError("inconsistent interaction set")
        return ou, oi
    return epoch_pairs_numpy(train, seed)


def _native_lib():
    try:
        from . import _native
        return _native.lib()
    except (ImportError, OSError):
        return None


def epoch_pairs_numpy(train, seed: int) -> tuple[np.ndarray, np.ndarray]:
    """The reference's construction verbatim in numpy (dataset.py:154-158)."""
    if train.num_pairs == 0:
        raise ValueError("training set has no pairs")
    counts = np.diff(train.offsets)
    users = np.repeat(np.arange(train.num_users, dtype=np.int32), counts)
    perm = np.random.Generator(np.random.PCG64(seed)).permutation(train.num_pairs)
    return users[perm], np.asarray(train.items)[perm].astype(np.int32)


def history_of(train, user: int, max_history: int) -> np.ndarray:
    if user < 0 or user >= train.num_users:
        raise ValueError(f"user {user} out of range [0, {train.num_users})")
    return train.slice(user)[:max_history]
