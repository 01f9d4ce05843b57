"""Seeded synthetic stand-ins for the paper's datasets.

BENCH AND TEST INPUT DATA, not product code: both bench.py arms (ours and
``--impl reference``), the tests and the golden-vector script build their
workloads here.  It is pure numpy and imports nothing from the product
package or the oracle, so the reference arm's data path never loads the
product's native library.

The public datasets (Gowalla, Yelp2018, Amazon-Books) are not
available offline.  BASELINE.json configs 2-4 carry their shapes; this module
generates interaction sets with those user/item/interaction counts:

- per-user degree d_u: geometric with mean 20 (config 1) or lognormal with
  median 20 and a sigma fitted by bisection so that sum(d_u) hits the
  interaction target exactly (configs 2-5), capped at num_items / 2;
- each user's d_u items are drawn WITHOUT replacement from a bounded
  Zipf(s) over popularity ranks (draw-until-distinct, first occurrences
  kept), and ranks map to item ids through a seeded permutation so hot rows
  are scattered across the table;
- optionally 20 % of each user's items are held out as the test split
  (int(d * f) items, at least one train item kept).

Everything is a pure function of (config, gen_seed); DESIGN.md records the
seed used by bench.py and the tests.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np



class InteractionSet:
    """Minimal CSR interaction set with the attributes the reference's
    ``InteractionSet`` exposes (dataset.py:29-52): ``items[offsets[u]:
    offsets[u+1]]`` is user u's sorted, distinct positives.  Both the product
    (duck-typed) and the reference accept it."""

    __slots__ = ("num_users", "num_items", "offsets", "items")

    def __init__(self, num_users: int, num_items: int, offsets, items):
        self.num_users, self.num_items = int(num_users), int(num_items)
        self.offsets = np.ascontiguousarray(offsets, dtype=np.int64)
        self.items = np.ascontiguousarray(items, dtype=np.int32)
        assert len(self.offsets) == self.num_users + 1
        assert self.offsets[-1] == len(self.items)

    def slice(self, user: int) -> np.ndarray:
        return self.items[self.offsets[user]:self.offsets[user + 1]]

    @property
    def num_pairs(self) -> int:
        return int(len(self.items))


def from_pairs(users, items, num_users: int, num_items: int) -> InteractionSet:
    """CSR from parallel (user, item) arrays: sorted per user, duplicates dropped."""
    key = np.unique(np.asarray(users, np.int64) * num_items + np.asarray(items, np.int64))
    u = key // num_items
    offsets = np.zeros(num_users + 1, dtype=np.int64)
    np.cumsum(np.bincount(u, minlength=num_users), out=offsets[1:])
    return InteractionSet(num_users, num_items, offsets, (key % num_items).astype(np.int32))


def init_table(rows: int, dim: int, seed: int = 0, std: float = 0.01) -> np.ndarray:
    """rows x dim float32 table drawn N(0, std) by numpy's PCG64 — the draw the
    reference's ``init_matrix(rows, dim, InitSpec(seed=seed))`` makes
    (embeddings.py:85-95), so S == T[:U] at init as with the CLI
    (cli.py:129-132)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    return rng.normal(0.0, std, size=(rows, dim)).astype(np.float32)

GEN_SEED = 12345


@dataclass(frozen=True)
class WorkloadSpec:
    name: str
    num_users: int
    num_items: int
    interactions: int
    zipf_s: float
    degree_law: str          # "geometric" | "lognormal"
    dim: int
    negatives: int
    theta: float
    mu: float
    batch: int
    learning_rate: float = 1e-3
    epochs: int = 1
    test_fraction: float = 0.0
    lognormal_median: float = 20.0
    extra: dict = field(default_factory=dict)


# BASELINE.json "configs" 1-5 (lr 1e-3 for all, SURVEY.md §8 size sheet).
CONFIGS: dict[str, WorkloadSpec] = {
    "c1": WorkloadSpec("c1", 1_000, 2_000, 20_000, 1.0, "geometric", 32, 10, 0.5, 10.0, 256),
    "c2": WorkloadSpec("c2", 30_000, 41_000, 1_030_000, 0.9, "lognormal", 64, 100, 0.9, 150.0,
                       1024, epochs=20, test_fraction=0.2),
    "c3": WorkloadSpec("c3", 32_000, 38_000, 1_560_000, 0.8, "lognormal", 64, 500, 0.9, 150.0,
                       1024),
    "c4": WorkloadSpec("c4", 53_000, 92_000, 2_980_000, 1.1, "lognormal", 128, 1000, 0.8, 300.0,
                       2048),
    "c5": WorkloadSpec("c5", 10_000_000, 2_000_000, 500_000_000, 1.0, "lognormal", 128, 1000,
                       0.8, 300.0, 8192),
}


def _fit_degrees(rng: np.random.Generator, spec: WorkloadSpec, num_users: int,
                 target: int) -> np.ndarray:
    cap = max(1, spec.num_items // 2)
    if spec.degree_law == "geometric":
        d = rng.geometric(1.0 / 20.0, size=num_users).astype(np.int64)
        d = np.clip(d, 1, cap)
    else:
        z = rng.standard_normal(num_users)
        mu = math.log(spec.lognormal_median)

        def total(sigma: float) -> int:
            return int(np.clip(np.rint(np.exp(mu + sigma * z)), 1, cap).sum())

        lo, hi = 0.0, 4.0
        for _ in range(60):
            mid = 0.5 * (lo + hi)
            if total(mid) < target:
                lo = mid
            else:
                hi = mid
        d = np.clip(np.rint(np.exp(mu + hi * z)), 1, cap).astype(np.int64)
    # exact fix-up: spread the remainder over random users within bounds
    diff = int(target - d.sum())
    while diff != 0:
        step = 1 if diff > 0 else -1
        cand = np.flatnonzero(d < cap) if step > 0 else np.flatnonzero(d > 1)
        take = rng.choice(cand, size=min(abs(diff), len(cand)), replace=False)
        d[take] += step
        diff -= step * len(take)
    return d


def _zipf_cdf(num_items: int, s: float) -> np.ndarray:
    w = 1.0 / np.power(np.arange(1, num_items + 1, dtype=np.float64), s)
    c = np.cumsum(w)
    return c / c[-1]


def _distinct_draws(rng, cdf, users_rep: np.ndarray, need: np.ndarray, num_items: int):
    """For a block of users, draw need[u] distinct Zipf ranks each.

    users_rep: local user index per slot; need: per local user counts.
    Returns (local_user, rank) arrays with exactly need[u] rows per user."""
    n_local = len(need)
    have_u = np.empty(0, np.int64)
    have_r = np.empty(0, np.int64)
    have_o = np.empty(0, np.int64)
    short = need.copy()
    order_base = 0
    factor = 1.3
    while True:
        todo = np.flatnonzero(short > 0)
        if len(todo) == 0:
            break
        m = np.ceil(short[todo] * factor).astype(np.int64) + 2
        uu = np.repeat(todo, m)
        rr = np.searchsorted(cdf, rng.random(len(uu)), side="right").astype(np.int64)
        rr = np.minimum(rr, num_items - 1)
        oo = order_base + np.arange(len(uu), dtype=np.int64)
        order_base += len(uu)
        cu = np.concatenate([have_u, uu])
        cr = np.concatenate([have_r, rr])
        co = np.concatenate([have_o, oo])
        key = cu * num_items + cr
        _, first = np.unique(key, return_index=True)
        cu, cr, co = cu[first], cr[first], co[first]
        # per user keep the first need[u] distinct ranks in draw order
        srt = np.lexsort((co, cu))
        cu, cr, co = cu[srt], cr[srt], co[srt]
        start = np.searchsorted(cu, np.arange(n_local), side="left")
        pos = np.arange(len(cu)) - start[cu]
        keep = pos < need[cu]
        have_u, have_r, have_o = cu[keep], cr[keep], co[keep]
        got = np.bincount(have_u, minlength=n_local)
        short = need - got
        factor *= 2.0
    return have_u, have_r


class _CsrBuilder:
    """Accumulates per-block (local user, item) arrays into a CSR set."""

    def __init__(self, num_users: int, num_items: int):
        self.num_users, self.num_items = num_users, num_items
        self.counts = np.zeros(num_users, dtype=np.int64)
        self.items: list[np.ndarray] = []

    def add_sorted(self, glob_users: np.ndarray, counts: np.ndarray, items: np.ndarray) -> None:
        """A block's per-user counts and its items already in CSR order."""
        if len(items):
            self.items.append(items)
        self.counts[glob_users] += counts

    def build(self) -> InteractionSet:
        offsets = np.zeros(self.num_users + 1, dtype=np.int64)
        np.cumsum(self.counts, out=offsets[1:])
        items = np.concatenate(self.items) if self.items else np.empty(0, np.int32)
        return InteractionSet(self.num_users, self.num_items, offsets, items)


_SHARED = None  # (cdf, rank_to_id, deg, num_items, tf) for forked block workers


def _split_block(rng, need, cdf, rank_to_id, num_items: int, tf: float):
    """One block of users: distinct Zipf draws, the optional per-user test
    split, each part as (counts per local user, items in CSR order)."""
    n_local = len(need)
    lu, lr = _distinct_draws(rng, cdf, None, need, num_items)
    items = rank_to_id[lr]

    def part(u, it):
        order = np.argsort(u * num_items + it, kind="stable")
        return np.bincount(u, minlength=n_local), it[order].astype(np.int32)

    if tf <= 0:
        return part(lu, items), None
    d = need[lu]
    n_test = (d * tf).astype(np.int64)
    n_test = np.where(d - n_test < 1, np.maximum(0, d - 1), n_test)
    key = rng.random(len(lu))
    srt = np.lexsort((key, lu))
    lu_s = lu[srt]
    start = np.searchsorted(lu_s, np.arange(n_local), side="left")
    rank = np.empty(len(lu), np.int64)
    rank[srt] = np.arange(len(lu)) - start[lu_s]
    is_test = rank < n_test
    return part(lu[~is_test], items[~is_test]), part(lu[is_test], items[is_test])


def _gen_block(args):
    b0, b1, seed = args
    cdf, rank_to_id, deg, num_items, tf = _SHARED
    rng = np.random.Generator(np.random.PCG64(seed))
    return b0, b1, _split_block(rng, deg[b0:b1], cdf, rank_to_id, num_items, tf)


def make_dataset(spec: WorkloadSpec | str, *, gen_seed: int = GEN_SEED,
                 test_fraction: float | None = None, users_per_block: int = 200_000,
                 scale: float = 1.0, sample_users: float | None = None, workers: int = 0):
    """(train, test, spec) for a workload.

    ``scale`` < 1 shrinks the user count and interaction target together
    (small, fast variants for tests).  ``sample_users`` = f keeps the FULL
    user universe (so S keeps its size and its random-access footprint) but
    generates interactions for a seeded random fraction f of the users only —
    the config-5 stand-in (10 M x 2 M tables, 5.1 GB + 1.0 GB, far beyond L2)
    without generating all 500 M interactions on the host.  ``workers`` > 1
    generates blocks in a process pool with one seeded stream per block (the
    full-size config 5: 500 M interactions)."""
    if isinstance(spec, str):
        spec = CONFIGS[spec]
    tf = spec.test_fraction if test_fraction is None else test_fraction
    rng = np.random.Generator(np.random.PCG64(gen_seed))
    if sample_users is not None:
        universe = spec.num_users
        num_users = max(1, int(round(universe * sample_users)))
        target = max(num_users, int(round(spec.interactions * sample_users)))
        user_ids = np.sort(rng.choice(universe, size=num_users, replace=False)).astype(np.int64)
    else:
        universe = None
        num_users = max(1, int(round(spec.num_users * scale)))
        target = max(num_users, int(round(spec.interactions * scale)))
        user_ids = None
    deg = _fit_degrees(rng, spec, num_users, target)
    rank_to_id = rng.permutation(spec.num_items).astype(np.int64)
    cdf = _zipf_cdf(spec.num_items, spec.zipf_s)
    nu = num_users if universe is None else universe
    # CSR built block by block: blocks cover increasing, disjoint user ranges
    # and a user's items are distinct by construction, so sorting each block
    # by (user, item) gives from_pairs' order without a global sort (500 M
    # interactions for config 5)
    tr = _CsrBuilder(nu, spec.num_items)
    te = _CsrBuilder(nu, spec.num_items)
    blocks = [(b0, min(num_users, b0 + users_per_block))
              for b0 in range(0, num_users, users_per_block)]
    if workers > 1:
        # scale-out path (config 5 at full size): one seeded stream per block
        # (SeedSequence.spawn), blocks generated by a process pool; a
        # different stream from the sequential path, equally a pure function
        # of (config, gen_seed)
        global _SHARED
        seeds = np.random.SeedSequence(gen_seed).spawn(len(blocks))
        _SHARED = (cdf, rank_to_id, deg, spec.num_items, tf)
        import multiprocessing as mp
        with mp.get_context("fork").Pool(workers) as pool:
            for b0, b1, parts in pool.imap(_gen_block, [(b0, b1, sd) for (b0, b1), sd in
                                                        zip(blocks, seeds)]):
                glob = (np.arange(b0, b1, dtype=np.int64) if user_ids is None
                        else user_ids[b0:b1])
                tr.add_sorted(glob, *parts[0])
                if tf > 0:
                    te.add_sorted(glob, *parts[1])
        _SHARED = None
    else:
        for b0, b1 in blocks:
            glob = (np.arange(b0, b1, dtype=np.int64) if user_ids is None else user_ids[b0:b1])
            parts = _split_block(rng, deg[b0:b1], cdf, rank_to_id, spec.num_items, tf)
            tr.add_sorted(glob, *parts[0])
            if tf > 0:
                te.add_sorted(glob, *parts[1])
    train = tr.build()
    test = te.build()
    return train, test, spec


def make_clustered(num_users: int, num_items: int, clusters: int, per_user: int, *,
                   affinity: float = 0.95, test_fraction: float = 0.2, seed: int = 0):
    """Planted-cluster data with a learnable signal (users of cluster c mostly
    interact with the items of block c).  Used by the convergence tests."""
    rng = np.random.Generator(np.random.PCG64(seed))
    block = num_items // clusters
    users = np.repeat(np.arange(num_users, dtype=np.int64), per_user)
    c = users % clusters
    lo = c * block
    hi = np.where(c == clusters - 1, num_items, lo + block)
    inside = rng.random(len(users)) < affinity
    items = np.where(inside, lo + (rng.random(len(users)) * (hi - lo)).astype(np.int64),
                     rng.integers(0, num_items, size=len(users)))
    key = np.unique(users * num_items + items)
    users, items = key // num_items, key % num_items
    r = rng.random(len(users))
    srt = np.lexsort((r, users))
    us = users[srt]
    start = np.searchsorted(us, np.arange(num_users), side="left")
    cnt = np.bincount(users, minlength=num_users)
    rank = np.empty(len(users), np.int64)
    rank[srt] = np.arange(len(users)) - start[us]
    n_test = (cnt * test_fraction).astype(np.int64)
    n_test = np.where(cnt - n_test < 1, np.maximum(0, cnt - 1), n_test)
    is_test = rank < n_test[users]
    train = from_pairs(users[~is_test], items[~is_test], num_users, num_items)
    test = from_pairs(users[is_test], items[is_test], num_users, num_items)
    return train, test
