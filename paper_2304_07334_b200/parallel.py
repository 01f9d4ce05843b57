"""Multi-GPU training: users sharded, item table replicated, per-step
item-delta exchange.  The reference has no distributed
mode (PAPER.md:876 leaves multi-node as future work); this is the B200
scale-out of its Hogwild data parallelism (trainer.py:398-447).

One process per GPU (torchrun), ``torch.distributed`` over NCCL.  An epoch's
pair order is the same on every rank (same ``epoch_pairs`` seed); the global
step is B consecutive pairs; rank r trains the pairs of the step whose user
it owns (``u % world == r``), keyed by their GLOBAL epoch position so the
negatives equal the 1-GPU run's (heat_train_range ``pair_index``).

Per step, on every rank:
  1. the throughput kernel runs in DELTA mode over the rank's pairs: user rows
     (owned by this rank only) are updated in place, item-row updates are
     logged as (row id, delta row) entries instead of applied;
  2. entry counts are all-gathered, the padded logs all-gathered (NCCL
     all_gather_into_tensor over NVLink);
  3. every replica applies the union in one deterministic order — entries
     stably sorted by row id, rank-major within a row, each row's run summed
     in that order by one warp (heat_apply_row_deltas, ordered) — so the
     item replicas stay bit-identical without a dense all-reduce.

Only rows touched in the step travel: B*(1+A) entries of 4K+4 bytes
(A = active negatives per pair), against 4*K*I bytes for a dense all-reduce.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist

from . import _native as N
from .device import DeviceModel, _p, _stream


def shard_epoch(ep_users: np.ndarray, world: int, rank: int, step_pairs: int):
    """Rank `rank`'s pairs of an epoch, in epoch order, and the step
    boundaries in its local list.

    Returns (local_pos int64[n]: global epoch positions of my pairs,
             bounds int64[steps+1]: local index where each global step starts).
    Every global position belongs to exactly one rank (owner = user % world).
    """
    ep_users = np.asarray(ep_users)
    mine = np.flatnonzero((ep_users.astype(np.int64) % world) == rank).astype(np.int64)
    n = len(ep_users)
    steps = (n + step_pairs - 1) // step_pairs
    starts = np.arange(steps + 1, dtype=np.int64) * step_pairs
    starts[-1] = n
    bounds = np.searchsorted(mine, starts, side="left").astype(np.int64)
    return mine, bounds


def delta_capacity(local_pairs_max: int, n_neg: int, l2: float, margin: int = 16) -> int:
    """Entries a step can log: the positive plus active negatives per pair
    (every negative when l2 != 0, which makes negative writes dense)."""
    per_pair = (n_neg + 1) if l2 != 0.0 else 1 + min(n_neg, margin)
    return max(1, local_pairs_max * per_pair)


def merge_order(all_ids: torch.Tensor, valid: torch.Tensor) -> torch.Tensor:
    """Deterministic application order of gathered entries: by row id, then by
    (rank, entry) position — a stable sort of the rank-major concatenation."""
    key = torch.where(valid, all_ids.to(torch.int64),
                      torch.full_like(all_ids, np.iinfo(np.int32).max, dtype=torch.int64))
    return torch.sort(key, stable=True).indices


def _all_gather_flat(out: torch.Tensor, inp: torch.Tensor, group=None) -> None:
    """all_gather_into_tensor (one NCCL call); list form for backends without it."""
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(out, inp, group=group)
    else:
        parts = list(out.chunk(dist.get_world_size(group)))
        dist.all_gather(parts, inp, group=group)


def exchange_deltas(ids: torch.Tensor, rows: torch.Tensor, count, group=None,
                    capacity: int | None = None):
    """All-gather every rank's delta log.  Returns (ids, rows, valid) of the
    rank-major concatenation, padded to world * max_count entries.

    `count` may be a host int or the kernel's device counter (int64[1]); with
    the device counter the only host synchronisation of the step is reading
    the gathered counts.  Raises if any rank's log overflowed `capacity`."""
    world = dist.get_world_size(group)
    dev = ids.device
    cnt = count if torch.is_tensor(count) else torch.tensor([count], dtype=torch.int64,
                                                              device=dev)
    counts = torch.empty(world, dtype=torch.int64, device=dev)
    _all_gather_flat(counts, cnt.reshape(1), group)
    host_counts = counts.cpu()  # the step's single host sync
    cmax = int(host_counts.max())
    if capacity is not None and cmax > capacity:
        raise RuntimeError(f"delta log overflow ({cmax} > {capacity} entries on some rank); "
                           "raise the capacity margin")
    K = rows.shape[1]
    if cmax == 0:
        z = torch.empty(0, dtype=ids.dtype, device=dev)
        return z, torch.empty((0, K), dtype=rows.dtype, device=dev), torch.empty(0, dtype=torch.bool, device=dev)
    send_ids = ids[:cmax].contiguous()
    send_rows = rows[:cmax].contiguous()
    all_ids = torch.empty(world * cmax, dtype=ids.dtype, device=dev)
    all_rows = torch.empty((world * cmax, K), dtype=rows.dtype, device=dev)
    _all_gather_flat(all_ids, send_ids, group)
    _all_gather_flat(all_rows, send_rows, group)
    pos = torch.arange(cmax, device=dev).repeat(world)
    valid = pos < counts.repeat_interleave(cmax)
    valid.n_valid = int(host_counts.sum())  # known on the host: no second sync
    return all_ids, all_rows, valid


@dataclass
class StepStats:
    entries: int
    exchanged_bytes: int


class ShardedTrainer:
    """Per-rank driver of the sharded epoch.  `model` holds full-size S and T
    on this rank's GPU (S rows of other ranks' users are never touched)."""

    def __init__(self, model: DeviceModel, world: int, rank: int, group=None):
        self.model = model
        self.world = world
        self.rank = rank
        self.group = group
        self._buf = None

    def _buffers(self, cap: int):
        K = self.model.dim
        dev = self.model.device
        if self._buf is None or self._buf[0].numel() < cap:
            self._buf = (torch.empty(cap, dtype=torch.int32, device=dev),
                         torch.empty((cap, K), dtype=torch.float32, device=dev),
                         torch.zeros(1, dtype=torch.int64, device=dev))
        return self._buf

    def apply_ordered(self, all_ids, all_rows, valid) -> None:
        if all_ids.numel() == 0:
            return
        order = merge_order(all_ids, valid)
        n_valid = getattr(valid, "n_valid", None)
        if n_valid is None:
            n_valid = int(valid.sum().item())
        ids_s = all_ids[order][:n_valid].contiguous()
        rows_s = all_rows[order][:n_valid].contiguous()
        cnt = torch.tensor([n_valid], dtype=torch.int64, device=ids_s.device)
        rc = N.lib().heat_apply_row_deltas(_p(self.model.T), self.model.T.shape[0],
                                           self.model.dim, _p(ids_s), _p(rows_s), _p(cnt),
                                           n_valid, 1, _stream(self.model.device))
        N.check(rc)

    def prepare_epoch(self, ep_users: np.ndarray, ep_items: np.ndarray, params: N.SgdParams,
                      step_pairs: int) -> None:
        """Upload this rank's shard of the epoch and size the delta log."""
        mine, bounds = shard_epoch(ep_users, self.world, self.rank, step_pairs)
        dev = self.model.device
        self.lu = torch.from_numpy(np.ascontiguousarray(ep_users[mine], dtype=np.int32)).to(dev)
        self.li = torch.from_numpy(np.ascontiguousarray(ep_items[mine], dtype=np.int32)).to(dev)
        self.lp = torch.from_numpy(mine).to(dev)
        self.bounds = bounds
        local_max = int(np.diff(bounds).max()) if len(bounds) > 1 else 0
        self.cap = delta_capacity(local_max, params.n_neg, params.l2)
        self._buffers(self.cap)
        self.params = N.SgdParams.from_buffer_copy(params)
        self.params.mode = N.MODE_DELTA

    @property
    def num_steps(self) -> int:
        return len(self.bounds) - 1

    def local_step(self, s: int, sync: bool = True):
        """Run step s on this rank's pairs; returns (ids, rows, count) of the
        log — count as a host int (sync=True) or as the device counter."""
        d_ids, d_rows, d_cnt = self._buf
        a, b = int(self.bounds[s]), int(self.bounds[s + 1])
        d_cnt.zero_()
        if b > a:
            self.model.train_range(self.lu, self.li, a, b, self.params,
                                   delta=(d_ids, d_rows, d_cnt, self.cap), pair_index=self.lp)
        if not sync:
            return d_ids, d_rows, d_cnt
        count = int(d_cnt.item())
        if count > self.cap:
            raise RuntimeError(f"delta log overflow ({count} > {self.cap} entries); "
                               "raise the capacity margin")
        return d_ids, d_rows, count

    def train_epoch(self, ep_users: np.ndarray, ep_items: np.ndarray, params: N.SgdParams,
                    step_pairs: int) -> list[StepStats]:
        """One epoch: per step, local DELTA kernel -> all-gather -> ordered apply."""
        self.prepare_epoch(ep_users, ep_items, params, step_pairs)
        stats = []
        for s in range(self.num_steps):
            d_ids, d_rows, d_cnt = self.local_step(s, sync=False)
            all_ids, all_rows, valid = exchange_deltas(d_ids, d_rows, d_cnt, self.group,
                                                       capacity=self.cap)
            self.apply_ordered(all_ids, all_rows, valid)
            stats.append(StepStats(valid.n_valid, valid.n_valid * (4 * self.model.dim + 4)))
        return stats


def gather_users(model: DeviceModel, world: int, rank: int, group=None) -> None:
    """Make every rank's S complete: each user row comes from its owner."""
    U = model.S.shape[0]
    owner = torch.arange(U, device=model.device) % world
    mask = (owner == rank).unsqueeze(1)
    part = torch.where(mask, model.S, torch.zeros_like(model.S))
    dist.all_reduce(part, group=group)
    model.S.copy_(part)
