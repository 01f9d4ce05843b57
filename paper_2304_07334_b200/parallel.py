"""Multi-GPU training: users sharded, item table replicated, per-step
item-delta exchange.  The reference has no distributed
mode (PAPER.md:876 leaves multi-node as future work); this is the B200
scale-out of its Hogwild data parallelism (trainer.py:398-447).

One process per GPU (torchrun), ``torch.distributed`` over NCCL.  An epoch's
pair order is the same on every rank (same ``epoch_pairs`` seed); the global
step is ``step_pairs`` consecutive pairs (bench.py: the config's B per rank,
i.e. world * B); rank r trains the pairs of the step whose user it owns
(``u % world == r``), keyed by their GLOBAL epoch position so the negatives
equal the 1-GPU run's (heat_train_range ``pair_index``).

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


def delta_capacity(local_pairs_max: int, n_neg: int, l2: float = 0.0) -> int:
    """Entries a step can log, exactly at worst: a pair writes its positive
    and at most every one of its N negatives (all of them when theta <= 0 or
    the tables collapse, or when l2 != 0 makes negative writes dense), so
    N + 1 per pair.  The log can therefore never overflow: no entry is ever
    dropped and no replica diverges.  Memory is the price (c4, B = 2048 per
    rank: 2.1 M entries x 516 B = 1.06 GB per log slot); `check_log_memory`
    refuses an epoch that would not fit before anything is mutated."""
    return max(1, int(local_pairs_max) * (int(n_neg) + 1))


def log_bytes(capacity: int, dim: int, slots: int, world: int, gather: bool) -> int:
    """Device bytes of a rank's delta logs: `slots` rotating logs of
    `capacity` (id, row) entries, plus the gathered copies of every rank's log
    in the gather exchange."""
    per = capacity * (4 * dim + 4)
    return slots * per * (1 + (world if gather else 0))


def native_log_slots() -> int:
    """Log slots heat_shard.cu allocates: max(lag, 2) + 1, lag = HEAT_SHARD_LAG
    (1..7; unset: 2 for stream-ordered steps, 3 for the persistent epoch, so 4
    slots).  The persistent epoch also keeps `lag` fixed-point accumulation
    buffers of the item table (8 bytes per element each)."""
    import os
    lag = min(max(int(os.environ.get("HEAT_SHARD_LAG", "3")), 1), 7)
    return max(lag, 2) + 1


def check_log_memory(capacity: int, dim: int, slots: int, world: int, gather: bool,
                     device) -> None:
    """ValueError (before the epoch mutates anything) when the logs would not
    fit in 90 % of the device's free memory; a smaller exchange period
    (pairs between exchanges) shrinks them proportionally."""
    if torch.device(device).type != "cuda":
        return
    need = log_bytes(capacity, dim, slots, world, gather)
    free, _ = torch.cuda.mem_get_info(device)
    if need > 0.9 * free:
        raise ValueError(f"delta logs need {need / 2**30:.1f} GiB ({slots} slots x {capacity} "
                         f"entries x {4 * dim + 4} B{' x (1 + world) gathered' if gather else ''})"
                         f" but {free / 2**30:.1f} GiB are free: lower the exchange period")


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


FIX_SCALE = 2.0 ** 40  # the fixed point of every order-free apply (heat_shard.cu)


def owner_exchange(T: torch.Tensor, ids: torch.Tensor, rows: torch.Tensor, count,
                   group=None) -> int:
    """One step of the persistent epoch's owner-computes exchange
    (csrc/heat_hogwild_stream.cu MODE 2/3), as collectives — the mirror the
    multi-process CPU tests run.  Item row id belongs to rank id % G.  The
    logged entries are all-gathered (the kernel's owners pull only their
    partition from the peers' logs; the mirror filters), each owner sums the
    entries of ITS rows in 2^-40 fixed point (integer adds: order-free) and
    converts each touched row once, T[id] += float(sum); the owners' new rows
    are then all-gathered into every replica, so every replica holds the one
    value its owner computed.  Returns the entries this rank applied."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    all_ids, all_rows, valid = exchange_deltas(ids, rows, count, group)
    K = T.shape[1]
    mine = valid & (all_ids.to(torch.int64) % world == rank) if all_ids.numel() else valid
    mids = all_ids[mine].to(torch.int64)
    acc = torch.zeros((T.shape[0], K), dtype=torch.int64, device=T.device)
    if mids.numel():
        fixed = torch.round(all_rows[mine].to(torch.float64) * FIX_SCALE).to(torch.int64)
        acc.index_add_(0, mids, fixed)
    touched = torch.unique(mids)
    if touched.numel():
        T[touched] += (acc[touched].to(torch.float64) / FIX_SCALE).to(torch.float32)
    # the owners' new rows into every replica (padded all-gather)
    n = torch.tensor([touched.numel()], dtype=torch.int64, device=T.device)
    ns = torch.empty(world, dtype=torch.int64, device=T.device)
    _all_gather_flat(ns, n, group)
    nmax = int(ns.max())
    if nmax:
        send_ids = torch.full((nmax,), -1, dtype=torch.int64, device=T.device)
        send_rows = torch.zeros((nmax, K), dtype=T.dtype, device=T.device)
        send_ids[:touched.numel()] = touched
        send_rows[:touched.numel()] = T[touched]
        g_ids = torch.empty(world * nmax, dtype=torch.int64, device=T.device)
        g_rows = torch.empty((world * nmax, K), dtype=T.dtype, device=T.device)
        _all_gather_flat(g_ids, send_ids, group)
        _all_gather_flat(g_rows, send_rows, group)
        keep = g_ids >= 0
        T[g_ids[keep]] = g_rows[keep]
    return int(mids.numel())


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
        slots, gather = self._log_layout()
        check_log_memory(self.cap, self.model.dim, slots, self.world, gather, dev)
        self._buffers(self.cap)
        self.params = N.SgdParams.from_buffer_copy(params)
        self.params.mode = N.MODE_DELTA

    def _log_layout(self):
        """(log slots, whether every rank's log is also gathered locally)."""
        return 1, True

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


# ---- pipelined exchange ---------------------------------------------------------
#
# The step loop above synchronises the host once per step and applies the
# union on the compute stream, so the GPU idles while the host sizes and
# issues the exchange.  The pipelined driver below overlaps them:
#
#   compute stream:  kernel(s) -> log slot s%2                (DELTA mode)
#   comm stream:     all-gather counts(s) -> pinned host copy
#   host:            waits for counts(s-1) while kernel(s) runs, then issues
#   comm stream:     all-gather logs(s-1) (cmax entries per rank), fixed-point
#                    apply(s-1) -> T, concurrently with kernel(s)
#
# kernel(s) waits for apply(s-2) (its log slot and the staleness bound): it
# reads T with every union up to s-2 applied and union s-1 possibly in flight,
# a one-step staleness that Hogwild tolerates.  T changes
# only through the applies, which every rank performs on the same gathered
# logs with an order-independent sum (heat_apply_row_deltas_fixed), so the
# replicas stay bit-identical however reads and applies interleave.

@dataclass
class GatherRequest:
    """One all-gather of the pipeline: out = concat over ranks of inp, issued on
    `stream` (the driver yields these; a runner executes them)."""
    out: torch.Tensor
    inp: torch.Tensor
    stream: torch.cuda.Stream


class ProcessGroupCollective:
    """All-gathers over torch.distributed (NCCL on GPUs)."""

    def __init__(self, group=None):
        self.group = group
        self.world = dist.get_world_size(group)

    def run(self, req: GatherRequest) -> None:
        with torch.cuda.stream(req.stream):
            _all_gather_flat(req.out, req.inp, self.group)


class LocalCollective:
    """world == 1: the gather is a copy (the single-GPU sharded path)."""

    world = 1

    def run(self, req: GatherRequest) -> None:
        with torch.cuda.stream(req.stream):
            req.out.copy_(req.inp)


def run_loopback(generators) -> None:
    """Drive G logical ranks' pipelines on one GPU in lockstep: every yielded
    gather is answered with the rank-order concatenation of all ranks' inputs
    (what NCCL's all_gather returns), each rank's stream waiting for all."""
    while True:
        reqs = [next(g, None) for g in generators]
        if all(r is None for r in reqs):
            return
        if any(r is None for r in reqs):
            raise RuntimeError("logical ranks out of step")
        evs = []
        for r in reqs:
            e = torch.cuda.Event()
            e.record(r.stream)
            evs.append(e)
        for r in reqs:
            for e in evs:
                r.stream.wait_event(e)
            with torch.cuda.stream(r.stream):
                r.out.copy_(torch.cat([q.inp for q in reqs]))


class PipelinedShardTrainer(ShardedTrainer):
    """ShardedTrainer whose steps overlap the exchange with the next step's
    kernel (see the note above).  `exchange_pairs` is the global step: the
    pairs trained between two exchanges (the config's B by default)."""

    def __init__(self, model: DeviceModel, world: int, rank: int, collective=None):
        super().__init__(model, world, rank)
        self._coll = collective
        dev = model.device
        self.comm = torch.cuda.Stream(dev)
        rows, K = model.T.shape
        self.acc = torch.zeros(rows * K, dtype=torch.int64, device=dev)
        self.flags = torch.zeros(rows, dtype=torch.int32, device=dev)
        self._slots = None
        self.stats: list[StepStats] = []

    @property
    def coll(self):
        """The collective the runner uses (created on first use, so logical
        ranks driven by run_loopback need no process group)."""
        if self._coll is None:
            self._coll = LocalCollective() if self.world == 1 else ProcessGroupCollective()
        return self._coll

    def _buffers(self, cap: int):  # logs live in the two pipeline slots
        return None

    def _log_layout(self):
        return 2, True

    def _alloc_slots(self, cap: int) -> None:
        K, dev, W = self.model.dim, self.model.device, self.world
        if self._slots is not None and self._slots[0]["ids"].numel() >= cap:
            return
        self._slots = [{
            "ids": torch.empty(cap, dtype=torch.int32, device=dev),
            "rows": torch.empty((cap, K), dtype=torch.float32, device=dev),
            "cnt": torch.zeros(1, dtype=torch.int64, device=dev),
            "counts": torch.zeros(W, dtype=torch.int64, device=dev),
            "host_counts": torch.zeros(W, dtype=torch.int64).pin_memory(),
            "g_ids": torch.empty(W * cap, dtype=torch.int32, device=dev),
            "g_rows": torch.empty((W * cap, K), dtype=torch.float32, device=dev),
            "log_ready": torch.cuda.Event(), "cnt_ready": torch.cuda.Event(),
            "ex_done": torch.cuda.Event(),
        } for _ in range(2)]

    def epoch_pipeline(self, ep_users: np.ndarray, ep_items: np.ndarray,
                       params: N.SgdParams, exchange_pairs: int, prepared: bool = False):
        """Generator of the epoch's GatherRequests (a runner executes them).
        `prepared`: prepare_epoch already ran with these arguments."""
        if not prepared:
            self.prepare_epoch(ep_users, ep_items, params, exchange_pairs)
        self._alloc_slots(self.cap)
        compute = torch.cuda.current_stream(self.model.device)
        self.stats = []
        n = self.num_steps
        for s in range(n + 1):
            if s < n:
                yield from self._launch(s, compute)
            if s >= 1:
                yield from self._exchange(s - 1)
        if n:
            compute.wait_event(self._slots[(n - 1) & 1]["ex_done"])
            if n >= 2:
                compute.wait_event(self._slots[(n - 2) & 1]["ex_done"])

    def _launch(self, s: int, compute):
        sl = self._slots[s & 1]
        if s >= 2:
            compute.wait_event(sl["ex_done"])  # slot free, union(s-2) applied
        sl["cnt"].zero_()
        a, b = int(self.bounds[s]), int(self.bounds[s + 1])
        if b > a:
            self.model.train_range(self.lu, self.li, a, b, self.params,
                                   delta=(sl["ids"], sl["rows"], sl["cnt"], self.cap),
                                   pair_index=self.lp)
        sl["log_ready"].record(compute)
        self.comm.wait_event(sl["log_ready"])
        yield GatherRequest(sl["counts"], sl["cnt"], self.comm)
        with torch.cuda.stream(self.comm):
            sl["host_counts"].copy_(sl["counts"], non_blocking=True)
        sl["cnt_ready"].record(self.comm)

    def _exchange(self, t: int):
        sl = self._slots[t & 1]
        sl["cnt_ready"].synchronize()  # kernel(t+1) is already queued: the GPU stays busy
        hc = sl["host_counts"].numpy()
        cmax = int(hc.max())
        if cmax > self.cap:
            raise RuntimeError(f"delta log overflow ({cmax} > {self.cap} entries on some rank); "
                               "raise the capacity margin")
        W = self.world
        if cmax > 0:
            yield GatherRequest(sl["g_ids"][:W * cmax], sl["ids"][:cmax], self.comm)
            yield GatherRequest(sl["g_rows"][:W * cmax], sl["rows"][:cmax], self.comm)
            T = self.model.T
            rc = N.lib().heat_apply_row_deltas_fixed(
                _p(T), T.shape[0], self.model.dim, _p(sl["g_ids"]), _p(sl["g_rows"]),
                _p(sl["counts"]), W, cmax, _p(self.acc), _p(self.flags),
                ctypes.c_void_p(self.comm.cuda_stream))
            N.check(rc)
        sl["ex_done"].record(self.comm)
        n_valid = int(hc.sum())
        self.stats.append(StepStats(n_valid, n_valid * (4 * self.model.dim + 4)))

    def train_epoch(self, ep_users: np.ndarray, ep_items: np.ndarray, params: N.SgdParams,
                    step_pairs: int, prepared: bool = False) -> list[StepStats]:
        for req in self.epoch_pipeline(ep_users, ep_items, params, step_pairs, prepared):
            self.coll.run(req)
        return self.stats


class NativeShardTrainer(ShardedTrainer):
    """The production multi-GPU driver (csrc/heat_shard.cu), with its own NCCL
    communicator (unique id broadcast over the default torch.distributed
    group).  Per step: DELTA kernel on one of two alternating compute streams;
    on a top-priority comm stream, an NCCL all-gather of the 8-byte entry
    counts (the cross-rank fence) and the fused gather+apply kernels, which
    read the peers' logs over NVLink through CUDA IPC mappings.  No Python and
    no host wait between steps; kernel(s) sees every applied step up to
    s - lag (lag 3, ``HEAT_SHARD_LAG``)."""

    def __init__(self, model: DeviceModel, world: int, rank: int, group=None,
                 transport: str = "nccl"):
        super().__init__(model, world, rank, group)
        self.stats = N.ShardStats()
        if transport == "host":
            self._h = self._create_host(group)
            return
        if transport != "nccl":
            raise ValueError("transport must be 'nccl' or 'host'")
        uid = None
        if world > 1:
            buf = (ctypes.c_ubyte * 128)()
            if rank == 0:
                N.check(N.lib().heat_nccl_unique_id(buf))
            obj = [bytes(buf)]
            dist.broadcast_object_list(obj, src=0, group=group)
            uid = (ctypes.c_ubyte * 128).from_buffer_copy(obj[0])
        h = ctypes.c_void_p()
        N.check(N.lib().heat_shard_create(world, rank, uid, model.device.index or 0,
                                          ctypes.byref(h)))
        self._h = h

    def _create_host(self, group):
        """heat_shard_create_host: the runtime's collectives as torch.distributed
        all-gathers of host bytes over `group` (gloo), for ranks that share
        one GPU.  The peers' logs still travel through CUDA IPC mappings."""
        world = self.world

        def allgather(_user, src, nbytes, dst):
            try:
                mine = torch.frombuffer((ctypes.c_ubyte * nbytes).from_address(src),
                                        dtype=torch.uint8).clone()
                parts = [torch.empty(nbytes, dtype=torch.uint8) for _ in range(world)]
                dist.all_gather(parts, mine, group=group)
                flat = torch.cat(parts).numpy()  # held until the copy is done
                ctypes.memmove(dst, flat.ctypes.data, nbytes * world)
                return 0
            except Exception:  # never unwind through the C caller
                import traceback
                traceback.print_exc()
                return 1

        self._hostx = N.HOST_ALLGATHER_FN(allgather)  # keep the thunk alive
        h = ctypes.c_void_p()
        N.check(N.lib().heat_shard_create_host(world, self.rank, self._hostx, None,
                                               self.model.device.index or 0, ctypes.byref(h)))
        return h

    def _buffers(self, cap: int):  # logs live in the native runtime
        return None

    def _log_layout(self):
        import os
        gather = self.world > 1 and os.environ.get("HEAT_SHARD_EXCHANGE") == "gather"
        return native_log_slots(), gather

    def close(self) -> None:
        if getattr(self, "_h", None):
            N.lib().heat_shard_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def train_epoch(self, ep_users: np.ndarray, ep_items: np.ndarray, params: N.SgdParams,
                    step_pairs: int, prepared: bool = False) -> N.ShardStats:
        if not prepared:
            self.prepare_epoch(ep_users, ep_items, params, step_pairs)
        bounds = np.ascontiguousarray(self.bounds, dtype=np.int64)
        m = self.model
        rc = N.lib().heat_shard_epoch(
            self._h, _p(m.S), m.S.shape[0], _p(m.T), m.T.shape[0], _p(self.lu), _p(self.li),
            _p(self.lp), bounds.ctypes.data_as(ctypes.c_void_p), len(bounds) - 1, self.cap,
            ctypes.byref(self.params), m.counters.ptr(), ctypes.byref(self.stats),
            _stream(m.device))
        if rc != N.HEAT_OK:
            msg = N.lib().heat_shard_last_error(self._h).decode(errors="replace")
            raise (ValueError if rc in (N.HEAT_ERR_INVALID, N.HEAT_ERR_UNSUPPORTED)
                   else N.HeatError)(msg)
        return self.stats


class LoopbackShardGroup:
    """`world` ranks of the native runtime (csrc/heat_shard.cu) in ONE process
    on one GPU — the multi-rank step logic under test where only one device
    exists.  Each rank has its own DeviceModel (S and a T replica); the NCCL
    collectives of the per-process runtime become event-ordered copies
    (heat_shard_epoch_loopback), so nothing spins on another rank's kernel."""

    def __init__(self, models: list):
        self.models = models
        self.world = len(models)
        dev = models[0].device
        arr = (ctypes.c_void_p * self.world)()
        N.check(N.lib().heat_shard_create_loopback(self.world, dev.index or 0, arr))
        self._hs = arr
        self.stats = (N.ShardStats * self.world)()

    def close(self) -> None:
        if getattr(self, "_hs", None) is not None:
            for h in self._hs:
                if h:
                    N.lib().heat_shard_destroy(h)
            self._hs = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def train_epoch(self, ep_users: np.ndarray, ep_items: np.ndarray, params: N.SgdParams,
                    step_pairs: int):
        W = self.world
        keep, ranks = [], (N.ShardRank * W)()
        nsteps = None
        for r, m in enumerate(self.models):
            mine, bounds = shard_epoch(ep_users, W, r, step_pairs)
            dev = m.device
            lu = torch.from_numpy(np.ascontiguousarray(ep_users[mine], dtype=np.int32)).to(dev)
            li = torch.from_numpy(np.ascontiguousarray(ep_items[mine], dtype=np.int32)).to(dev)
            lp = torch.from_numpy(mine).to(dev)
            b = np.ascontiguousarray(bounds, dtype=np.int64)
            local_max = int(np.diff(b).max()) if len(b) > 1 else 0
            cap = delta_capacity(local_max, params.n_neg, params.l2)
            check_log_memory(cap, m.dim, native_log_slots(), W, False, dev)
            keep += [lu, li, lp, b]
            ranks[r] = N.ShardRank(_p(m.S), m.S.shape[0], _p(m.T), m.T.shape[0], _p(lu), _p(li),
                                   _p(lp), b.ctypes.data, cap, m.counters.ptr())
            nsteps = len(b) - 1
        q = N.SgdParams.from_buffer_copy(params)
        q.mode = N.MODE_DELTA
        rc = N.lib().heat_shard_epoch_loopback(self._hs, W, ranks, nsteps, ctypes.byref(q),
                                               self.stats, _stream(self.models[0].device))
        if rc != N.HEAT_OK:
            msg = N.lib().heat_shard_last_error(self._hs[0]).decode(errors="replace")
            raise (ValueError if rc in (N.HEAT_ERR_INVALID, N.HEAT_ERR_UNSUPPORTED)
                   else N.HeatError)(msg)
        del keep
        return list(self.stats)
