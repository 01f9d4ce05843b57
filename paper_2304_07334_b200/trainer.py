"""Drop-in ``train_epoch`` / ``train`` running on the B200.

Signature, validation order, report fields and error types follow
/root/reference/pkg/src/heatcf/trainer.py:385-466 (``train_epoch``) and
480-533 (``train``).  The epoch's pair order comes from the same
``epoch_pairs`` call (trainer.py:390-392); the pairs are then trained by the
CUDA kernels of csrc/ through the C ABI:

- ``num_threads == 1`` (the reference's deterministic mode) runs the EXACT
  kernel: pairs strictly in order, bit-identical S, T and loss to the
  reference (tests/test_gpu_parity.py);
- ``num_threads > 1`` (the reference's Hogwild mode) runs the throughput
  kernel: up to ``window`` pairs in flight with lock-free atomic row updates.

``configure(mode=…, window=…)`` or the env vars ``HEAT_B200_MODE``
(``exact`` | ``hogwild``) and ``HEAT_B200_WINDOW`` override the mapping.
Behaviour aggregation (SimpleX, trainer.py:148-173, 299-331) runs in both
modes: bit-identical in EXACT, in steps of ``window`` pairs with the shared W
frozen inside a step in Hogwild (csrc/heat_agg_hogwild.cu).  The tiling
sampler is outside the built path and raises ValueError (no CPU fallback).
"""

from __future__ import annotations

import ctypes
import os
import time
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native as N
from .dataset import epoch_pairs
from .device import DeviceModel
from .rng import epoch_stream, shuffle_seed

PHASE_NAMES = ("read_emb", "similarity", "loss", "gradient", "update", "aggregate")


@dataclass
class EpochReport:
    """trainer.py:90-100."""

    epoch: int
    mean_loss: float
    wall_time: float
    phase_times: dict[str, float]
    degenerate_count: int
    num_pairs: int
    num_threads: int
    active_negatives: int = 0


@dataclass
class TrainResult:
    reports: list
    evaluations: list
    final_metrics: object
    best_recall: float
    best_epoch: int


@dataclass
class GpuOptions:
    mode: str | None = None  # None: exact when num_threads == 1, else hogwild
    window: int = 0          # hogwild: pairs in flight (0 = default_window())
    fp64: bool = False       # hogwild: binary64 dot products
    device: object = None


_OPTIONS = GpuOptions(
    mode=os.environ.get("HEAT_B200_MODE") or None,
    window=int(os.environ.get("HEAT_B200_WINDOW", "0") or 0),
)


def configure(**kw) -> GpuOptions:
    """Set process-wide GPU options (mode, window, fp64, device)."""
    for k, v in kw.items():
        if not hasattr(_OPTIONS, k):
            raise TypeError(f"unknown option {k!r}")
        setattr(_OPTIONS, k, v)
    if _OPTIONS.mode not in (None, "exact", "hogwild"):
        raise ValueError(f"unknown mode {_OPTIONS.mode!r}")
    return _OPTIONS


def options() -> GpuOptions:
    return _OPTIONS


def _check_shapes(S, T, train, cfg, weights) -> None:
    """trainer.py:366-382, before any mutation."""
    if S.dim != cfg.emb_dim or T.dim != cfg.emb_dim:
        raise ValueError(
            f"matrix dims ({S.dim}, {T.dim}) do not match config emb_dim {cfg.emb_dim}")
    if S.rows < train.num_users:
        raise ValueError(f"user matrix has {S.rows} rows for {train.num_users} users")
    if T.rows < train.num_items:
        raise ValueError(f"item matrix has {T.rows} rows for {train.num_items} items")
    if cfg.aggregator.enabled:
        if weights is None:
            raise ValueError("aggregator enabled but no weight matrix given")
        if np.shape(weights) != (cfg.emb_dim, cfg.emb_dim):
            raise ValueError(
                f"aggregator weights shape {np.shape(weights)} != ({cfg.emb_dim}, {cfg.emb_dim})")


def _check_supported(cfg) -> None:
    if cfg.sampler.kind != "uniform":
        raise ValueError("the B200 path implements the uniform sampler only "
                         f"(got {cfg.sampler.kind!r}); no CPU fallback")
    resolve_mode(cfg)  # raises for combinations the device path does not implement


def _make_aggregator(model: DeviceModel, weights, train, cfg):
    from .device import DeviceAggregator
    if not cfg.aggregator.enabled:
        return None
    return DeviceAggregator(np.asarray(weights), train, cfg.aggregator, cfg.learning_rate,
                            model.device)


AGG_HOGWILD_DIMS = (16, 32, 64, 128)


def resolve_mode(cfg) -> int:
    mode = _OPTIONS.mode or ("exact" if cfg.num_threads == 1 else "hogwild")
    if cfg.aggregator.enabled and mode == "hogwild" and cfg.emb_dim not in AGG_HOGWILD_DIMS:
        # the throughput aggregator is built for these widths; otherwise the
        # deterministic kernel runs (a valid schedule of a multi-thread run)
        if _OPTIONS.mode == "hogwild":
            raise ValueError(f"hogwild aggregation supports emb_dim in {AGG_HOGWILD_DIMS}, "
                             f"got {cfg.emb_dim}; no CPU fallback")
        mode = "exact"
    return N.MODE_EXACT if mode == "exact" else N.MODE_HOGWILD


# Hogwild window when none is configured: one pair in flight per 512 pairs of
# the epoch (never fewer than the reference's thread count), capped by the
# kernels at the GPU's resident workers.  The BASELINE configs run with
# 1/815 (c2, B = 1024) and 1/1455 (c4, B = 2048) of an epoch in flight; a
# small interaction set then keeps the same staleness instead of putting a
# quarter of its epoch in flight at once (e.g. 7.7 k pairs -> 15 in flight,
# the reference's 8-thread pool runs 8).
WINDOW_PAIRS_PER_SLOT = 512


def default_window(cfg, num_pairs: int) -> int:
    if _OPTIONS.window > 0:
        return _OPTIONS.window
    return max(int(cfg.num_threads), int(num_pairs) // WINDOW_PAIRS_PER_SLOT, 1)


def sgd_params(model: DeviceModel, cfg, epoch: int, mode: int, num_pairs: int = 0) -> N.SgdParams:
    return model.params(n_neg=cfg.num_negatives, lr=cfg.learning_rate, l2=cfg.l2_reg,
                        mu=cfg.loss.mu, theta=cfg.loss.theta, cosine=cfg.similarity == "cosine",
                        mode=mode, stream_base=epoch_stream(cfg.seed, epoch),
                        window=default_window(cfg, num_pairs) if num_pairs else _OPTIONS.window,
                        fp64=_OPTIONS.fp64)


def run_epoch_on_device(model: DeviceModel, train, cfg, epoch: int, *, mode: int | None = None,
                        pairs=None, agg=None, before_read=None,
                        before_sync=None) -> tuple[EpochReport, dict]:
    """One epoch on device-resident tables; no table transfer.  `before_read`
    (optional) queues more stream work (e.g. the table write-back) ahead of
    the single synchronisation that reads the counters; `before_sync` runs
    host work while the device is busy."""
    if mode is None:
        mode = resolve_mode(cfg)
    t0 = time.perf_counter()
    if pairs is None:
        ep_users, ep_items = epoch_pairs(train, shuffle_seed(cfg.seed, epoch))
        pairs = model.upload_pairs(ep_users, ep_items)
    du, di = pairs
    npairs = int(du.shape[0])
    model.counters.reset()
    if agg is not None:
        agg.reset_epoch()  # per-epoch accumulator state (trainer.py:398-400)
    # (the throughput aggregator keeps its own step: window 0 = 4096 pairs)
    params = sgd_params(model, cfg, epoch, mode, num_pairs=npairs if agg is None else 0)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record()
    model.train_range(du, di, 0, npairs, params, agg=agg)
    ev1.record()
    model.counters.fetch()
    if before_read is not None:
        before_read()
    if before_sync is not None:
        before_sync()
    torch.cuda.current_stream(model.device).synchronize()
    c = model.counters.values()
    wall = time.perf_counter() - t0
    rep = EpochReport(epoch=epoch, mean_loss=c.loss / npairs, wall_time=wall,
                      phase_times={n: 0.0 for n in PHASE_NAMES}, degenerate_count=c.degenerate,
                      num_pairs=npairs, num_threads=cfg.num_threads, active_negatives=c.active)
    return rep, {"kernel_s": ev0.elapsed_time(ev1) / 1e3}


def train_epoch(S, T, train, cfg, weights=None, epoch: int = 0,
                collect_phases: bool = False) -> EpochReport:
    """Drop-in for heatcf.trainer.train_epoch (trainer.py:385-466).

    S.values / T.values are updated in place, like the reference.  The epoch
    order comes from the native shuffle, prefetched up to four epochs ahead on host
    thread (hostio.PairPrefetcher); the caller's tables are page-locked once
    so the per-call host<->device copies are async DMA.  wall_time spans the
    whole call.  With collect_phases the phase dict carries the reference's
    phases (trainer.py:120-331, seconds averaged over the workers as
    trainer.py:452-455 averages its threads), measured on the device with
    clock64 by the phase-instrumented kernels (heat_phase_collect): EXACT
    mode runs the serial kernel (same bits), Hogwild mode at dim 64/128 the
    register-streamed kernel with its fused phases split by where the time
    goes.  Launches without an instrumented kernel
    (other dims, the Hogwild aggregator) leave the phases at zero.
    """
    from .hostio import PREFETCH, pin_array

    _check_shapes(S, T, train, cfg, weights)
    _check_supported(cfg)
    if train.num_pairs == 0:  # dataset.py:154 raises inside epoch_pairs
        raise ValueError("training set has no pairs")
    t_start = time.perf_counter()
    model = _session_model(S.values, T.values)  # raises without CUDA: no CPU fallback
    bufs = PREFETCH.get(train, shuffle_seed(cfg.seed, epoch))
    dev = model.device
    pin_array(S.values)
    pin_array(T.values)
    model.S.copy_(torch.from_numpy(S.values), non_blocking=True)
    model.T.copy_(torch.from_numpy(T.values), non_blocking=True)
    pairs = bufs[2].to(dev, non_blocking=True)  # users and items in one copy
    du, di = pairs[0], pairs[1]
    agg = _make_aggregator(model, weights, train, cfg)

    def write_back():  # queued behind the kernel; one host sync for everything
        torch.from_numpy(S.values).copy_(model.S, non_blocking=True)
        torch.from_numpy(T.values).copy_(model.T, non_blocking=True)

    def prefetch():  # host threads produce the next orders while the GPU runs
        for ahead in range(1, PREFETCH.depth_for(train.num_pairs) + 1):
            PREFETCH.prefetch(train, shuffle_seed(cfg.seed, epoch + ahead))

    if collect_phases:
        _phase_begin()
    try:
        rep, _ = run_epoch_on_device(model, train, cfg, epoch, pairs=(du, di), agg=agg,
                                     before_read=write_back, before_sync=prefetch)
    finally:
        phases = _phase_end() if collect_phases else None
    PREFETCH.release(bufs)
    if agg is not None:  # the reference updates the shared weights in place
        np.copyto(weights, agg.W.cpu().numpy())
    t_end = time.perf_counter()
    rep.wall_time = t_end - t_start
    if phases is not None:
        rep.phase_times.update(phases)
    return rep


def _phase_begin() -> None:
    L = N.lib()
    N.check(L.heat_phase_read((ctypes.c_double * 6)(), None, None, 1))  # zero the sums
    N.check(L.heat_phase_collect(1))


def _phase_end() -> dict:
    """Seconds per phase (PHASE_NAMES order) of the launches since
    _phase_begin, averaged over the workers; collection off again."""
    L = N.lib()
    sec = (ctypes.c_double * 6)()
    workers = ctypes.c_int64(0)
    try:
        N.check(L.heat_phase_read(sec, ctypes.byref(workers), None, 1))
    finally:
        N.check(L.heat_phase_collect(0))
    return {name: float(sec[i]) for i, name in enumerate(PHASE_NAMES)}


_SESSION: dict = {}


def _session_model(S: np.ndarray, T: np.ndarray) -> DeviceModel:
    """Reusable device buffers for the drop-in call (contents are always
    overwritten from the caller's arrays, so reuse never leaks state)."""
    from .device import require_cuda
    dev = require_cuda(_OPTIONS.device)
    key = (str(dev), S.shape, T.shape)
    m = _SESSION.get(key)
    if m is None:
        _SESSION.clear()
        m = DeviceModel(S, T, dev)
        _SESSION[key] = m
    return m


def train(S, T, train_set, test_set, cfg, weights=None, *, eval_interval: int = 0, k: int = 20,
          out_dir: str | None = None, on_epoch=None, on_eval=None) -> TrainResult:
    """trainer.py:480-533 with the tables kept on the device between epochs."""
    from .embeddings import save_model
    from .evaluator import evaluate_device

    _check_shapes(S, T, train_set, cfg, weights)
    _check_supported(cfg)
    reports: list = []
    evaluations: list = []
    best = {"recall": -1.0, "epoch": -1}
    model = DeviceModel(S.values, T.values, _OPTIONS.device)
    agg = _make_aggregator(model, weights, train_set, cfg)

    def run_eval(epoch: int):
        metrics = evaluate_device(model, S, T, train_set, test_set, cfg,
                                  weights=agg.W if agg is not None else None, k=k)
        evaluations.append((epoch, metrics))
        if on_eval is not None:
            on_eval(epoch, metrics)
        if metrics.recall_at_k > best["recall"]:
            best["recall"] = metrics.recall_at_k
            best["epoch"] = epoch
            if out_dir is not None:
                model.download(S.values, T.values)
                if agg is not None:
                    np.copyto(weights, agg.W.cpu().numpy())
                save_model(f"{out_dir}/best.ckpt", S, T, weights if agg is not None else None)
        return metrics

    from .hostio import PREFETCH
    depth = PREFETCH.depth_for(train_set.num_pairs)
    for epoch in range(cfg.epochs):
        t0 = time.perf_counter()
        # the epoch order from the host prefetcher (shuffles of the next
        # epochs run on host threads while this one trains), one copy up
        bufs = PREFETCH.get(train_set, shuffle_seed(cfg.seed, epoch))
        pairs = bufs[2].to(model.device, non_blocking=True)

        def ahead(e=epoch):
            for k in range(1, min(depth, cfg.epochs - 1 - e) + 1):
                PREFETCH.prefetch(train_set, shuffle_seed(cfg.seed, e + k))

        rep, _ = run_epoch_on_device(model, train_set, cfg, epoch, pairs=(pairs[0], pairs[1]),
                                     agg=agg, before_sync=ahead)
        PREFETCH.release(bufs)
        rep.wall_time = time.perf_counter() - t0
        reports.append(rep)
        if on_epoch is not None:
            on_epoch(rep)
        if eval_interval and (epoch + 1) % eval_interval == 0:
            run_eval(epoch + 1)
    final = run_eval(cfg.epochs)
    model.download(S.values, T.values)
    if agg is not None:
        np.copyto(weights, agg.W.cpu().numpy())
    if out_dir is not None:
        save_model(f"{out_dir}/final.ckpt", S, T, weights if agg is not None else None)
    return TrainResult(reports=reports, evaluations=evaluations, final_metrics=final,
                       best_recall=best["recall"], best_epoch=best["epoch"])
