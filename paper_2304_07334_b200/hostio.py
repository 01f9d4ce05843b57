"""Host side of the drop-in call: epoch-order prefetch and page-locked I/O.

The reference's ``train_epoch`` mutates the caller's numpy tables in place
(trainer.py:417) and builds the epoch order on the host every call
(trainer.py:390-392).  For the device path that means a host->device copy of
S, T and the pair order and a device->host copy of S and T per call.  This
module keeps that host work off the critical path:

* ``PairPrefetcher`` — after epoch e's order is produced, the orders of
  epochs e+1 .. e+DEPTH (same interaction set, same seed) are computed on
  host threads by the native shuffle (csrc/heat_host.cpp, GIL released) into
  page-locked buffers, so a training loop calling train_epoch(epoch=e+1)
  finds it ready;
* ``pin_array`` — page-locks a caller's numpy buffer once (cudaHostRegister)
  so table copies run as async DMA at full PCIe rate; registrations are kept
  in a small LRU that also holds a reference to the array, so a registered
  address can never be freed and reused behind our back.
"""

from __future__ import annotations

import os
import threading
from collections import OrderedDict

import numpy as np
import torch

from .dataset import epoch_pairs


def _train_key(train) -> tuple:
    return (id(train), id(train.items), id(train.offsets), int(train.num_pairs),
            int(train.num_users))


class PairPrefetcher:
    """One-slot look-ahead cache of epoch orders in pinned host memory."""

    def __init__(self):
        self._lock = threading.Lock()
        self._pending: dict = {}  # key -> (thread, holder)
        self._pool: list = []     # reusable pinned (users, items) buffers

    def _buffers(self, P: int):
        """(users, items, both): two views of one page-locked [2, P] block, so
        an epoch order goes to the device in a single copy."""
        with self._lock:
            for i, b in enumerate(self._pool):
                if b[0].numel() == P:
                    return self._pool.pop(i)
        pin = torch.cuda.is_available()
        both = torch.empty((2, P), dtype=torch.int32, pin_memory=pin)
        return (both[0], both[1], both)

    def release(self, bufs) -> None:
        with self._lock:
            if len(self._pool) < 6:
                self._pool.append(bufs)

    def _compute(self, train, seed: int, bufs):
        epoch_pairs(train, seed, out=(bufs[0].numpy(), bufs[1].numpy()))
        return bufs

    def get(self, train, seed: int):
        """(users, items) pinned torch tensors of the order for `seed`."""
        key = (_train_key(train), seed)
        with self._lock:
            hit = self._pending.pop(key, None)
        if hit is not None:
            th, holder = hit
            th.join()
            # the key holds ids only: reuse the prefetched order only if it was
            # computed from this very object (its arrays), never from an
            # earlier set whose ids CPython has since recycled
            src = holder.get("train")
            same = (src is not None and src[0] is train and src[1] is train.items
                    and src[2] is train.offsets)
            if "err" not in holder and same:
                return holder["bufs"]
            if "bufs" in holder:
                self.release(holder["bufs"])
        return self._compute(train, seed, self._buffers(train.num_pairs))

    # epochs computed ahead, one host thread each: the shuffle is sequential
    # (numpy's Fisher-Yates) and takes longer than a GPU epoch, so several
    # epochs are in flight at once when the host has the cores
    DEPTH = 4 if (os.cpu_count() or 1) >= 8 else 2
    MAX_PENDING = DEPTH + 1

    @classmethod
    def depth_for(cls, num_pairs: int) -> int:
        """Look-ahead for an epoch of num_pairs: the full depth while the
        pinned buffers stay small, one epoch ahead for scale-out epochs
        (500 M pairs = 4 GB of pinned order per epoch)."""
        return cls.DEPTH if num_pairs * 8 <= (512 << 20) else 1

    def prefetch(self, train, seed: int) -> None:
        key = (_train_key(train), seed)
        with self._lock:
            if key in self._pending:
                return
            stale = []
            while len(self._pending) >= self.MAX_PENDING:  # drop the oldest look-ahead
                old = next(iter(self._pending))
                stale.append(self._pending.pop(old))
        for th, holder in stale:
            th.join()
            if "bufs" in holder:
                self.release(holder["bufs"])
        # strong references to the set the order is computed from (checked by
        # identity in get())
        holder: dict = {"train": (train, train.items, train.offsets)}
        bufs = self._buffers(train.num_pairs)

        def run():
            try:
                holder["bufs"] = self._compute(train, seed, bufs)
            except BaseException as exc:  # surfaced as a miss; recomputed inline
                holder["err"] = exc

        th = threading.Thread(target=run, daemon=True)
        with self._lock:
            self._pending[key] = (th, holder)
        th.start()


PREFETCH = PairPrefetcher()

_pins: "OrderedDict[tuple, np.ndarray]" = OrderedDict()
_PIN_SLOTS = 6


def pin_array(a: np.ndarray) -> bool:
    """Page-lock `a`'s buffer (idempotent); returns whether it is pinned."""
    if not torch.cuda.is_available() or a.nbytes == 0 or not a.flags.c_contiguous:
        return False
    key = (a.ctypes.data, a.nbytes)
    if key in _pins:
        _pins.move_to_end(key)
        return True
    cudart = torch.cuda.cudart()
    rc = cudart.cudaHostRegister(a.ctypes.data, a.nbytes, 0)
    if int(rc) != 0:
        return False
    _pins[key] = a
    while len(_pins) > _PIN_SLOTS:
        (ptr, _), old = _pins.popitem(last=False)
        cudart.cudaHostUnregister(ptr)
    return True
