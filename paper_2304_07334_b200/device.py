"""Device-resident model state and the calls into libheat_b200.so.

``DeviceModel`` owns device copies of the user table S and item table T
(float32, row-major, exactly the host layout of embeddings.py:40-61) and the
per-epoch pair order; it is the unit the drop-in ``train_epoch`` uses for one
call and that multi-epoch callers keep alive across epochs (no per-epoch
host round trip).  torch provides device memory and the stream; every byte
of compute happens in the CUDA kernels of csrc/ reached through the C ABI.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from .rng import epoch_stream


def require_cuda(device=None) -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2304_07334_b200 needs a CUDA device (no CPU fallback)")
    N.lib()  # fail loudly if the native library is missing
    if device is None:
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device(device)


def _p(t: torch.Tensor | None):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


def _stream(dev: torch.device):
    return ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)


@dataclass
class CounterValues:
    loss: float
    degenerate: int
    active: int
    pairs: int


class DeviceCounters:
    """The 32-byte heat_counters struct in device memory."""

    def __init__(self, dev: torch.device):
        self.buf = torch.zeros(N.COUNTERS_BYTES, dtype=torch.uint8, device=dev)
        self.host = torch.zeros(N.COUNTERS_BYTES, dtype=torch.uint8).pin_memory()

    def reset(self, loss: float = 0.0) -> None:
        if loss == 0.0:
            self.buf.zero_()  # stream-ordered memset, no host round trip
            return
        host = np.zeros(N.COUNTERS_BYTES, dtype=np.uint8)
        host[:8] = np.frombuffer(np.float64(loss).tobytes(), dtype=np.uint8)
        self.buf.copy_(torch.from_numpy(host))

    def fetch(self) -> None:
        """Queue the device->host copy (read with `values()` after a sync)."""
        self.host.copy_(self.buf, non_blocking=True)

    def values(self) -> CounterValues:
        h = self.host.numpy()
        loss = float(h[:8].view(np.float64)[0])
        ints = h[8:32].view(np.int64)
        return CounterValues(loss, int(ints[0]), int(ints[1]), int(ints[2]))

    def read(self) -> CounterValues:
        self.fetch()
        torch.cuda.current_stream(self.buf.device).synchronize()
        return self.values()

    def ptr(self):
        return _p(self.buf)


class DeviceModel:
    """Device copies of S and T plus the state of an epoch in flight."""

    def __init__(self, S: np.ndarray, T: np.ndarray, device=None):
        self.device = require_cuda(device)
        if S.dtype != np.float32 or T.dtype != np.float32:
            raise ValueError("embedding tables must be float32")
        if S.ndim != 2 or T.ndim != 2 or S.shape[1] != T.shape[1]:
            raise ValueError(f"table shapes {S.shape} / {T.shape} do not share a dim")
        self.dim = int(S.shape[1])
        self.S = torch.from_numpy(np.ascontiguousarray(S)).to(self.device)
        self.T = torch.from_numpy(np.ascontiguousarray(T)).to(self.device)
        self.counters = DeviceCounters(self.device)
        self._scratch = None

    # -- host sync --------------------------------------------------------
    def download(self, S_out: np.ndarray, T_out: np.ndarray) -> None:
        """Write device tables back into the caller's arrays in place."""
        torch.from_numpy(S_out).copy_(self.S)
        torch.from_numpy(T_out).copy_(self.T)

    def upload(self, S: np.ndarray, T: np.ndarray) -> None:
        self.S.copy_(torch.from_numpy(np.ascontiguousarray(S)))
        self.T.copy_(torch.from_numpy(np.ascontiguousarray(T)))

    def upload_pairs(self, ep_users: np.ndarray, ep_items: np.ndarray):
        u = torch.from_numpy(np.ascontiguousarray(ep_users, dtype=np.int32)).to(self.device)
        i = torch.from_numpy(np.ascontiguousarray(ep_items, dtype=np.int32)).to(self.device)
        return u, i

    # -- training ---------------------------------------------------------
    def scratch(self, n_neg: int) -> torch.Tensor:
        need = int(N.lib().heat_scratch_bytes(n_neg, self.dim, self.S.shape[0],
                                              self.T.shape[0]))
        if self._scratch is None or self._scratch.numel() < need:
            self._scratch = torch.empty(need, dtype=torch.uint8, device=self.device)
        return self._scratch

    def params(self, *, n_neg: int, lr: float, l2: float, mu: float, theta: float,
               cosine: bool, mode: int, stream_base: int, window: int = 0,
               fp64: bool = False) -> N.SgdParams:
        return N.SgdParams(dim=self.dim, n_neg=n_neg, use_cosine=int(bool(cosine)), mode=mode,
                           lr=lr, l2=l2, mu=mu, theta=theta, stream_base=stream_base,
                           window=window, flags=1 if fp64 else 0)

    def train_range(self, users: torch.Tensor, items: torch.Tensor, start: int, stop: int,
                    params: N.SgdParams, delta=None, pair_index: torch.Tensor | None = None,
                    stream=None, agg: "DeviceAggregator | None" = None) -> None:
        """Launch pairs [start, stop) on the current stream (asynchronous)."""
        scratch = None
        if params.mode == N.MODE_EXACT:
            scratch = self.scratch(params.n_neg)
        elif agg is not None:
            scratch = agg.work(self.dim, params.window)
        d_ids = d_rows = d_cnt = None
        cap = 0
        if delta is not None:
            d_ids, d_rows, d_cnt, cap = delta
        rc = N.lib().heat_train_range(
            _p(self.S), self.S.shape[0], _p(self.T), self.T.shape[0], _p(users), _p(items),
            start, stop, ctypes.byref(params), self.counters.ptr(), _p(d_ids), _p(d_rows),
            _p(d_cnt), cap, _p(pair_index), ctypes.byref(agg.params()) if agg else None,
            _p(scratch),
            _stream(self.device) if stream is None else ctypes.c_void_p(stream.cuda_stream))
        N.check(rc)


class DeviceAggregator:
    """Device state of the SimpleX behaviour aggregation (aggregator.py):
    the shared K x K weights W, the train CSR that holds the histories, and
    the per-epoch weight-gradient accumulator + flush counter
    (_ThreadState.agg_accu / agg_ctr, trainer.py:348-349)."""

    def __init__(self, W: np.ndarray, train, cfg_agg, lr: float, device):
        K = W.shape[0]
        self.device = device
        self.W = torch.from_numpy(np.ascontiguousarray(W, dtype=np.float32)).to(device)
        self.tr_offsets = torch.from_numpy(np.ascontiguousarray(train.offsets, np.int64)).to(device)
        items = np.ascontiguousarray(train.items, np.int32)
        self.tr_items = torch.from_numpy(items if len(items) else np.zeros(1, np.int32)).to(device)
        self.accu = torch.zeros((K, K), dtype=torch.float64, device=device)
        self.counter = torch.zeros(1, dtype=torch.int64, device=device)
        self.gamma = float(cfg_agg.gamma)
        self.lr = float(cfg_agg.learning_rate if cfg_agg.learning_rate is not None else lr)
        self.mini_batch = int(cfg_agg.mini_batch_size)
        self.max_history = int(cfg_agg.max_history)
        self.history_grad = bool(cfg_agg.history_grad)
        self._p = None
        self._work = None

    def work(self, dim: int, window: int) -> torch.Tensor:
        """Per-step buffers of the throughput aggregator (heat_agg_scratch_bytes)."""
        need = int(N.lib().heat_agg_scratch_bytes(dim, window))
        if self._work is None or self._work.numel() < need:
            self._work = torch.empty(need, dtype=torch.uint8, device=self.device)
        return self._work

    def reset_epoch(self) -> None:
        self.accu.zero_()
        self.counter.zero_()

    def params(self) -> N.AggParams:
        self._p = N.AggParams(W=self.W.data_ptr(), tr_offsets=self.tr_offsets.data_ptr(),
                              tr_items=self.tr_items.data_ptr(), gamma=self.gamma, lr=self.lr,
                              mini_batch=self.mini_batch, max_history=self.max_history,
                              history_grad=int(self.history_grad), reserved=0,
                              accu=self.accu.data_ptr(), counter=self.counter.data_ptr())
        return self._p


def stream_base(seed: int, epoch: int) -> int:
    return epoch_stream(seed, epoch)
