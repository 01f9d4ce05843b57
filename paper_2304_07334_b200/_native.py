"""ctypes binding of libheat_b200.so (include/heat_b200.h).

The library is the only compute path: if it is missing or cannot be loaded,
``lib()`` raises — there is no CPU fallback anywhere in the product.
"""

from __future__ import annotations

import ctypes
import os

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "libheat_b200.so")

HEAT_OK = 0
HEAT_ERR_INVALID = 1
HEAT_ERR_CUDA = 2
HEAT_ERR_UNSUPPORTED = 3

MODE_EXACT = 0
MODE_HOGWILD = 1
MODE_DELTA = 2

EXPORTS = ("heat_train_range", "heat_scratch_bytes", "heat_sample_negatives",
           "heat_eval_users", "heat_apply_row_deltas", "heat_apply_row_deltas_fixed",
           "heat_epoch_pairs", "heat_aggregate_users", "heat_agg_scratch_bytes",
           "heat_exact_stats", "heat_nccl_unique_id", "heat_shard_create", "heat_shard_epoch",
           "heat_shard_last_error", "heat_shard_destroy", "heat_shard_create_host",
           "heat_shard_create_loopback",
           "heat_shard_epoch_loopback", "heat_phase_collect", "heat_phase_read",
           "heat_probe_l2_read", "heat_probe_l2_gather", "heat_last_error", "heat_version")


# heat_host_allgather_fn: int (*)(void *user, const void *in, int64_t nbytes, void *out)
HOST_ALLGATHER_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                                     ctypes.c_int64, ctypes.c_void_p)


class SgdParams(ctypes.Structure):
    _fields_ = [
        ("dim", ctypes.c_int32),
        ("n_neg", ctypes.c_int32),
        ("use_cosine", ctypes.c_int32),
        ("mode", ctypes.c_int32),
        ("lr", ctypes.c_double),
        ("l2", ctypes.c_double),
        ("mu", ctypes.c_double),
        ("theta", ctypes.c_double),
        ("stream_base", ctypes.c_uint64),
        ("window", ctypes.c_int32),
        ("flags", ctypes.c_int32),
    ]


class AggParams(ctypes.Structure):
    """heat_agg_params (include/heat_b200.h)."""
    _fields_ = [
        ("W", ctypes.c_void_p),
        ("tr_offsets", ctypes.c_void_p),
        ("tr_items", ctypes.c_void_p),
        ("gamma", ctypes.c_double),
        ("lr", ctypes.c_double),
        ("mini_batch", ctypes.c_int64),
        ("max_history", ctypes.c_int64),
        ("history_grad", ctypes.c_int32),
        ("reserved", ctypes.c_int32),
        ("accu", ctypes.c_void_p),
        ("counter", ctypes.c_void_p),
    ]


class Counters(ctypes.Structure):
    _fields_ = [
        ("loss", ctypes.c_double),
        ("degenerate", ctypes.c_int64),
        ("active", ctypes.c_int64),
        ("pairs", ctypes.c_int64),
    ]


COUNTERS_BYTES = ctypes.sizeof(Counters)


class ShardStats(ctypes.Structure):
    _fields_ = [
        ("steps", ctypes.c_int64),
        ("entries", ctypes.c_int64),
        ("exchanged_bytes", ctypes.c_int64),
        ("max_entries", ctypes.c_int64),
        ("launches", ctypes.c_int64),
    ]


class ShardRank(ctypes.Structure):
    """heat_shard_rank (include/heat_b200.h): one loopback rank's epoch inputs."""
    _fields_ = [
        ("S", ctypes.c_void_p),
        ("s_rows", ctypes.c_int64),
        ("T", ctypes.c_void_p),
        ("t_rows", ctypes.c_int64),
        ("local_users", ctypes.c_void_p),
        ("local_items", ctypes.c_void_p),
        ("pair_index", ctypes.c_void_p),
        ("step_bounds", ctypes.c_void_p),
        ("capacity", ctypes.c_int64),
        ("counters", ctypes.c_void_p),
    ]


_lib = None


class HeatError(RuntimeError):
    pass


def lib():
    """Load (never build) the native library; raise if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -m paper_2304_07334_b200.build` "
            "(or __graft_entry__.build()); there is no CPU fallback")
    L = ctypes.CDLL(LIB_PATH)
    P, i32, i64, u64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64
    L.heat_train_range.restype = ctypes.c_int
    L.heat_train_range.argtypes = [P, i64, P, i64, P, P, i64, i64, ctypes.POINTER(SgdParams), P,
                                   P, P, P, i64, P, ctypes.POINTER(AggParams), P, P]
    L.heat_scratch_bytes.restype = i64
    L.heat_scratch_bytes.argtypes = [i32, i32, i64, i64]
    L.heat_sample_negatives.restype = ctypes.c_int
    L.heat_sample_negatives.argtypes = [u64, i64, i64, i32, i64, P, P]
    L.heat_eval_users.restype = ctypes.c_int
    L.heat_eval_users.argtypes = [P, i32, P, i64, i32, P, i64, P, P, i64, P, P, i32, i32, P, P,
                                  P, P, P, P]
    L.heat_apply_row_deltas.restype = ctypes.c_int
    L.heat_apply_row_deltas.argtypes = [P, i64, i32, P, P, P, i64, i32, P]
    L.heat_apply_row_deltas_fixed.restype = ctypes.c_int
    L.heat_apply_row_deltas_fixed.argtypes = [P, i64, i32, P, P, P, i32, i64, P, P, P]
    L.heat_nccl_unique_id.restype = ctypes.c_int
    L.heat_nccl_unique_id.argtypes = [P]
    L.heat_shard_create.restype = ctypes.c_int
    L.heat_shard_create.argtypes = [i32, i32, P, i32, ctypes.POINTER(ctypes.c_void_p)]
    L.heat_shard_epoch.restype = ctypes.c_int
    L.heat_shard_epoch.argtypes = [P, P, i64, P, i64, P, P, P, P, i64, i64,
                                   ctypes.POINTER(SgdParams), P, ctypes.POINTER(ShardStats), P]
    L.heat_shard_last_error.restype = ctypes.c_char_p
    L.heat_shard_last_error.argtypes = [P]
    L.heat_shard_destroy.restype = ctypes.c_int
    L.heat_shard_destroy.argtypes = [P]
    L.heat_shard_create_host.restype = ctypes.c_int
    L.heat_shard_create_host.argtypes = [i32, i32, HOST_ALLGATHER_FN, P, i32,
                                         ctypes.POINTER(ctypes.c_void_p)]
    L.heat_shard_create_loopback.restype = ctypes.c_int
    L.heat_shard_create_loopback.argtypes = [i32, i32, P]
    L.heat_shard_epoch_loopback.restype = ctypes.c_int
    L.heat_shard_epoch_loopback.argtypes = [P, i32, P, i64, ctypes.POINTER(SgdParams), P, P]
    L.heat_epoch_pairs.restype = ctypes.c_int
    L.heat_epoch_pairs.argtypes = [P, i64, P, i64, u64, u64, u64, u64, i32, ctypes.c_uint32, P, P]
    L.heat_aggregate_users.restype = ctypes.c_int
    L.heat_aggregate_users.argtypes = [P, i64, P, P, i32, P, P, i64, ctypes.c_double, i64, P, P]
    L.heat_agg_scratch_bytes.restype = i64
    L.heat_agg_scratch_bytes.argtypes = [i32, i32]
    L.heat_exact_stats.restype = ctypes.c_int
    L.heat_exact_stats.argtypes = [P, ctypes.c_int]
    L.heat_probe_l2_read.restype = ctypes.c_int
    L.heat_probe_l2_read.argtypes = [P, i64, i32, P, P]
    L.heat_probe_l2_gather.restype = ctypes.c_int
    L.heat_probe_l2_gather.argtypes = [P, i64, i32, i32, P, P, P]
    L.heat_phase_collect.restype = ctypes.c_int
    L.heat_phase_collect.argtypes = [i32]
    L.heat_phase_read.restype = ctypes.c_int
    L.heat_phase_read.argtypes = [P, P, P, i32]
    L.heat_last_error.restype = ctypes.c_char_p
    L.heat_last_error.argtypes = []
    L.heat_version.restype = ctypes.c_int
    _lib = L
    return L


def check(rc: int) -> None:
    """Map a status code to the reference's exception types."""
    if rc == HEAT_OK:
        return
    msg = lib().heat_last_error().decode(errors="replace")
    if rc in (HEAT_ERR_INVALID, HEAT_ERR_UNSUPPORTED):
        raise ValueError(msg)
    raise HeatError(msg)
