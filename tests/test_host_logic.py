"""CPU tests of the host-side logic: data model, validation errors (raised
before any device work, like trainer.py:366-382), the sharding and
delta-exchange protocol of the multi-GPU path (gloo, world_size 2), and the
C-ABI library's exported symbols."""

import ctypes
import os
import re
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT
from paper_2304_07334_b200 import (AggregatorConfig, InitSpec, LossParams, SamplerConfig,
                                   TrainingConfig, from_user_lists, init_matrix)
from paper_2304_07334_b200 import rng as R
from paper_2304_07334_b200.dataset import epoch_pairs, from_pairs, with_universe
from paper_2304_07334_b200.parallel import delta_capacity, merge_order, shard_epoch
from workloads import CONFIGS, make_clustered, make_dataset


def test_abi_exports_every_declared_symbol():
    from paper_2304_07334_b200 import _native
    hdr = open(os.path.join(ROOT, "include", "heat_b200.h")).read()
    declared = set(re.findall(r"^\w[\w\s\*]*?\b(heat_\w+)\s*\(", hdr, re.M))
    assert declared == set(_native.EXPORTS), declared
    lib = ctypes.CDLL(_native.LIB_PATH)
    for name in declared:
        assert hasattr(lib, name), name
    assert _native.lib().heat_version() == 1
    assert _native.lib().heat_scratch_bytes(10, 32, 100, 200) >= 10 * 32 * 4 + 300 * 4


def test_abi_rejects_bad_arguments_without_a_gpu():
    from paper_2304_07334_b200 import _native as N
    L = N.lib()
    p = N.SgdParams(dim=0, n_neg=1, use_cosine=1, mode=0, lr=0.1, l2=0.0, mu=1.0, theta=0.5,
                    stream_base=0, window=0, flags=0)
    rc = L.heat_train_range(None, 1, None, 1, None, None, 0, 1, ctypes.byref(p), None,
                            None, None, None, 0, None, None, None, None)
    assert rc == N.HEAT_ERR_INVALID
    fake = ctypes.c_void_p(16)
    rc = L.heat_train_range(fake, 1, fake, 1, fake, fake, 0, 1, ctypes.byref(p), fake,
                            None, None, None, 0, None, None, None, None)
    assert rc == N.HEAT_ERR_INVALID and b"dim" in L.heat_last_error()
    p.dim, p.theta = 4, 1.5
    rc = L.heat_train_range(fake, 1, fake, 1, fake, fake, 0, 1, ctypes.byref(p), fake,
                            None, None, None, 0, None, None, None, None)
    assert rc == N.HEAT_ERR_INVALID and b"theta" in L.heat_last_error()
    with pytest.raises(ValueError):
        N.check(N.HEAT_ERR_INVALID)
    assert L.heat_sample_negatives(0, 0, 1, 0, 10, fake, None) == N.HEAT_ERR_INVALID
    assert L.heat_sample_negatives(0, 0, 1, 4, 0, fake, None) == N.HEAT_ERR_INVALID
    # aggregation: DELTA mode is unsupported, odd widths in HOGWILD mode too
    p.dim, p.theta, p.mode = 48, 0.5, N.MODE_DELTA
    agg = N.AggParams(W=16, tr_offsets=16, tr_items=16, gamma=0.5, lr=0.1, mini_batch=4,
                      max_history=10, history_grad=0, reserved=0, accu=None, counter=None)
    rc = L.heat_train_range(fake, 1, fake, 1, fake, fake, 0, 1, ctypes.byref(p), fake,
                            fake, fake, fake, 1, None, ctypes.byref(agg), None, None)
    assert rc == N.HEAT_ERR_UNSUPPORTED
    p.mode = N.MODE_HOGWILD
    rc = L.heat_train_range(fake, 1, fake, 1, fake, fake, 0, 1, ctypes.byref(p), fake,
                            None, None, None, 0, None, ctypes.byref(agg), None, None)
    assert rc == N.HEAT_ERR_UNSUPPORTED and b"dim" in L.heat_last_error()
    p.mode = N.MODE_EXACT  # EXACT aggregation needs the accumulator state
    rc = L.heat_train_range(fake, 1, fake, 1, fake, fake, 0, 1, ctypes.byref(p), fake,
                            None, None, None, 0, None, ctypes.byref(agg), None, None)
    assert rc == N.HEAT_ERR_INVALID
    assert L.heat_agg_scratch_bytes(128, 4096) >= 3 * 4096 * 128 * 4
    # multi-GPU runtime and the order-independent apply reject bad arguments
    h = ctypes.c_void_p()
    assert L.heat_shard_create(0, 0, None, 0, ctypes.byref(h)) == N.HEAT_ERR_INVALID
    assert L.heat_shard_create(2, 2, None, 0, ctypes.byref(h)) == N.HEAT_ERR_INVALID
    st = N.ShardStats()
    assert L.heat_shard_epoch(None, fake, 1, fake, 1, fake, fake, None, None, 1, 1,
                              ctypes.byref(p), fake, ctypes.byref(st), None) == N.HEAT_ERR_INVALID
    assert L.heat_apply_row_deltas_fixed(None, 1, 4, fake, fake, fake, 1, 1, fake, fake,
                                         None) == N.HEAT_ERR_INVALID
    assert L.heat_apply_row_deltas_fixed(fake, 1, 4, fake, fake, fake, 0, 1, fake, fake,
                                         None) == N.HEAT_ERR_INVALID


def test_config_validation_matches_reference():
    with pytest.raises(ValueError):
        TrainingConfig(num_negatives=0)
    with pytest.raises(ValueError):
        TrainingConfig(learning_rate=0.0)
    with pytest.raises(ValueError):
        TrainingConfig(similarity="euclid")
    with pytest.raises(ValueError):
        LossParams(mu=-1.0)
    with pytest.raises(ValueError):
        LossParams(theta=1.5)
    with pytest.raises(ValueError):
        SamplerConfig(kind="magic")
    with pytest.raises(ValueError):
        AggregatorConfig(gamma=2.0)
    with pytest.raises(ValueError):
        InitSpec(kind="normal", std=0.0)


def _small():
    train = from_user_lists({0: [1, 2], 1: [0], 3: [4, 2, 2]}, num_users=5, num_items=6)
    S = init_matrix(5, 8, InitSpec(seed=1))
    T = init_matrix(6, 8, InitSpec(seed=2))
    return train, S, T


def test_train_epoch_validates_before_touching_anything():
    from paper_2304_07334_b200.trainer import train_epoch
    train, S, T = _small()
    s0, t0 = S.values.copy(), T.values.copy()
    with pytest.raises(ValueError):
        train_epoch(S, T, train, TrainingConfig(emb_dim=16, num_negatives=2), epoch=0)
    with pytest.raises(ValueError):  # aggregator without weights
        train_epoch(S, T, train, TrainingConfig(emb_dim=8, num_negatives=2,
                                                aggregator=AggregatorConfig(enabled=True)))
    small_S = init_matrix(3, 8, InitSpec(seed=1))
    with pytest.raises(ValueError):
        train_epoch(small_S, T, train, TrainingConfig(emb_dim=8, num_negatives=2))
    with pytest.raises(ValueError):  # outside the built path: no CPU fallback
        train_epoch(S, T, train, TrainingConfig(emb_dim=8, num_negatives=2,
                                                sampler=SamplerConfig(kind="tiling")))
    empty = from_user_lists({}, num_users=5, num_items=6)
    with pytest.raises(ValueError):
        train_epoch(S, T, empty, TrainingConfig(emb_dim=8, num_negatives=2))
    assert np.array_equal(S.values, s0) and np.array_equal(T.values, t0)


def test_gpu_path_fails_loudly_without_cuda():
    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    from paper_2304_07334_b200.trainer import train_epoch
    train, S, T = _small()
    with pytest.raises(RuntimeError, match="CUDA"):
        train_epoch(S, T, train, TrainingConfig(emb_dim=8, num_negatives=2))


def test_dataset_semantics():
    s = from_user_lists({0: [3, 1, 3], 2: [0]}, num_users=3, num_items=4)
    assert s.offsets.tolist() == [0, 2, 2, 3] and s.items.tolist() == [1, 3, 0]
    with pytest.raises(ValueError):
        from_user_lists({0: [-1]}, num_users=1)
    with pytest.raises(ValueError):
        from_user_lists({5: [1]}, num_users=2)
    w = with_universe(s, 5, 9)
    assert w.num_users == 5 and w.offsets.tolist() == [0, 2, 2, 3, 3, 3]
    with pytest.raises(ValueError):
        with_universe(s, 2, 9)
    u, i = epoch_pairs(s, 7)
    assert sorted(zip(u.tolist(), i.tolist())) == [(0, 1), (0, 3), (2, 0)]
    u2, i2 = epoch_pairs(s, 7)
    assert np.array_equal(u, u2) and np.array_equal(i, i2)
    f = from_pairs(np.array([1, 0, 1]), np.array([2, 2, 2]), 2)
    assert f.offsets.tolist() == [0, 1, 2]


def test_rng_helpers():
    s0 = R.epoch_stream(3, 5)
    seq = R.SplitMix64(3, R.EPOCH_SALT, 5, 0)
    assert [seq.next_u64() for _ in range(10)] == [R.counter_draw(s0, n) for n in range(10)]
    with pytest.raises(ValueError):
        R.SplitMix64(0).below(0)
    assert R.stream_state(1, 2)[0] == np.uint64(R.derive_stream(1, 2))


def test_synthetic_workloads_hit_baseline_shapes():
    tr, te, spec = make_dataset("c1")
    assert (tr.num_users, tr.num_items, tr.num_pairs) == (1000, 2000, 20000)
    tr, te, spec = make_dataset("c2", scale=0.05)
    assert tr.num_pairs + te.num_pairs == round(1_030_000 * 0.05)
    counts = np.diff(tr.offsets)
    assert counts.min() >= 1  # at least one train item per user
    for u in range(0, tr.num_users, 97):  # distinct, sorted
        sl = tr.slice(u)
        assert np.all(np.diff(sl) > 0)
    assert set(CONFIGS) == {"c1", "c2", "c3", "c4", "c5"}
    a, b = make_clustered(50, 100, 5, 10, seed=1)
    assert a.num_pairs > 0 and b.num_pairs > 0


def test_block_parallel_generator_builds_valid_csr():
    """The scale-out generator (process pool, one stream per block, per-block
    CSR): exact interaction count, sorted distinct items per user, ids in
    range, deterministic, and the sequential path is unchanged by it."""
    tr, _, _ = make_dataset("c5", sample_users=0.0004, workers=2, users_per_block=1000)
    tr2, _, _ = make_dataset("c5", sample_users=0.0004, workers=2, users_per_block=1000)
    assert tr.num_pairs == round(500_000_000 * 0.0004)
    assert (tr.offsets == tr2.offsets).all() and (tr.items == tr2.items).all()
    assert tr.items.dtype == np.int32 and tr.items.min() >= 0 and tr.items.max() < 2_000_000
    deg = np.diff(tr.offsets)
    assert deg.sum() == tr.num_pairs and (deg >= 0).all()
    for u in np.flatnonzero(deg)[::37]:
        sl = tr.slice(u)
        assert np.all(np.diff(sl) > 0)
    seq, _, _ = make_dataset("c5", sample_users=0.0004, users_per_block=1000)
    assert seq.num_pairs == tr.num_pairs and (np.diff(seq.offsets) == deg).all()


def test_shard_epoch_partitions_pairs_by_owner():
    rng = np.random.default_rng(0)
    ep_users = rng.integers(0, 1000, 10_001).astype(np.int32)
    B = 256
    seen = np.zeros(len(ep_users), dtype=np.int64)
    for world in (1, 2, 3, 8):
        seen[:] = 0
        for r in range(world):
            mine, bounds = shard_epoch(ep_users, world, r, B)
            assert np.all(ep_users[mine] % world == r)
            assert np.all(np.diff(mine) > 0)  # epoch order kept
            assert bounds[0] == 0 and bounds[-1] == len(mine)
            for s in range(len(bounds) - 1):  # step s holds global [sB, (s+1)B)
                seg = mine[bounds[s]:bounds[s + 1]]
                assert np.all((seg >= s * B) & (seg < (s + 1) * B))
            seen[mine] += 1
        assert np.all(seen == 1)
    assert delta_capacity(100, 50, 0.0) == 100 * 51  # N + 1 per pair: never overflows
    assert delta_capacity(100, 50, 0.1) == 100 * 51


def test_merge_order_is_rank_major_stable():
    ids = torch.tensor([5, 1, 5, 0, 1, 5, 9, 9], dtype=torch.int32)
    valid = torch.tensor([1, 1, 1, 0, 1, 1, 1, 0], dtype=torch.bool)
    order = merge_order(ids, valid).tolist()
    assert [ids[i].item() for i in order[:6]] == [1, 1, 5, 5, 5, 9]
    assert order[:6] == [1, 4, 0, 2, 5, 6]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _exchange_worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2304_07334_b200.parallel import exchange_deltas, merge_order
    K = 4
    rng = np.random.default_rng(100 + rank)
    n = [3, 7][rank]  # ragged logs
    cap = 10
    ids = torch.zeros(cap, dtype=torch.int32)
    rows = torch.zeros((cap, K), dtype=torch.float32)
    ids[:n] = torch.from_numpy(rng.integers(0, 6, n).astype(np.int32))
    rows[:n] = torch.from_numpy(rng.standard_normal((n, K)).astype(np.float32))
    all_ids, all_rows, valid = exchange_deltas(ids, rows, n)
    order = merge_order(all_ids, valid)
    nv = int(valid.sum())
    T = np.zeros((6, K), dtype=np.float32)
    ids_s = all_ids[order][:nv].numpy()
    rows_s = all_rows[order][:nv].numpy()
    for j in range(nv):  # numpy stand-in for the ordered-apply kernel (checker)
        T[ids_s[j]] += rows_s[j]
    out[rank] = (T, ids[:n].numpy(), rows[:n].numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_delta_exchange_keeps_replicas_identical():
    world = 2
    port = _free_port()
    with mp.Manager() as man:
        out = man.dict()
        mp.spawn(_exchange_worker, args=(world, port, out), nprocs=world, join=True)
        res = dict(out)
    T0, T1 = res[0][0], res[1][0]
    assert T0.tobytes() == T1.tobytes()  # bit-identical replicas
    K = T0.shape[1]
    want = np.zeros_like(T0)
    for r in range(world):  # rank-major, stable by row id
        _, ids, rows = res[r]
        for j in range(len(ids)):
            want[ids[j]] += rows[j]
    assert np.allclose(T0, want, atol=1e-6)


def _owner_worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2304_07334_b200.parallel import owner_exchange
    K, rows_n = 4, 9
    T = torch.from_numpy((np.random.default_rng(7).standard_normal((rows_n, K)) * 0.1)
                         .astype(np.float32))  # the same initial replica everywhere
    logs = []
    for step in range(3):
        rng = np.random.default_rng(1000 * step + 100 + rank)
        n = [5, 11, 0][(rank + step) % 3]  # ragged logs, an empty one
        cap = 12
        ids = torch.zeros(cap, dtype=torch.int32)
        rows = torch.zeros((cap, K), dtype=torch.float32)
        ids[:n] = torch.from_numpy(rng.integers(0, rows_n, n).astype(np.int32))
        rows[:n] = torch.from_numpy((rng.standard_normal((n, K)) * 1e-3).astype(np.float32))
        owner_exchange(T, ids, rows, n)
        logs.append((ids[:n].numpy(), rows[:n].numpy()))
    out[rank] = (T.numpy().copy(), logs)
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_owner_exchange_matches_every_rank_applying_everything():
    """The persistent epoch's owner-computes exchange (row id owned by rank
    id % G, which alone sums its rows' entries in fixed point and stores the
    new rows into every replica) against applying every rank's log on every
    rank with the same fixed point: bit-identical replicas, bit-identical to
    the all-apply result, over three ragged steps (one log empty)."""
    world = 2
    port = _free_port()
    with mp.Manager() as man:
        out = man.dict()
        mp.spawn(_owner_worker, args=(world, port, out), nprocs=world, join=True)
        res = dict(out)
    T0, T1 = res[0][0], res[1][0]
    assert T0.tobytes() == T1.tobytes()
    want = (np.random.default_rng(7).standard_normal((9, 4)) * 0.1).astype(np.float32)
    for step in range(3):  # every rank applies every log: per row, one fixed-point sum
        acc = np.zeros((9, 4), dtype=np.int64)
        hit = np.zeros(9, dtype=bool)
        for r in range(world):
            ids, rows = res[r][1][step]
            for j in range(len(ids)):
                acc[ids[j]] += np.round(rows[j].astype(np.float64) * 2.0 ** 40).astype(np.int64)
                hit[ids[j]] = True
        want[hit] += (acc[hit].astype(np.float64) / 2.0 ** 40).astype(np.float32)
    assert T0.tobytes() == want.tobytes()


def test_native_epoch_shuffle_is_numpy_bit_identical():
    import time
    from paper_2304_07334_b200.dataset import epoch_pairs_numpy
    for name, scale in (("c1", 1.0), ("c2", 0.2)):
        tr, _, _ = make_dataset(name, scale=scale)
        for seed in (0, 1, 12345, R.shuffle_seed(0, 3), 2**62 + 7):
            u, i = epoch_pairs(tr, seed)
            un, inn = epoch_pairs_numpy(tr, seed)
            assert np.array_equal(u, un) and np.array_equal(i, inn)
    tiny = from_user_lists({0: [4], 2: [1, 3]}, num_users=3, num_items=5)
    for seed in range(20):
        assert [a.tolist() for a in epoch_pairs(tiny, seed)] == \
            [a.tolist() for a in epoch_pairs_numpy(tiny, seed)]
    tr, _, _ = make_dataset("c2")
    t0 = time.perf_counter(); epoch_pairs(tr, 5); t1 = time.perf_counter()
    epoch_pairs_numpy(tr, 5); t2 = time.perf_counter()
    print(f"native shuffle {1e3*(t1-t0):.1f} ms vs numpy {1e3*(t2-t1):.1f} ms")


def test_metrics_json_schema():
    """test_evaluator.py:176-181 of the reference: one JSON object per line."""
    import json
    from paper_2304_07334_b200.evaluator import MetricsReport, metrics_json
    obj = json.loads(metrics_json(3, MetricsReport(0.5, 0.25, 20, 11)))
    assert obj == {"epoch": 3, "recall@20": 0.5, "ndcg@20": 0.25, "users": 11}


def test_reference_arm_never_loads_the_product():
    """bench.py --impl reference: data from workloads.py, epoch order and the
    timed training from oracle/ — no module of the product package imported
    and libheat_b200.so never mapped (Next 1)."""
    import json
    import subprocess
    import sys
    code = (
        "import runpy, sys, json\n"
        "sys.argv = ['bench.py', '--impl', 'reference', '--config', 'c1', '--steps', '1',"
        " '--warmup', '0', '--ref-sample', '2000']\n"
        "try:\n"
        "    runpy.run_path('bench.py', run_name='__main__')\n"
        "except SystemExit:\n"
        "    pass\n"
        "mods = sorted(m for m in sys.modules if m.startswith('paper_2304_07334_b200'))\n"
        "maps = open('/proc/self/maps').read()\n"
        "print('CHECK ' + json.dumps({'mods': mods, 'so': 'libheat_b200' in maps}))\n")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True,
                         timeout=600, check=True).stdout
    lines = out.strip().splitlines()
    line = json.loads(lines[0])
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] == 0
    chk = json.loads(lines[-1][len("CHECK "):])
    assert chk == {"mods": [], "so": False}, chk
