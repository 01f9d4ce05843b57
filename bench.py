"""Benchmark of the SimpleX-MF-CCL training step on B200.

Metric (BASELINE.json): training samples/s, one sample = one (user, positive,
N negatives) pair — the reference's ``pairs_per_s`` (bench.py:83 of heatcf).
A bench "step" is one epoch over the synthetic workload's training pairs
(the unit the reference's bench times).  Default workload: BASELINE config 4
(53k users x 92k items, 2.98M interactions, K=128, N=1000, theta 0.8, mu 300,
B=2048) — the largest configuration stated for one GPU and the one the
1->8 GPU target names — with the Hogwild kernel and B pairs in flight.
``--config c1..c5`` selects another (c2/c3 are parity-test shapes; c5 keeps
its full 10 M x 2 M tables with a 2 % user sample of its interactions).

JSON line keys beyond the base contract:
  roofline      algorithmic bytes of the fused kernel / its CUDA-event time.
                bound "l2" when S+T fit the 126 MB L2 (c1-c4; ncu: >=98.6 %
                L2 hit rate), against the L2 ceiling measured live in this run
                (best of a streaming read and random-row gathers of T in the
                kernels' access pattern); bound "hbm" otherwise (c5), against
                MEASURED_PEAKS.json hbm_gbs
  cpu_baseline  the C oracle port (restatement of trainer.py:103-466, pthreads
                Hogwild, all host cores) on a bounded sample of the same pairs
  e2e           the same metric through the public drop-in API
                ``train_epoch(S, T, train, cfg)`` with host numpy tables:
                shuffle + H2D of tables and pairs + kernel + D2H of tables

The ``--impl reference`` arm imports nothing from the product package and
never maps libheat_b200.so.  It times the UNMODIFIED reference, heatcf's own
``train_epoch`` (numba, all host cores) from baseline/_ref, on a bounded
sample of the workload cut with the oracle's numpy shuffle
(cpu_baseline.kind "reference"); if heatcf or numba cannot be imported it
falls back to the C oracle port (kind "port").
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "training samples/sec (user,pos,N negs) at 1/2/4/8 B200; % HBM roofline"


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """SM clock and throttle reasons polled (NVML, every 2 ms) during the
    timed region."""

    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
               "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80}

    def __init__(self, index: int):
        self.index = index
        self.samples: list[tuple[float, float, int]] = []
        self._stop = threading.Event()
        self._t = None

    def _sample(self):
        import pynvml
        sm = pynvml.nvmlDeviceGetClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        try:
            rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(self._h)
        except Exception:
            rs = pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(self._h)
        self.samples.append((float(sm), float(self._max), int(rs)))

    def _poll(self):
        while not self._stop.wait(0.002):
            self._sample()

    def start(self):
        """NVML is initialised here, and the first sample taken, before the
        timed region begins; a thread then polls every 2 ms."""
        try:
            import pynvml
            pynvml.nvmlInit()
            self._h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self._max = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
            self._sample()
            self._t = threading.Thread(target=self._poll, daemon=True)
            self._t.start()
        except Exception:
            self._t = None

    def stop(self) -> dict:
        if self._t is not None:
            try:
                self._sample()  # the state at the end of the timed region
            except Exception:
                pass
        self._stop.set()
        if self._t is not None:
            self._t.join(timeout=5)
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"], "samples": 0}
        reasons = sorted({n for _, _, r in self.samples for n, bit in self.REASONS.items()
                          if r & bit})
        return {"sm_mhz": statistics.median(s for s, _, _ in self.samples),
                "sm_max_mhz": max(m for _, m, _ in self.samples), "reasons": reasons,
                "samples": len(self.samples)}


def build_workload(name: str):
    """Synthetic stand-in of a BASELINE config (workloads.py; pure numpy, no
    product import).  c5 keeps its full 10 M x 2 M tables (5.1 GB + 1.0 GB:
    the HBM-bound case) with interactions generated for a seeded 2 % of the
    users (10 M of its 500 M interactions).  S and T are float32 numpy
    arrays drawn as the reference's init_matrix(InitSpec(seed=0)) draws."""
    from workloads import init_table, make_dataset
    if name == "c5":
        train, test, spec = make_dataset(name, sample_users=0.02)
    else:
        train, test, spec = make_dataset(name)
    S = init_table(train.num_users, spec.dim, seed=0)
    T = init_table(train.num_items, spec.dim, seed=0)
    return train, test, spec, S, T


def workload_config(spec, train) -> dict:
    """The `config` object both arms print (identical for the same workload)."""
    return {"workload": spec.name, "users": train.num_users, "items": train.num_items,
            "train_pairs": train.num_pairs, "dim": spec.dim, "negatives": spec.negatives,
            "theta": spec.theta, "mu": spec.mu, "batch": spec.batch, "lr": spec.learning_rate,
            "similarity": "cosine", "sampler": "uniform", "l2_reg": 0.0,
            "init": "N(0, 0.01) seed 0 (S and T)", "gen_seed": 12345}


def train_config(spec, threads: int):
    from paper_2304_07334_b200.config import LossParams, TrainingConfig
    return TrainingConfig(emb_dim=spec.dim, num_negatives=spec.negatives,
                          learning_rate=spec.learning_rate, epochs=1, num_threads=threads,
                          loss=LossParams(mu=spec.mu, theta=spec.theta), seed=0)


def algorithmic_bytes(npairs: int, K: int, N: int, active: int) -> int:
    """4K(N+2)+8 read + 4K(2+A_p) written per pair."""
    return npairs * (4 * K * (N + 2) + 8 + 4 * K * 2) + 4 * K * active


def cpu_baseline(spec, train, S0, T0, sample_pairs: int, threads: int, epoch: int = 0) -> dict:
    """Oracle port (C, pthreads Hogwild, the reference's chunk-claiming
    driver) on the first `sample_pairs` pairs of the epoch."""
    from oracle import oracle as O
    u, i = O.epoch_pairs(train.offsets, train.items, train.num_users, O.shuffle_seed(0, epoch))
    n = min(sample_pairs, len(u))
    S, T = S0.copy(), T0.copy()
    O.lib()
    t0 = time.perf_counter()
    O.train_epoch_threads(S, T, u[:n], i[:n], seed=0, epoch=epoch, num_threads=threads,
                          n_neg=spec.negatives, lr=spec.learning_rate, mu=spec.mu,
                          theta=spec.theta)
    dt = time.perf_counter() - t0
    return {"value": n / dt, "unit": "samples/s", "cores": threads, "kind": "port",
            "sample": f"first {n} pairs of epoch {epoch} of {spec.name} "
                      f"(oracle/heat_oracle.c, {threads} threads, chunk 2048)",
            "seconds": dt}


def cpu_baseline_timed(spec, train, S0, T0, threads: int, seconds: float = 10.0) -> dict:
    """cpu_baseline over a bounded sample of about `seconds` of host work:
    a probe of up to 200 k pairs sizes the sample, which then runs over consecutive
    epochs (tables carried, as a training run would) until it is used up."""
    from oracle import oracle as O
    probe = cpu_baseline(spec, train, S0, T0, 20000, threads)  # thread start-up, JIT-free
    if probe["seconds"] * 10 < seconds:  # refine on a longer probe
        probe = cpu_baseline(spec, train, S0, T0, min(200_000, train.num_pairs), threads)
    target = max(20000, int(probe["value"] * seconds))
    S, T = S0.copy(), T0.copy()
    done, dt, e = 0, 0.0, 0
    while done < target:
        u, i = O.epoch_pairs(train.offsets, train.items, train.num_users, O.shuffle_seed(0, e))
        n = min(target - done, len(u))
        t0 = time.perf_counter()
        O.train_epoch_threads(S, T, u[:n], i[:n], seed=0, epoch=e, num_threads=threads,
                              n_neg=spec.negatives, lr=spec.learning_rate, mu=spec.mu,
                              theta=spec.theta)
        dt += time.perf_counter() - t0
        done += n
        e += 1
    full, rest = divmod(done, train.num_pairs)
    what = (f"{full} epoch(s) + {rest} pairs" if full else f"first {rest} pairs of epoch 0")
    return {"value": done / dt, "unit": "samples/s", "cores": threads, "kind": "port",
            "sample": f"{done} pairs = {what} of {spec.name}, {dt:.1f} s "
                      f"(oracle/heat_oracle.c, {threads} threads, chunk 2048)",
            "seconds": dt}


def _heatcf():
    """The UNMODIFIED reference package (heatcf: Python + numba, installed by
    build() into baseline/_ref, which travels to the GPU box) or None when it
    or numba cannot be imported.  Nothing of the product is involved."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if os.environ.get("HEAT_BENCH_REF") == "port" or \
            not os.path.isdir(os.path.join(ref, "heatcf")):
        return None
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    sys.dont_write_bytecode = True
    try:
        import numba  # noqa: F401
        if ref not in sys.path:
            sys.path.insert(0, ref)
        import heatcf.dataset
        import heatcf.embeddings
        import heatcf.trainer
        return heatcf
    except Exception as exc:  # fall back to the C port, and say so
        print(f"[bench] heatcf not usable ({exc!r}); reference arm = the C port",
              file=sys.stderr)
        return None


def heatcf_sample(H, spec, train, sample_pairs: int):
    """A bounded sample of the workload as a heatcf InteractionSet: the first
    `sample_pairs` pairs of epoch 0's order over the SAME user and item
    universe, so a pair costs what it costs in the full epoch (same tables,
    N, K, chunk size).  Built with numpy from the oracle's shuffle (test
    infrastructure, allowed in this arm)."""
    from oracle import oracle as O
    u, i = O.epoch_pairs(train.offsets, train.items, train.num_users, O.shuffle_seed(0, 0))
    n = min(sample_pairs, len(u))
    u, i = u[:n].astype(np.int64), i[:n].astype(np.int32)
    order = np.lexsort((i, u))
    offsets = np.zeros(train.num_users + 1, dtype=np.int64)
    np.cumsum(np.bincount(u, minlength=train.num_users), out=offsets[1:])
    return H.dataset.InteractionSet(train.num_users, train.num_items, offsets, i[order])


def run_reference_heatcf(H, args):
    """`--impl reference`, the reference itself: heatcf.trainer.train_epoch
    (trainer.py:385-466: the threaded Hogwild driver over the numba chunk
    loop) with every host core, each step one epoch over a bounded sample of
    the workload; value = heatcf's own pairs_per_s (bench.py:75-84:
    num_pairs / EpochReport.wall_time, i.e. without the shuffle)."""
    train, _, spec, S, T = build_workload(args.config)
    threads = os.cpu_count() or 1
    sample = args.ref_sample or {"c1": 20000, "c2": 2_000_000, "c3": 600_000, "c4": 200_000,
                                 "c5": 100_000}[spec.name]
    sub = heatcf_sample(H, spec, train, sample)
    cfg = H.trainer.TrainingConfig(
        emb_dim=spec.dim, num_negatives=spec.negatives, learning_rate=spec.learning_rate,
        epochs=1, num_threads=threads, similarity="cosine",
        loss=H.trainer.LossParams(mu=spec.mu, theta=spec.theta), seed=0, l2_reg=0.0,
        chunk_pairs=2048)
    Sm, Tm = H.embeddings.EmbeddingMatrix(S.copy()), H.embeddings.EmbeddingMatrix(T.copy())
    small = heatcf_sample(H, spec, train, min(sample, 4096 * threads))
    for w in range(max(args.warmup, 1)):  # (the first call also JIT-compiles the chunk loop)
        H.trainer.train_epoch(Sm, Tm, small, cfg, epoch=w)
    vals, secs = [], []
    for s in range(args.steps):
        r = H.trainer.train_epoch(Sm, Tm, sub, cfg, epoch=args.warmup + s)
        vals.append(r.num_pairs)
        secs.append(r.wall_time)
    v = float(np.sum(vals) / np.sum(secs))  # heatcf bench: num_pairs / mean epoch time
    what = (f"{sub.num_pairs} pairs = the first {sub.num_pairs} pairs of epoch 0 of {spec.name} "
            f"as one heatcf epoch ({float(np.mean(secs)):.1f} s; heatcf.trainer."
            f"train_epoch, numba, {threads} threads, chunk 2048)")
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "samples/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": float(np.mean(secs)) * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(spec, train),
            "run": {"mode": "hogwild (host threads)", "threads": threads,
                    "step": "one heatcf epoch over a bounded sample (cpu_baseline.sample)",
                    "code": "heatcf.trainer.train_epoch from baseline/_ref (unmodified)"},
            "cpu_baseline": {"value": v, "unit": "samples/s", "cores": threads,
                             "kind": "reference", "sample": what},
            "e2e": {"value": v, "unit": "samples/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    H = _heatcf()
    if H is not None:
        return run_reference_heatcf(H, args)
    train, _, spec, S, T = build_workload(args.config)
    threads = os.cpu_count() or 1
    sample = args.ref_sample or {"c1": 20000, "c2": 400_000, "c3": 100_000, "c4": 60_000,
                                 "c5": 40_000}[spec.name]
    for w in range(args.warmup):
        cpu_baseline(spec, train, S, T, min(sample, 20000), threads, epoch=w)
    vals = []
    secs = []
    for s in range(args.steps):
        r = cpu_baseline(spec, train, S, T, sample, threads, epoch=args.warmup + s)
        vals.append(r["value"])
        secs.append(r["seconds"])
    v = float(np.mean(vals))
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "samples/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": float(np.mean(secs)) * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(spec, train),
            "run": {"mode": "hogwild (host threads)", "threads": threads,
                    "step": "a bounded sample of one epoch (cpu_baseline.sample)"},
            "cpu_baseline": {"value": v, "unit": "samples/s", "cores": threads, "kind": "port",
                             "sample": r["sample"]},
            "e2e": {"value": v, "unit": "samples/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


def _ncu_traffic(config: str):
    """DRAM bytes per launch of the Hogwild kernel from the committed ncu
    summary (profiles/ncu_<config>.json, written from an `ncu --set full`
    capture of this bench command), or None."""
    path = os.path.join(ROOT, "profiles", f"ncu_{config}.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return d
    except Exception:
        return None


L2_BYTES = 126 * 1024 * 1024


def l2_probe(dev, table_bytes: int, T=None) -> dict:
    """The L2 read ceiling measured live on this GPU, the best of:
    * "48MB" / "tables": heat_probe_l2_read streaming a 48 MB buffer (and one
      the size of S+T) 50 times after a warming pass;
    * "gather": heat_probe_l2_gather, random rows of the item table T itself
      in the training kernels' access pattern (8 lanes x 16 B per row) with no
      arithmetic — random 512-byte gathers sustain MORE than the streaming
      read on B200 (r02_gather_ceiling.txt), so it is the honest ceiling of a
      gather-bound kernel;
    each timed with CUDA events on the launching stream, best of 5 runs."""
    import ctypes

    import torch

    from paper_2304_07334_b200 import _native as N
    L = N.lib()
    stream = torch.cuda.current_stream(dev)
    sink = torch.zeros(1, dtype=torch.float32, device=dev)
    out = {}
    sizes = {"48MB": 48 * 1024 * 1024}
    if table_bytes < L2_BYTES * 0.9:
        sizes["tables"] = max(4 * 1024 * 1024, int(table_bytes))
    for name, nbytes in sizes.items():
        buf = torch.ones(nbytes // 4, dtype=torch.float32, device=dev)
        best = 0.0
        for _ in range(5):
            N.check(L.heat_probe_l2_read(buf.data_ptr(), buf.numel(), 1, sink.data_ptr(),
                                         ctypes.c_void_p(stream.cuda_stream)))
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            N.check(L.heat_probe_l2_read(buf.data_ptr(), buf.numel(), 50, sink.data_ptr(),
                                         ctypes.c_void_p(stream.cuda_stream)))
            e1.record(stream)
            e1.synchronize()
            best = max(best, buf.numel() * 4.0 * 50 / (e0.elapsed_time(e1) * 1e-3) / 1e9)
        out[name] = best
        del buf
    if T is not None and T.shape[1] in (64, 128):
        rows_read = ctypes.c_int64(0)
        best = 0.0
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            N.check(L.heat_probe_l2_gather(T.data_ptr(), T.shape[0], T.shape[1], 200,
                                           sink.data_ptr(), ctypes.byref(rows_read),
                                           ctypes.c_void_p(stream.cuda_stream)))
            e1.record(stream)
            e1.synchronize()
            best = max(best, rows_read.value * T.shape[1] * 4.0 /
                       (e0.elapsed_time(e1) * 1e-3) / 1e9)
        out["gather"] = best
    return out


def shard_lag(persistent: bool) -> int:
    """The staleness bound heat_shard.cu runs with (HEAT_SHARD_LAG, else 3 for
    both the persistent epoch and the stream-ordered steps)."""
    v = os.environ.get("HEAT_SHARD_LAG")
    return min(max(int(v), 1), 7 if persistent else 3) if v else 3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20, help="timed epochs")
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c4")
    ap.add_argument("--mode", default="hogwild", choices=["hogwild", "exact"])
    ap.add_argument("--window", type=int, default=0, help="pairs in flight (0: config batch)")
    ap.add_argument("--fp64", action="store_true")
    ap.add_argument("--sharded", action="store_true", help="user-sharded path even at N=1")
    ap.add_argument("--shard-driver", choices=("native", "python"), default="native",
                    help="sharded path: step scheduler (native C++ runtime or the Python "
                         "reference pipeline)")
    ap.add_argument("--exchange-pairs", type=int, default=0,
                    help="sharded path: global pairs between item-delta exchanges "
                         "(default: the config's batch B per rank, i.e. B * world)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=10.0,
                    help="host seconds for each cpu_baseline sample (16 threads, 1 thread)")
    ap.add_argument("--ref-sample", type=int, default=0)
    ap.add_argument("--e2e-steps", type=int, default=20)
    args = ap.parse_args()
    args.e2e_steps = max(0, args.e2e_steps)
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    from paper_2304_07334_b200 import _native as N
    from paper_2304_07334_b200.dataset import epoch_pairs
    from paper_2304_07334_b200.device import DeviceModel
    from paper_2304_07334_b200.rng import epoch_stream, shuffle_seed
    from paper_2304_07334_b200.trainer import configure, train_epoch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    sharded = world > 1 or args.sharded

    train, test, spec, S, T = build_workload(args.config)
    window = args.window or spec.batch
    mode = N.MODE_HOGWILD if args.mode == "hogwild" else N.MODE_EXACT
    K, NN = spec.dim, spec.negatives
    total_epochs = args.warmup + args.steps
    npairs = train.num_pairs
    model = DeviceModel(S, T, dev)
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)

    def params(e):
        return model.params(n_neg=NN, lr=spec.learning_rate, l2=0.0, mu=spec.mu,
                            theta=spec.theta, cosine=True, mode=mode,
                            stream_base=epoch_stream(0, e), window=window, fp64=args.fp64)

    launches_per_epoch = 1
    if not sharded:
        pairs_dev = []
        for e in range(total_epochs):  # inputs resident in HBM before timing
            u, i = epoch_pairs(train, shuffle_seed(0, e))
            pairs_dev.append(model.upload_pairs(u, i))

        def one_epoch(e):
            model.counters.reset()
            flush.zero_()  # L2 flush between steps, outside the timed region
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ev0.record(stream)
            du, di = pairs_dev[e]
            model.train_range(du, di, 0, npairs, params(e))
            ev1.record(stream)
            ev1.synchronize()
            return ev0.elapsed_time(ev1) / 1e3, model.counters.read()
    else:
        from paper_2304_07334_b200.parallel import NativeShardTrainer, PipelinedShardTrainer
        trainer = (PipelinedShardTrainer if args.shard_driver == "python"
                   else NativeShardTrainer)(model, world, rank)
        host_pairs = [epoch_pairs(train, shuffle_seed(0, e)) for e in range(total_epochs)]
        # global step = B pairs per rank (each GPU keeps the config's batch
        # between exchanges, as a data-parallel batch of B per GPU)
        exchange_pairs = args.exchange_pairs or spec.batch * world

        def one_epoch(e):
            nonlocal launches_per_epoch
            u, i = host_pairs[e]
            trainer.prepare_epoch(u, i, params(e), exchange_pairs)  # shard upload, untimed
            model.counters.reset()
            flush.zero_()
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ev0.record(stream)
            trainer.train_epoch(u, i, params(e), exchange_pairs, prepared=True)
            ev1.record(stream)
            ev1.synchronize()
            # the persistent epoch: one launch; stream-ordered steps: the DELTA
            # kernel + two apply kernels per step
            st = getattr(trainer, "stats", None)
            launches_per_epoch = (int(st.launches) if isinstance(st, N.ShardStats)
                                  else 3 * trainer.num_steps)
            return ev0.elapsed_time(ev1) / 1e3, model.counters.read()

    for e in range(args.warmup):
        one_epoch(e)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    times, actives, losses, pairs_done = [], [], [], []
    for s in range(args.steps):
        dt, c = one_epoch(args.warmup + s)
        times.append(dt)
        actives.append(c.active)
        losses.append(c.loss)
        pairs_done.append(c.pairs)
    torch.cuda.synchronize()
    clk = clocks.stop()
    total = sum(times)
    act_total = float(np.sum(actives))
    loss_total = float(np.sum(losses))
    if world > 1:
        t = torch.tensor([total], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total = float(t.item())
        agg = torch.tensor([act_total, loss_total, float(sum(pairs_done))], dtype=torch.float64,
                           device=dev)
        dist.all_reduce(agg)
        act_total, loss_total = float(agg[0]), float(agg[1])
        assert int(agg[2]) == npairs * args.steps, "every pair trained exactly once"
        dist.barrier()
    value = npairs * args.steps / total  # whole job: every pair of every timed epoch
    kernel_s = total / args.steps
    bytes_per_epoch = algorithmic_bytes(npairs, K, NN, int(act_total / args.steps))
    peak, peak_kind = _peaks()
    achieved = bytes_per_epoch / kernel_s / 1e9 / world  # per GPU, vs the per-GPU peak

    # e2e: the public drop-in API with host numpy tables (1 GPU path)
    e2e = None
    if not sharded and args.e2e_steps:
        configure(mode=args.mode, window=window, fp64=args.fp64)
        cfg = train_config(spec, threads=8 if args.mode == "hogwild" else 1)
        from paper_2304_07334_b200.embeddings import EmbeddingMatrix
        Se, Te = EmbeddingMatrix(S.copy()), EmbeddingMatrix(T.copy())
        train_epoch(Se, Te, train, cfg, epoch=0)
        train_epoch(Se, Te, train, cfg, epoch=1)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for e in range(args.e2e_steps):
            rep = train_epoch(Se, Te, train, cfg, epoch=2 + e)
            assert np.isfinite(rep.mean_loss)  # the step's result, read back on the host
        e2e_s = (time.perf_counter() - t0) / args.e2e_steps
        e2e = {"value": npairs / e2e_s, "unit": "samples/s",
               "h2d_bytes_per_step": S.nbytes + T.nbytes + 8 * npairs,
               "d2h_bytes_per_step": S.nbytes + T.nbytes + 32,
               "path": "paper_2304_07334_b200.train_epoch (host numpy S/T, shuffle, H2D, "
                       "kernel, D2H), steady state over consecutive epochs"}
    elif sharded and args.e2e_steps:
        # the multi-GPU public API keeps the tables device-resident (as train()
        # does); per epoch it takes the host epoch order: shard + H2D of the
        # rank's pairs and positions, the pipelined steps, the loss read back
        xp = exchange_pairs
        e2e_times = []
        h2d = 0
        for e in range(args.e2e_steps):
            u, i = host_pairs[e % len(host_pairs)]
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            model.counters.reset()
            trainer.train_epoch(u, i, params(e), xp)
            c = model.counters.read()
            assert np.isfinite(c.loss)
            dt = time.perf_counter() - t0
            if world > 1:
                tt = torch.tensor([dt], device=dev)
                dist.all_reduce(tt, op=dist.ReduceOp.MAX)
                dt = float(tt.item())
            e2e_times.append(dt)
            h2d = int(trainer.lu.numel()) * 8 + int(trainer.lp.numel()) * 8
        e2e = {"value": npairs / float(np.median(e2e_times)), "unit": "samples/s",
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": 32,
               "path": "NativeShardTrainer.train_epoch with the host epoch order (shard, H2D "
                       "of this rank's pairs, pipelined steps, loss read); tables "
                       "device-resident across epochs as in train(); max over ranks"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        threads = os.cpu_count() or 1
        # about 10 s of host work each (bounded samples of the same workload)
        cpu = cpu_baseline_timed(spec, train, S, T, threads, args.cpu_seconds)
        cpu.pop("seconds", None)
        # the single-thread figure beside it
        one = cpu_baseline_timed(spec, train, S, T, 1, args.cpu_seconds)
        cpu["value_1_thread"] = one["value"]
        cpu["sample_1_thread"] = one["sample"]

    if rank == 0:
        prof = _ncu_traffic(spec.name)
        table_bytes = S.nbytes + T.nbytes
        hbm = {"hbm_peak": peak, "hbm_peak_kind": peak_kind, "frac_of_hbm": achieved / peak}
        if table_bytes < L2_BYTES * 0.9:
            # S+T stay in L2 (ncu: >= 98.6 % sector hit rate on c2-c4): the L2
            # read ceiling, measured live, bounds the kernel; HBM frac kept beside
            probe = l2_probe(dev, table_bytes, model.T)
            l2_peak = max(probe.values())
            roofline = {"bound": "l2", "achieved": achieved, "peak": l2_peak,
                        "peak_kind": "measured live (GB/s): best of heat_probe_l2_read streaming "
                                     "reads (48 MB, S+T-sized) and heat_probe_l2_gather random-row "
                                     "gathers of T " +
                                     json.dumps({k: round(v, 1) for k, v in probe.items()}),
                        "unit": "GB/s", "frac": achieved / l2_peak, **hbm}
        else:
            roofline = {"bound": "hbm", "achieved": achieved, "peak": peak,
                        "peak_kind": peak_kind, "unit": "GB/s", "frac": achieved / peak}
        roofline.update({
            "traffic": prof.get("dram_bytes_per_launch") if prof else None,
            "traffic_source": prof.get("source") if prof else None,
            "l2_hit_rate_pct": prof.get("l2_hit_rate_pct") if prof else None,
            "bytes_per_launch": bytes_per_epoch,
            "bytes_per_pair": "4K(N+2)+8 read + 4K(2+A_p) written (SURVEY.md §8(d))",
            "table_bytes": table_bytes,
            "active_negatives_per_pair": act_total / args.steps / npairs})
        if clk.get("sm_mhz"):
            # the same rate per SM clock, at the median clock sampled DURING the
            # timed region (the live ceiling probe is a short burst at the box's
            # top clock; a long epoch may run under sw_power_cap): an SM's L2
            # fill port moves 64 B per clock
            n_sm = torch.cuda.get_device_properties(dev).multi_processor_count
            roofline["achieved_bytes_per_clk_per_sm"] = achieved * 1e9 / (n_sm * clk["sm_mhz"] * 1e6)
        line = {
            "metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": kernel_s * 1e3,
            "higher_is_better": True, "scaling": "strong" if sharded else "weak",
            "vs_baseline": None, "dtype": "f64" if args.fp64 else "f32", "data": "synthetic",
            "config": workload_config(spec, train),
            "run": {"window": window, "mode": args.mode, "step": "one epoch",
                    "l2_flush": "512 MiB write before every timed epoch; S+T "
                                f"{(S.nbytes + T.nbytes) / 1e6:.1f} MB",
                    "parallelism": (f"users sharded x{world}, item-delta exchange every "
                                    f"{exchange_pairs} global pairs ("
                                    + ("persistent epoch: one launch, device-gated steps"
                                       if launches_per_epoch == 1
                                       else "stream-ordered steps, P2P gather+apply")
                                    + f", lag {shard_lag(launches_per_epoch == 1)})"
                                    if sharded else "single GPU")},
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches_per_epoch * args.steps,
            "clocks": clk,
            "mean_loss": loss_total / args.steps / npairs,
        }
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
