"""One rank of the two-process run of csrc/heat_shard.cu on ONE GPU
(tests/test_gpu_shard_ipc.py starts `world` of these).

    python shard_ipc_worker.py RANK WORLD PORT SCENARIO

The ranks are separate processes, so the peers' delta logs are reached through
CUDA IPC mappings (cudaIpcGetMemHandle / cudaIpcOpenMemHandle, which work
between processes on one device) — the production mapping path; the runtime's
collectives ride on gloo (heat_shard_create_host: NCCL refuses two ranks on
one GPU).  Stream-ordered steps only, so no kernel waits on another process.

Scenarios:
  exact   one pair in flight, lag 1: the world-2 tables equal the world-1
          runtime's bit for bit (users are disjoint between ranks, the
          fixed-point apply is order-free), replicas identical
  p2p     256 pairs in flight, lag 2, IPC reads: every pair once, replicas
          bit-identical, loss within 3 % of world 1
  gather  the same through the gather fallback (logs all-gathered)
Exit code 0 = every assertion held on this rank.
"""

import os
import sys

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, ROOT)


def main() -> int:
    rank, world, port, scenario = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3], sys.argv[4]
    os.environ["HEAT_SHARD_LAG"] = "1" if scenario == "exact" else "2"
    os.environ["HEAT_SHARD_EXCHANGE"] = "gather" if scenario == "gather" else "p2p"
    if scenario == "exact":
        os.environ["HEAT_HOGWILD_IMPL"] = "wide"  # one warp per pair: deterministic at window 1
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2304_07334_b200 import _native as N
    from paper_2304_07334_b200.dataset import epoch_pairs
    from paper_2304_07334_b200.device import DeviceModel
    from paper_2304_07334_b200.embeddings import InitSpec, init_matrix
    from paper_2304_07334_b200.parallel import NativeShardTrainer
    from paper_2304_07334_b200.rng import epoch_stream, shuffle_seed
    from workloads import make_dataset

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    torch.cuda.set_device(0)
    K = 128 if scenario == "exact" else 64
    train, _, _ = make_dataset("c2", scale=0.02 if scenario == "exact" else 0.05)
    S = init_matrix(train.num_users, K, InitSpec(seed=0)).values
    T = init_matrix(train.num_items, K, InitSpec(seed=0)).values
    window, step = (1, 256) if scenario == "exact" else (256, 1024)

    def params(m, e):
        return m.params(n_neg=100, lr=0.01, l2=0.0, mu=20.0, theta=0.3, cosine=True,
                        mode=N.MODE_DELTA, stream_base=epoch_stream(0, e), window=window)

    mine = DeviceModel(S, T)
    sh = NativeShardTrainer(mine, world, rank, transport="host")
    ref = DeviceModel(S, T)
    one = NativeShardTrainer(ref, 1, 0)
    for e in range(2):
        u, i = epoch_pairs(train, shuffle_seed(0, e))
        mine.counters.reset()
        st = sh.train_epoch(u, i, params(mine, e), step)
        ref.counters.reset()
        one.train_epoch(u, i, params(ref, e), step)
        torch.cuda.synchronize()
        c = mine.counters.read()
        tot = torch.tensor([float(c.pairs), c.loss], dtype=torch.float64)
        dist.all_reduce(tot)
        assert int(tot[0]) == len(u), (int(tot[0]), len(u))
        assert st.steps == sh.num_steps and st.entries >= len(u)
        assert st.launches > 1, "the host transport runs stream-ordered steps"
        if scenario != "gather":
            assert st.exchanged_bytes > 0  # read from the peer's log through the IPC mapping
        Tm = mine.T.cpu()
        parts = [torch.empty_like(Tm) for _ in range(world)]
        dist.all_gather(parts, Tm)
        for q in range(world):  # replicas identical
            assert parts[q].numpy().tobytes() == Tm.numpy().tobytes(), f"replica {q} differs"
        want = ref.counters.read().loss
        if scenario == "exact":
            assert Tm.numpy().tobytes() == ref.T.cpu().numpy().tobytes(), "T != world-1 epoch"
            own = np.arange(train.num_users) % world == rank
            assert (mine.S.cpu().numpy()[own].tobytes() ==
                    ref.S.cpu().numpy()[own].tobytes()), "owned S rows != world-1 epoch"
            assert abs(float(tot[1]) - want) <= 1e-9 * abs(want)
        else:
            assert np.isfinite(float(tot[1])) and abs(float(tot[1]) - want) <= 0.03 * abs(want)
    sh.close()
    one.close()
    dist.barrier()
    dist.destroy_process_group()
    print(f"rank {rank}/{world} {scenario}: ok")
    return 0


if __name__ == "__main__":
    sys.exit(main())
