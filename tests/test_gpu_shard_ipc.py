"""csrc/heat_shard.cu at world 2 as TWO PROCESSES on one GPU: the peers'
delta logs are read through CUDA IPC mappings — the production mapping path,
which the in-process loopback group (test_gpu_shard_loopback.py) cannot
reach — and the runtime's collectives (capacity agreement, IPC handle
exchange, the "every rank mapped every peer" vote, the per-step count fence)
ride on gloo through heat_shard_create_host.  Stream-ordered steps only:
no kernel of one process waits on a kernel of the other.

What is NOT covered on a one-GPU box: NCCL itself, NVLink, and the persistent
epoch between processes.  The reference's only parallel driver is the
threaded chunk loop (heatcf trainer.py:398-447); this is its scale-out form.
"""

import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("scenario", ["exact", "p2p", "gather"])
def test_two_processes_one_gpu(scenario):
    import torch
    assert torch.cuda.is_available()
    port = str(_free_port())
    env = dict(os.environ)
    for k in ("HEAT_SHARD_LAG", "HEAT_SHARD_EXCHANGE", "HEAT_HOGWILD_IMPL"):
        env.pop(k, None)
    procs = [subprocess.Popen([sys.executable, os.path.join(HERE, "shard_ipc_worker.py"), str(r),
                               "2", port, scenario], env=env, stdout=subprocess.PIPE,
                              stderr=subprocess.STDOUT, text=True) for r in range(2)]
    outs = []
    try:
        for p in procs:
            outs.append(p.communicate(timeout=420)[0])
    finally:
        for p in procs:  # only the processes started here
            if p.poll() is None:
                p.kill()
    for r, (p, o) in enumerate(zip(procs, outs)):
        assert p.returncode == 0, f"rank {r} failed:\n{o[-4000:]}"
        assert f"rank {r}/2 {scenario}: ok" in o
