import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["HEAT_HOGWILD_IMPL"] = "resident"
import numpy as np, torch
from paper_2304_07334_b200 import _native as N
from paper_2304_07334_b200.dataset import epoch_pairs
from paper_2304_07334_b200.device import DeviceModel
from paper_2304_07334_b200.embeddings import InitSpec, init_matrix
from paper_2304_07334_b200.rng import epoch_stream, shuffle_seed
from paper_2304_07334_b200.synth import make_dataset
for cfg, K, NN, th, mu in (("c1", 32, 10, 0.5, 10.0), ("c2", 64, 100, 0.9, 150.0)):
    tr, _, _ = make_dataset(cfg, scale=0.2)
    S = init_matrix(tr.num_users, K, InitSpec(seed=0)).values
    T = init_matrix(tr.num_items, K, InitSpec(seed=0)).values
    m = DeviceModel(S, T)
    u, i = epoch_pairs(tr, shuffle_seed(0, 0))
    du, di = m.upload_pairs(u, i)
    p = m.params(n_neg=NN, lr=1e-3, l2=0.0, mu=mu, theta=th, cosine=True, mode=N.MODE_HOGWILD,
                 stream_base=epoch_stream(0, 0), window=1024)
    m.counters.reset()
    m.train_range(du, di, 0, len(u), p)
    torch.cuda.synchronize()
    print(cfg, m.counters.read(), flush=True)
