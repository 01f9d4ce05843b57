import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2304_07334_b200 import _native as N
from paper_2304_07334_b200.dataset import epoch_pairs
from paper_2304_07334_b200.device import DeviceModel
from paper_2304_07334_b200.embeddings import InitSpec, init_matrix
from paper_2304_07334_b200.rng import epoch_stream, shuffle_seed
from paper_2304_07334_b200.synth import make_dataset
train, _, _ = make_dataset("c1")
u, i = epoch_pairs(train, shuffle_seed(0, 0))
for generic in (0, 1):
    if generic: os.environ["HEAT_FORCE_GENERIC"] = "1"
    for P in (1, 2, 3, 5, 10, 50, 200, 2000, 20000):
        res = {}
        for mode in (N.MODE_EXACT, N.MODE_HOGWILD):
            S = init_matrix(1000, 32, InitSpec(seed=0)).values
            T = init_matrix(2000, 32, InitSpec(seed=0)).values
            m = DeviceModel(S, T)
            du, di = m.upload_pairs(u, i)
            p = m.params(n_neg=10, lr=1e-3, l2=0.0, mu=10.0, theta=0.5, cosine=True, mode=mode,
                         stream_base=epoch_stream(0, 0), window=1)
            m.counters.reset()
            m.train_range(du, di, 0, P, p)
            c = m.counters.read()
            m.download(S, T)
            res[mode] = (S, T, c)
        (S0, T0, c0), (S1, T1, c1) = res[0], res[1]
        ds = np.abs(S1 - S0).max() / np.abs(S0).max(); dt = np.abs(T1 - T0).max() / np.abs(T0).max()
        rows = np.flatnonzero(np.any(np.abs(S1 - S0) > 1e-6 * np.abs(S0).max(), axis=1))
        print(f"generic={generic} P={P} dS={ds:.3e} dT={dt:.3e} loss {c0.loss:.6f} {c1.loss:.6f} act {c0.active} {c1.active} Srows {rows[:5]}", flush=True)
