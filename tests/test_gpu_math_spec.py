"""the device path pinned to the reference's unit-level
math spec (kernels.py:57-159), the way heatcf's test_kernels.py:20-79 and
test_acceptance.py:90-145 (c01-c03) pin heatcf's own kernels.

Single constructed pairs go through the real training kernels (EXACT, and
the throughput kernel at one pair in flight): user row u, positive row v+,
and a table whose every other row is v- (the stream base is chosen so no
negative draws the positive's row).  From the kernel's outputs:

* the pair's loss equals ccl_loss(cos(u, v+), [cos(u, v-)] * N) (EXACT: to
  1e-13 relative — the reference's own arithmetic; throughput: 1e-6);
* with lr = 1 the row updates give the gradients back
  (S' - S = -(dpos * grad_u(u, v+) + sum_j dneg_j * grad_u(u, v-)),
  T'[+] - v+ = -dpos * grad_v(u, v+), and each negative's row moves by
  -dneg * grad_v(u, v-) per draw), which must equal kernels.py's
  cosine_grad_user / cosine_grad_item (c03's loss-gradient rule included)
  and the finite differences of the cosine (c01), and be orthogonal to their
  vectors (c02), with c01's 1e-4 and c02's 1e-6 bounds.  Each read-back
  element carries the float32 rounding of the updated table value
  (2^-24 |value| per write), which the tolerances add explicitly; on top of
  that EXACT agrees to 1e-12 (binary64 arithmetic) and the throughput kernel
  to 1e-5 (fp32 coefficients).
"""

import numpy as np
import pytest

from oracle import kernels_spec as KS

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    assert torch.cuda.is_available()
    from paper_2304_07334_b200 import _native
    _native.lib()
    return torch


ROWS = 64  # T: row 0 = v+, rows 1..63 = v-


def _stream_base(N: int, seed: int) -> int:
    from paper_2304_07334_b200.rng import counter_draw
    s0 = 0x1234_5678_9ABC_DEF0 ^ (seed * 0x9E3779B97F4A7C15 & 0xFFFFFFFFFFFFFFFF)
    while any(counter_draw(s0, j) % ROWS == 0 for j in range(N)):
        s0 = (s0 + 1) & 0xFFFFFFFFFFFFFFFF
    return s0


def _run_pair(u, vp, vn, N, mu, theta, mode, seed):
    from paper_2304_07334_b200 import _native as NN
    from paper_2304_07334_b200.device import DeviceModel
    from paper_2304_07334_b200.rng import counter_draw
    K = len(u)
    S = u.reshape(1, K).astype(np.float32)
    T = np.empty((ROWS, K), np.float32)
    T[0] = vp
    T[1:] = vn
    s0 = _stream_base(N, seed)
    hits = np.bincount([counter_draw(s0, j) % ROWS for j in range(N)], minlength=ROWS)
    m = DeviceModel(S, T)
    du, di = m.upload_pairs(np.zeros(1, np.int32), np.zeros(1, np.int32))
    p = m.params(n_neg=N, lr=1.0, l2=0.0, mu=mu, theta=theta, cosine=True, mode=mode,
                 stream_base=s0, window=1)
    m.counters.reset()
    m.train_range(du, di, 0, 1, p)
    c = m.counters.read()
    S1, T1 = S.copy(), T.copy()
    m.download(S1, T1)
    return c, S1[0].astype(np.float64), T1.astype(np.float64), hits


def _expected(u, vp, vn, N, mu, theta):
    sp = KS.cosine_forward(u, vp)[3]
    sn = KS.cosine_forward(u, vn)[3]
    loss = KS.ccl_loss(sp, [sn] * N, mu, theta)
    dpos, dnegs = KS.ccl_loss_grad(sp, [sn] * N, mu, theta)
    gu = dpos * KS.cosine_grad_user(u, vp) + dnegs.sum() * KS.cosine_grad_user(u, vn)
    gvp = dpos * KS.cosine_grad_item(u, vp)
    gvn = dnegs[0] * KS.cosine_grad_item(u, vn)  # per draw
    return loss, gu, gvp, gvn


def _rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - b) / max(np.linalg.norm(b), 1e-300))


def _check(u, vp, vn, N, mu, theta, mode, seed, loss_tol):
    c, S1, T1, hits = _run_pair(u, vp, vn, N, mu, theta, mode, seed)
    u64, vp64, vn64 = (np.asarray(x, np.float64) for x in (u, vp, vn))
    loss, gu, gvp, gvn = _expected(u64, vp64, vn64, N, mu, theta)
    assert c.pairs == 1 and c.degenerate == 0
    assert abs(c.loss - loss) <= loss_tol * max(abs(loss), 1e-12), (c.loss, loss)
    # gradients read back from the lr = 1 updates
    # each read-back element carries one float32 rounding of the updated
    # value per write (|error| <= 2^-24 |value|), plus the kernel's own
    # arithmetic (binary64 in EXACT, fp32 in the throughput kernel)
    eps = 2.0 ** -24
    arith = 1e-12 if loss_tol < 1e-9 else 1e-5

    def close(got, want, base, writes=1):
        err = np.linalg.norm(got - want)
        scale = np.linalg.norm(base) + np.linalg.norm(want)  # |old| and |new| values
        assert err <= arith * np.linalg.norm(want) + 2 * eps * writes * scale + 1e-30, \
            (err, np.linalg.norm(want), mode)

    g_user = -(S1 - u64)
    g_pos = -(T1[0] - vp64)
    close(g_user, gu, u64)
    close(g_pos, gvp, vp64)
    for r in np.flatnonzero(hits):
        close(-(T1[r] - vn64), hits[r] * gvn, vn64, writes=hits[r])
    return g_pos, g_user


def _modes():
    from paper_2304_07334_b200 import _native as NN
    return [(NN.MODE_EXACT, 1e-13), (NN.MODE_HOGWILD, 1e-6)]


def test_hand_values(torch_cuda):
    """test_kernels.py hand cases through the kernels: identical vectors
    (sim 1, no gradient), orthogonal negative (sim 0, inactive), 45 degrees
    (sim 1/sqrt 2) with an active negative."""
    for mode, tol in _modes():
        # identical user and positive: loss 0, positive gradient 0
        c, S1, T1, _ = _run_pair(np.array([1, 0], np.float32), np.array([1, 0], np.float32),
                                 np.array([0, 1], np.float32), 1, 1.0, 0.8, mode, 1)
        assert abs(c.loss) <= tol
        assert np.allclose(S1, [1.0, 0.0], rtol=0, atol=tol)
        assert np.allclose(T1[0], [1.0, 0.0], rtol=0, atol=tol)
        # 45 degrees to both rows, theta 0.5: (1 - 1/sqrt2) + mu * (1/sqrt2 - 0.5)
        u = np.array([1, 1], np.float32)
        c, *_ = _run_pair(u, np.array([1, 0], np.float32), np.array([0, 1], np.float32), 1,
                          2.0, 0.5, mode, 2)
        want = (1 - 2 ** -0.5) + 2.0 * (2 ** -0.5 - 0.5)
        assert abs(c.loss - want) <= tol
        _check(u, np.array([1, 0], np.float32), np.array([0, 1], np.float32), 1, 2.0, 0.5, mode,
               2, tol)


@pytest.mark.parametrize("dim", [2, 64, 128])
def test_c01_c02_c03_through_the_kernels(torch_cuda, dim):
    """Random pairs (c01/c02 draw u, v ~ N(0, 1); c03 draws mu in [0, 3],
    theta in [-0.9, 0.9], 1..8 negatives): loss and gradients equal the
    spec's, gradients match central finite differences of the cosine within
    1e-4 (c01) and are orthogonal to their vectors (c02)."""
    rng = np.random.default_rng(101 + dim)
    for case in range(40):
        u = rng.standard_normal(dim).astype(np.float32)
        vp = rng.standard_normal(dim).astype(np.float32)
        vn = rng.standard_normal(dim).astype(np.float32)
        mu = float(rng.uniform(0.0, 3.0))
        theta = float(rng.uniform(-0.9, 0.9))
        sn = KS.cosine_forward(u, vn)[3]
        if abs(sn - theta) < 1e-4:  # off the hinge kink (c03)
            theta = sn - 0.1
        N = int(rng.integers(1, 9))
        for mode, tol in _modes():
            g_pos, _ = _check(u, vp, vn, N, mu, theta, mode, case, tol)
        # c01: the read-back item gradient against finite differences (the
        # read-back adds float32 rounding of v+: 2^-23 |v+| absolute)
        fu, fv = KS.fd_cosine_grads(u.astype(np.float64), vp.astype(np.float64))
        vp64 = vp.astype(np.float64)
        assert np.linalg.norm(g_pos + fv) <= 1e-4 * np.linalg.norm(fv) + \
            2.0 ** -23 * (np.linalg.norm(vp64) + np.linalg.norm(fv))
        # c02: orthogonal to its vector, up to the same read-back rounding
        assert abs(float(g_pos @ vp64)) <= 1e-6 * np.linalg.norm(g_pos) * np.linalg.norm(vp64) + \
            2.0 ** -23 * (np.linalg.norm(vp64) + np.linalg.norm(g_pos)) * np.linalg.norm(vp64)
