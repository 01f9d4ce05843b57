"""TEST INFRASTRUCTURE — restatement of the reference's unit-level math spec.

/root/reference/pkg/src/heatcf/kernels.py:57-159 (cosine_forward,
ccl_loss, ccl_loss_grad, cosine_grad_user, cosine_grad_item) and the
finite-difference helper of pkg/tests/helpers.py, in plain numpy, so the GPU
tests can pin the device path to the reference's spec the way
pkg/tests/test_kernels.py and test_acceptance.py:90-145 (c01-c03) pin
heatcf's own kernels.  Only tests/ import this module; the product never
does.
"""

from __future__ import annotations

import math

import numpy as np


def _dot(u, v) -> float:
    """kernels.py:57-62: float64 accumulation in sequential k order."""
    acc = 0.0
    for a, b in zip(np.asarray(u, dtype=np.float64), np.asarray(v, dtype=np.float64)):
        acc += float(a) * float(b)
    return acc


def cosine_forward(u, v):
    """kernels.py:65-73 -> (ss, tt, st, sim, degenerate)."""
    ss, tt, st = _dot(u, u), _dot(v, v), _dot(u, v)
    if ss <= 0.0 or tt <= 0.0:
        return ss, tt, st, 0.0, True
    return ss, tt, st, st / (math.sqrt(ss) * math.sqrt(tt)), False


def _grad_into(u, v, ss, tt, st) -> np.ndarray:
    """kernels.py:76-85: (v*ss - st*u) / (ss*sqrt(ss)*sqrt(tt)); zero when degenerate."""
    u = np.asarray(u, dtype=np.float64)
    v = np.asarray(v, dtype=np.float64)
    if ss <= 0.0 or tt <= 0.0:
        return np.zeros(len(u))
    denom = ss * math.sqrt(ss) * math.sqrt(tt)
    return (v * ss - st * u) / denom


def cosine_grad_user(u, v) -> np.ndarray:
    """kernels.py:139-152."""
    ss, tt, st, _, _ = cosine_forward(u, v)
    return _grad_into(u, v, ss, tt, st)


def cosine_grad_item(u, v) -> np.ndarray:
    """kernels.py:155-159: the mirror of cosine_grad_user."""
    ss, tt, st, _, _ = cosine_forward(u, v)
    return _grad_into(v, u, tt, ss, st)


def ccl_loss(sim_pos: float, sim_negs, mu: float, theta: float) -> float:
    """kernels.py:88-95 / 113-118."""
    sim_negs = np.asarray(sim_negs, dtype=np.float64)
    hinge = 0.0
    for s in sim_negs:
        d = float(s) - theta
        if d > 0.0:
            hinge += d
    return (1.0 - sim_pos) + (mu / len(sim_negs)) * hinge


def ccl_loss_grad(sim_pos: float, sim_negs, mu: float, theta: float):
    """kernels.py:121-136: dpos = -1; mu/|N| per negative strictly above theta."""
    sim_negs = np.asarray(sim_negs, dtype=np.float64)
    return -1.0, np.where(sim_negs > theta, mu / len(sim_negs), 0.0)


def fd_cosine_grads(u, v, step: float = 1e-6):
    """pkg/tests/helpers.py: central finite differences of the cosine."""
    u = np.asarray(u, dtype=np.float64)
    v = np.asarray(v, dtype=np.float64)

    def cos_rows(U, w):
        un = np.sqrt(np.sum(U * U, axis=1))
        wn = math.sqrt(float(w @ w))
        out = U @ w
        good = (un > 0) & (wn > 0)
        out[good] /= un[good] * wn
        out[~good] = 0.0
        return out

    eye = np.eye(len(u)) * step
    gu = (cos_rows(u[None, :] + eye, v) - cos_rows(u[None, :] - eye, v)) / (2 * step)
    gv = (cos_rows(v[None, :] + eye, u) - cos_rows(v[None, :] - eye, u)) / (2 * step)
    return gu, gv
