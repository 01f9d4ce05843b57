"""SplitMix64 streams — host side of the negative sampler.

Restates /root/reference/pkg/src/heatcf/rng.py:26-81.  The device sampler
(csrc/heat_common.cuh: ``heat_neg_id``) uses the *counter form* of the same
stream: the n-th draw (0-based) of a stream whose state is ``s0`` is
``mix64(s0 + (n + 1) * GAMMA)``.  A single-thread reference epoch draws
negative j of the pair at epoch position p as draw ``p * N + j`` of the
stream ``derive_stream(seed, 0x45504F43, epoch, 0)`` (trainer.py:134-139,
340, 399), so any decomposition of the epoch over warps/GPUs that keeps the
global pair index reproduces the reference's negative ids bit for bit.
"""

from __future__ import annotations

import numpy as np

MASK = 0xFFFFFFFFFFFFFFFF
GAMMA = 0x9E3779B97F4A7C15
_MIX1 = 0xBF58476D1CE4E5B9
_MIX2 = 0x94D049BB133111EB

EPOCH_SALT = 0x45504F43    # trainer.py:43
SHUFFLE_SALT = 0x53485546  # trainer.py:44


def mix64(x: int) -> int:
    """SplitMix64 finalizer (rng.py:26-31)."""
    x &= MASK
    x = ((x ^ (x >> 30)) * _MIX1) & MASK
    x = ((x ^ (x >> 27)) * _MIX2) & MASK
    return x ^ (x >> 31)


def derive_stream(seed: int, *words: int) -> int:
    """Stream state from a base seed and salt words (rng.py:34-39)."""
    state = mix64(seed)
    for w in words:
        state = mix64((state + GAMMA + (w & MASK)) & MASK)
    return state


class SplitMix64:
    """Sequential stream, bit-compatible with rng.py:42-60."""

    def __init__(self, seed: int, *words: int):
        self.state = derive_stream(seed, *words)

    def next_u64(self) -> int:
        self.state = (self.state + GAMMA) & MASK
        return mix64(self.state)

    def below(self, n: int) -> int:
        if n <= 0:
            raise ValueError(f"bound must be positive, got {n}")
        return self.next_u64() % n

    def uniform(self) -> float:
        return (self.next_u64() >> 11) * (1.0 / (1 << 53))


def stream_state(seed: int, *words: int) -> np.ndarray:
    """uint64[1] state array, as rng.py:79-81."""
    return np.array([derive_stream(seed, *words)], dtype=np.uint64)


def counter_draw(s0: int, n: int) -> int:
    """The n-th (0-based) draw of the stream whose state is s0."""
    return mix64((s0 + ((n + 1) * GAMMA)) & MASK)


def epoch_stream(seed: int, epoch: int) -> int:
    """Stream base of the single-thread reference epoch (trainer.py:399)."""
    return derive_stream(seed, EPOCH_SALT, epoch, 0)


def shuffle_seed(seed: int, epoch: int) -> int:
    """Seed handed to epoch_pairs (trainer.py:390-392)."""
    return derive_stream(seed, SHUFFLE_SALT, epoch) >> 1
