"""Training configuration types, field-for-field with the reference.

``LossParams`` follows kernels.py:43-54, ``SamplerConfig`` trainer.py:47-59,
``AggregatorConfig`` aggregator.py:30-47 and ``TrainingConfig``
trainer.py:62-87, including their validation errors.  The GPU path reads any
object with these attribute names (the reference's own dataclasses work
unchanged), so ``install()`` can hand it the reference's configs.

Options outside the north_star path (tiling sampler, aggregator) validate
here but are rejected by the GPU trainer with ValueError — there is no CPU
fallback.
"""

from __future__ import annotations

from dataclasses import dataclass, field


@dataclass(frozen=True)
class LossParams:
    mu: float = 1.0
    theta: float = 0.8

    def __post_init__(self):
        if self.mu < 0:
            raise ValueError(f"mu must be >= 0, got {self.mu}")
        if not -1.0 <= self.theta <= 1.0:
            raise ValueError(f"theta must be in [-1, 1], got {self.theta}")


@dataclass(frozen=True)
class SamplerConfig:
    kind: str = "uniform"
    tile_size: int = 1024
    refresh_interval: int = 4096

    def __post_init__(self):
        if self.kind not in ("uniform", "tiling"):
            raise ValueError(f"unknown sampler kind: {self.kind!r}")
        if self.kind == "tiling" and (self.tile_size < 1 or self.refresh_interval < 1):
            raise ValueError("tiling needs tile_size >= 1 and refresh_interval >= 1")


@dataclass(frozen=True)
class AggregatorConfig:
    enabled: bool = False
    gamma: float = 0.5
    max_history: int = 100
    mini_batch_size: int = 32
    history_grad: bool = False
    learning_rate: float | None = None

    def __post_init__(self):
        if not 0.0 <= self.gamma <= 1.0:
            raise ValueError(f"gamma must be in [0, 1], got {self.gamma}")
        if self.max_history < 0:
            raise ValueError(f"max_history must be >= 0, got {self.max_history}")
        if self.mini_batch_size < 1:
            raise ValueError(f"mini_batch_size must be >= 1, got {self.mini_batch_size}")


@dataclass(frozen=True)
class TrainingConfig:
    emb_dim: int = 128
    num_negatives: int = 64
    learning_rate: float = 0.05
    epochs: int = 100
    num_threads: int = 1
    similarity: str = "cosine"
    loss: LossParams = field(default_factory=LossParams)
    sampler: SamplerConfig = field(default_factory=SamplerConfig)
    aggregator: AggregatorConfig = field(default_factory=AggregatorConfig)
    seed: int = 0
    l2_reg: float = 0.0
    chunk_pairs: int = 2048

    def __post_init__(self):
        if self.num_negatives < 1:
            raise ValueError(f"num_negatives must be >= 1, got {self.num_negatives}")
        if not self.learning_rate > 0:
            raise ValueError(f"learning_rate must be positive, got {self.learning_rate}")
        if self.num_threads < 1:
            raise ValueError(f"num_threads must be >= 1, got {self.num_threads}")
        if self.similarity not in ("cosine", "dot"):
            raise ValueError(f"unknown similarity: {self.similarity!r}")
