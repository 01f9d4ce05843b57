"""B200-native SimpleX-MF-CCL training path (HEAT, arXiv 2304.07334).

A drop-in for the hot path of the reference package ``heatcf``:
``train_epoch`` / ``train`` / ``evaluate`` with the reference's signatures and
data types, running on hand-written sm_100a CUDA kernels (csrc/) through the
C ABI of include/heat_b200.h.  ``install()`` patches a running heatcf so its
own ``train()``, CLI and bench use this path unchanged.
"""

from .config import AggregatorConfig, LossParams, SamplerConfig, TrainingConfig
from .dataset import InteractionSet, epoch_pairs, from_pairs, from_user_lists, history_of, \
    with_universe
from .embeddings import CorruptCheckpointError, EmbeddingMatrix, InitSpec, init_matrix, \
    load_checkpoint, load_model, save_checkpoint, save_model
from .rng import SplitMix64, derive_stream, mix64, stream_state

__version__ = "0.1.0"


def __getattr__(name):
    # GPU-facing modules import torch lazily so the host types stay light.
    if name in ("train_epoch", "train", "EpochReport", "TrainResult", "configure", "PHASE_NAMES",
                "options"):
        from . import trainer
        return getattr(trainer, name)
    if name in ("evaluate", "MetricsReport", "topk_items", "metrics_json", "EmptyTestSetError"):
        from . import evaluator
        return getattr(evaluator, name)
    if name in ("DeviceModel",):
        from . import device
        return getattr(device, name)
    if name == "install":
        from .install import install
        return install
    raise AttributeError(name)


__all__ = [
    "AggregatorConfig", "CorruptCheckpointError", "EmbeddingMatrix", "EpochReport", "InitSpec", "InteractionSet",
    "LossParams", "MetricsReport", "SamplerConfig", "SplitMix64", "TrainResult",
    "TrainingConfig", "configure", "derive_stream", "epoch_pairs", "evaluate", "from_pairs",
    "from_user_lists", "history_of", "init_matrix", "install", "load_checkpoint", "load_model", "mix64",
    "save_checkpoint", "save_model", "stream_state", "topk_items", "train", "train_epoch", "with_universe",
]
