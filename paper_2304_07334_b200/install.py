"""Install the B200 path into a running reference package (heatcf).

The reference is read-only and ``TrainingConfig`` is frozen, so the GPU path
is selected by rebinding module globals:

- ``heatcf.trainer.train_epoch``  (called by ``train``, trainer.py:516)
- ``heatcf.bench.train_epoch``    (bound at import, bench.py:31)
- ``heatcf.evaluator.evaluate``   (imported inside ``train``, trainer.py:493)
- ``heatcf.evaluator.topk_items``

The reference's own dataclasses flow through unchanged (duck typing on
``.values``, ``.offsets``, ``cfg.loss.mu`` …).  ``uninstall()`` restores the
originals.
"""

from __future__ import annotations

import importlib
import importlib.util
import sys

_saved: dict = {}


def install(heatcf=None) -> None:
    from . import evaluator, trainer

    if heatcf is None:
        heatcf = importlib.import_module("heatcf")
    targets = [("heatcf.trainer", "train_epoch", trainer.train_epoch),
               ("heatcf.evaluator", "evaluate", evaluator.evaluate),
               ("heatcf.evaluator", "topk_items", evaluator.topk_items),
               ("heatcf", "train_epoch", trainer.train_epoch),
               ("heatcf", "evaluate", evaluator.evaluate)]
    if "heatcf.bench" in sys.modules or importlib.util.find_spec("matplotlib") is not None:
        try:
            importlib.import_module("heatcf.bench")
            targets.append(("heatcf.bench", "train_epoch", trainer.train_epoch))
        except ImportError:
            pass
    for mod_name, attr, fn in targets:
        mod = importlib.import_module(mod_name)
        _saved.setdefault((mod_name, attr), getattr(mod, attr))
        setattr(mod, attr, fn)


def uninstall() -> None:
    for (mod_name, attr), fn in _saved.items():
        setattr(importlib.import_module(mod_name), attr, fn)
    _saved.clear()
