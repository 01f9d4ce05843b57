"""HEATEMB1 files (embeddings.py:8-21, 98-183 of the reference): the
behaviours heatcf's test_embeddings.py pins, restated against this
package's host code, plus byte interoperability with the reference's own
reader and writer when the reference is importable (build container)."""

import os
import struct
import sys

import numpy as np
import pytest

from paper_2304_07334_b200.embeddings import (CorruptCheckpointError, EmbeddingMatrix, InitSpec,
                                              init_matrix, load_checkpoint, load_model,
                                              save_checkpoint, save_model)
from paper_2304_07334_b200.embeddings import encode_block


def test_init_validation_and_statistics():
    for bad in (lambda: InitSpec(kind="normal", std=0.0), lambda: InitSpec(kind="orthogonal"),
                lambda: init_matrix(0, 4, InitSpec(seed=1)),
                lambda: init_matrix(4, 0, InitSpec(seed=1))):
        with pytest.raises(ValueError):
            bad()
    m = init_matrix(1000, 64, InitSpec(kind="normal", mean=0.0, std=0.1, seed=7))
    assert abs(float(m.values.mean())) < 0.01 and abs(float(m.values.std()) - 0.1) < 0.01
    spec = InitSpec(kind="normal", std=0.1, seed=7)
    assert init_matrix(50, 8, spec).values.tobytes() == init_matrix(50, 8, spec).values.tobytes()
    x = init_matrix(300, 24, InitSpec(kind="xavier", seed=3))
    assert np.all(np.abs(x.values) <= np.sqrt(6.0 / 324))


def test_checkpoint_round_trips_bit_exact(tmp_path):
    rng = np.random.default_rng(112)
    for rows, dim in ((3, 4), (1, 1), (12, 9), (17, 9)):
        m = EmbeddingMatrix((rng.standard_normal((rows, dim)) * rng.uniform(0.01, 100))
                            .astype(np.float32))
        p = str(tmp_path / f"m{rows}.emb")
        save_checkpoint(m, p)
        assert load_checkpoint(p).values.tobytes() == m.values.tobytes()


def test_checkpoint_corruption_is_detected(tmp_path):
    cases = {"magic": b"NOTMAGIC" + b"\x00" * 32,
             "short": b"HEATEMB1" + struct.pack("<II", 2, 2) + b"\x00" * 12,
             "header": b"HEATEMB1" + b"\x01"}
    for name, blob in cases.items():
        p = tmp_path / name
        p.write_bytes(blob)
        with pytest.raises(CorruptCheckpointError):
            load_checkpoint(str(p))
    p = str(tmp_path / "trail.emb")
    save_checkpoint(init_matrix(2, 2, InitSpec(seed=1)), p)
    with open(p, "ab") as f:
        f.write(b"x")
    with pytest.raises(CorruptCheckpointError):
        load_checkpoint(p)


def test_model_bundles(tmp_path):
    S = init_matrix(5, 4, InitSpec(seed=1))
    T = init_matrix(9, 4, InitSpec(seed=2))
    p = str(tmp_path / "m.ckpt")
    save_model(p, S, T)
    s2, t2, w2 = load_model(p)
    assert s2.values.tobytes() == S.values.tobytes() and t2.values.tobytes() == T.values.tobytes()
    assert w2 is None
    w = np.random.default_rng(3).standard_normal((4, 4)).astype(np.float32)
    save_model(p, S, T, w)
    assert load_model(p)[2].tobytes() == w.tobytes()
    with pytest.raises(ValueError):
        save_model(str(tmp_path / "bad.ckpt"), S, T, np.zeros((3, 3), dtype=np.float32))
    bad = tmp_path / "dims.ckpt"
    with open(bad, "wb") as f:
        f.write(encode_block(init_matrix(3, 4, InitSpec(seed=1)).values))
        f.write(encode_block(init_matrix(3, 5, InitSpec(seed=2)).values))
    with pytest.raises(CorruptCheckpointError):
        load_model(str(bad))
    save_model(p, S, T)
    with open(p, "ab") as f:
        f.write(b"WHAT" + b"\x00" * 8)
    with pytest.raises(CorruptCheckpointError):
        load_model(p)


REF = "/root/reference/pkg/src"


def test_bundles_interoperate_with_the_reference(tmp_path, monkeypatch):
    """Our bundles load in heatcf and heatcf's load here, byte for byte."""
    if not os.path.isdir(REF):
        pytest.skip("reference not present")
    monkeypatch.setenv("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    monkeypatch.syspath_prepend(REF)
    sys.dont_write_bytecode = True
    try:
        import heatcf.embeddings as R
    except Exception as exc:  # pragma: no cover
        pytest.skip(f"heatcf not importable: {exc}")
    S = init_matrix(6, 8, InitSpec(seed=4))
    T = init_matrix(11, 8, InitSpec(seed=5))
    w = np.random.default_rng(6).standard_normal((8, 8)).astype(np.float32)
    ours, theirs = str(tmp_path / "ours.ckpt"), str(tmp_path / "theirs.ckpt")
    save_model(ours, S, T, w)
    R.save_model(theirs, R.EmbeddingMatrix(S.values), R.EmbeddingMatrix(T.values), w)
    assert open(ours, "rb").read() == open(theirs, "rb").read()
    s2, t2, w2 = R.load_model(ours)
    assert s2.values.tobytes() == S.values.tobytes() and w2.tobytes() == w.tobytes()
