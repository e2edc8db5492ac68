"""Shared fixtures: seeded reference models, encoder frames and graphs.

Inputs follow SURVEY.md §8(d): init_model weights (DetRng), blank bias on
out_b[0], features ~ DetRng(seed + stream).gaussian(), encoder frames from
the reference encoder (identical bits go to both sides)."""
from __future__ import annotations

import functools
import os

import numpy as np

from oracle.py_oracle import Graph as OGraph
from oracle.py_oracle import Oracle, Reference, Weights

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@functools.lru_cache(maxsize=1)
def ref():
    return Reference()


@functools.lru_cache(maxsize=1)
def orc():
    return Oracle()


@functools.lru_cache(maxsize=8)
def model(V=500, F=80, D=512, E=512, J=512, seed=1, blank_bias=0.4):
    return ref().model(V, F, D, E, J, seed, blank_bias)


def frames(m, Ts, seed0=1000):
    """(features, encoder frames, frame_splits) for streams of lengths Ts."""
    F = m.w.F
    splits = np.zeros(len(Ts) + 1, np.int32)
    splits[1:] = np.cumsum(Ts)
    feats = np.concatenate([ref().features(seed0 + i, T, F) for i, T in enumerate(Ts)] + [np.zeros((0, F), np.float32)])
    enc = m.encoder(feats, splits)
    return feats, enc, splits


def api_weights(w: Weights):
    from paper_2211_00484_b200.api import ModelWeights

    return ModelWeights.from_dict(w.p)


def decoder_env(m, **env):
    """A Decoder created with the given RNNTG_* environment switches set (they
    are read when the model is created), the environment restored after."""
    from paper_2211_00484_b200.api import Decoder

    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        return Decoder(api_weights(m.w))
    finally:
        for k, v in old.items():
            if v is None:
                del os.environ[k]
            else:
                os.environ[k] = v


def assert_scores_equal(got, want):
    """fp64 scores bit-equal to the reference's (exact log-softmax: the
    reference's index-order sum with glibc exp / log, glibc_f64.h)."""
    g = np.asarray(got, np.float64)
    w = np.asarray(want, np.float64)
    assert g.shape == w.shape, (g.shape, w.shape)
    bad = np.flatnonzero(g.view(np.int64) != w.view(np.int64))
    assert bad.size == 0, f"{bad.size} scores differ, first {bad[:4].tolist()}: {g[bad[:4]]} vs {w[bad[:4]]}"


def ref_logits(m, n, seed=0):
    """n real joiner rows of the reference (encoder frames x random contexts)."""
    _, enc, _ = frames(m, [n], seed0=seed)
    V = m.w.V
    ctx = np.random.default_rng(seed).integers(0, V * V, n).astype(np.int32)
    return m.joiner_logits(enc, ctx)
