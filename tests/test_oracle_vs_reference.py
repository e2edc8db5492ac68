"""Pins the C restatement (oracle/rnnt_oracle.cpp) to the compiled reference
(oracle/_ref/librnnt_ref.so, built from /root/reference by oracle/Makefile).

CPU only; sizes chosen so the whole file runs in well under a minute.  These
are the differential runs that pin V=500/D=512 behaviour, which the
reference's own unit fixtures (toy V<=8) do not cover."""
import numpy as np
import pytest

from oracle.py_oracle import synthetic_arpa
from tests import helpers as H


@pytest.fixture(scope="module")
def m500():
    return H.model(V=500, seed=1, blank_bias=0.4)


def test_encoder_bit_exact(m500):
    feats, enc, splits = H.frames(m500, [9])
    mine = H.orc().encoder(m500.w, feats)
    assert np.array_equal(mine.view(np.uint32), enc.view(np.uint32))


def test_joiner_pieces_bit_exact(m500):
    _, enc, _ = H.frames(m500, [6])
    ctxs = np.array([0, 7, 500, 1234, 249999, 31337], np.int32)
    pd = H.orc().decoder_project(m500.w, ctxs)
    assert np.array_equal(pd.view(np.uint32), m500.decoder_project(ctxs).view(np.uint32))
    pe = H.orc().affine(m500.w.p["j_we"], None, enc)
    lo = H.orc().joiner_logits(m500.w, pe, pd)
    assert np.array_equal(lo.view(np.uint32), m500.joiner_logits(enc, ctxs).view(np.uint32))
    assert np.array_equal(H.orc().log_softmax(lo), H.ref().log_softmax(lo))


def test_greedy_matches_reference(m500):
    feats, enc, splits = H.frames(m500, [40, 0, 25, 3, 40, 40])
    assert H.orc().greedy(m500.w, enc, splits) == m500.greedy(feats, splits)


@pytest.mark.parametrize("merge_op,ln,cap", [(0, 0, 0), (1, 0, 0), (0, 1, 0), (0, 0, 2)])
def test_beam_matches_reference(m500, merge_op, ln, cap):
    feats, enc, splits = H.frames(m500, [20, 0, 12, 20], seed0=50)
    got, _ = H.orc().beam(m500.w, enc, splits, beam=4, merge_op=merge_op, length_norm=ln, max_total=cap)
    assert got == m500.beam(feats, splits, beam=4, merge_op=merge_op, length_norm=ln, max_total=cap)


def test_beam_toy_models():
    for seed, V, bias in [(400, 4, -1.0), (401, 4, 0.0), (500, 3, -1.5)]:
        m = H.ref().model(V, 4, 8, 8, 8, seed, bias)
        feats, enc, splits = H.frames(m, [3, 4, 5, 6, 7], seed0=seed)
        for beam in (1, 2, 4, 8):
            for mo in (0, 1):
                got, _ = H.orc().beam(m.w, enc, splits, beam=beam, merge_op=mo)
                assert got == m.beam(feats, splits, beam=beam, merge_op=mo)


def _parse_lattice(text):
    arcs, finals = [], {}
    for line in text.splitlines():
        if not line or line.startswith("#"):
            continue
        f = line.split()
        if len(f) == 4:
            arcs.append((int(f[0]), int(f[1]), int(f[2]), float(f[3])))
        else:
            finals[int(f[0])] = float(f[1])
    return arcs, finals


def _check_fsa(m, feats, enc, splits, rg, params):
    got, sc, lats = H.orc().fsa(m.w, enc, splits, rg.g, *params, lattices=True)
    want, wsc, texts = m.fsa(feats, splits, rg, *params, lattice_texts=True)
    assert got == want
    assert np.array_equal(sc, wsc)
    for lat, text in zip(lats, texts):
        arcs, finals = _parse_lattice(text)
        mine = list(zip(lat["src"].tolist(), lat["dst"].tolist(), lat["label"].tolist(), lat["score"].tolist()))
        assert mine == arcs
        assert finals == {lat["num_nodes"] - 1: 0.0}


def test_fsa_trivial_matches_reference(m500):
    feats, enc, splits = H.frames(m500, [15, 0, 9, 15], seed0=70)
    tg = H.ref().graph_trivial(500)
    _check_fsa(m500, feats, enc, splits, tg, (4.0, 8, 4))


def test_fsa_ngram_matches_reference():
    m = H.model(V=500, seed=1, blank_bias=-1.4)
    rg = H.ref().graph_from_arpa(synthetic_arpa(500, 300, 600), 500)
    feats, enc, splits = H.frames(m, [10, 4], seed0=80)
    _check_fsa(m, feats, enc, splits, rg, (8.0, 64, 8))


def test_fsa_toy_graph_matches_reference():
    rng = np.random.default_rng(3)
    m = H.ref().model(4, 4, 8, 8, 8, 21, -0.5)
    S = 3
    src = [s for s in range(S) for _ in range(6)]
    dst = [int(rng.integers(S)) for _ in src]
    lab = [int(rng.integers(1, 4)) for _ in src]
    w = [float(rng.uniform(-1, 0)) for _ in src]
    rg = H.ref().graph_from_arcs(S, src, dst, lab, w, {1: 0.0})
    feats, enc, splits = H.frames(m, [1, 4, 6, 0], seed0=5)
    for params in [(1e9, 1 << 30, 1 << 30), (1.0, 3, 2), (0.0, 1, 1)]:
        _check_fsa(m, feats, enc, splits, rg, params)
