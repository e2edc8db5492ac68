"""The reference's own FSA-search property tests, re-expressed through the
public GPU search (fsa_search_test.cpp).

The reference checks its lattices against exact DP oracles on small random
models (enc/emb/joiner dims 8, feat dim 4, V = 2..6), batching and order
transparency with a zero-frame stream, and the graph-weight shift.  Here the
same models and graphs go through the GPU decoder and every lattice must be
byte-identical (serialize_fsa_text) to the reference's own on the same
inputs -- which carries the reference's DP-oracle guarantees over -- plus the
properties themselves where they are stated on the GPU output.  (The step-API
KATs of fsa_search_test.cpp:104-307 feed hand-made log-prob rows through
init_streams / expand_arcs / prune_streams, which the GPU decoder does not
expose: out of scope.)"""
import numpy as np
import pytest

from tests import helpers as H

pytestmark = pytest.mark.gpu

BIG = 2**31 - 1


def _small(seed, V, blank_bias=0.0):
    return H.ref().model(V, 4, 8, 8, 8, seed, blank_bias)  # oracle::random_model(seed, V, 4)


def _trivial(dec, ref, V):
    from paper_2211_00484_b200.api import Graph

    return Graph.trivial(dec), ref.graph_trivial(V)


def _texts(dec, n):
    return [dec.fsa_lattice_text(i) for i in range(n)]


def test_unpruned_trivial_graph_matches_reference_lattices():
    """fsa_search_test.cpp:340-362: 50 models, V = 2..6, T = 3..12,
    unpruned search (beam 1e9, no state / context caps).  The reference
    checks total_logprob against the S = 1 log-add DP and best_path against
    Viterbi; here every GPU lattice equals the reference's byte for byte, and
    the log-add best sequence equals the reference's."""
    from paper_2211_00484_b200.api import Decoder, FsaParams, UnsupportedError

    ref = H.ref()
    checked = 0
    for seed in range(50):
        V = 2 + seed % 5
        T = 3 + seed % 10
        m = _small(seed, V)
        feats = ref.features(10_000 + seed, T, 4)
        splits = np.array([0, T], np.int32)
        enc = m.encoder(feats, splits)
        dec = Decoder(H.api_weights(m.w))
        g, rg = _trivial(dec, ref, V)
        try:
            toks, sc = dec.fsa_beam_search(enc, splits, g, FsaParams(1e9, BIG, BIG))
        except UnsupportedError:
            # > 32 distinct contexts in one CTA frame (V = 6 has 36): a device cap
            assert V == 6
            dec.close()
            continue
        want, wsc, wtexts = m.fsa(feats, splits, rg, 1e9, BIG, BIG, lattice_texts=True)
        assert toks == want, seed
        H.assert_scores_equal(sc, wsc)
        assert _texts(dec, 1) == wtexts, seed
        lt, llp = dec.fsa_lattice_best(nbest=100, seed=seed)
        rt, rlp = m.fsa_logadd(feats, splits, rg, 1e9, BIG, BIG, nbest=100, seed=seed)
        assert lt == rt, seed
        H.assert_scores_equal(llp, rlp)
        dec.close()
        checked += 1
    assert checked >= 40


def test_batch_composition_and_order_transparency():
    """fsa_search_test.cpp:364-393: streams T = 3..10 plus a zero-frame
    stream, default pruned parameters; decoded together, alone and in reverse
    order the lattices are identical (and the reference's); the zero-frame
    stream accepts only the empty sequence at score 0."""
    from paper_2211_00484_b200.api import Decoder, FsaParams

    ref = H.ref()
    m = _small(1234, 4, -0.5)
    Ts = list(range(3, 11)) + [0]
    feats = np.concatenate([ref.features(20_000 + i, T, 4) for i, T in enumerate(Ts)])
    splits = np.zeros(len(Ts) + 1, np.int32)
    splits[1:] = np.cumsum(Ts)
    enc = m.encoder(feats, splits)
    p = FsaParams()  # FsaSearchParams defaults (20, 64, 8)
    dec = Decoder(H.api_weights(m.w))
    g, rg = _trivial(dec, ref, 4)
    toks, sc = dec.fsa_beam_search(enc, splits, g, p)
    together = _texts(dec, len(Ts))
    solo = []
    for i, T in enumerate(Ts):
        s1 = np.array([0, T], np.int32)
        dec.fsa_beam_search(enc[splits[i] : splits[i + 1]], s1, g, p)
        solo.append(dec.fsa_lattice_text(0))
    rsplits = np.zeros(len(Ts) + 1, np.int32)
    rsplits[1:] = np.cumsum(Ts[::-1])
    renc = np.concatenate([enc[splits[i] : splits[i + 1]] for i in reversed(range(len(Ts)))])
    dec.fsa_beam_search(renc, rsplits, g, p)
    reversed_texts = _texts(dec, len(Ts))[::-1]
    assert together == solo == reversed_texts
    _, _, wtexts = m.fsa(feats, splits, rg, p.beam, p.max_states, p.max_contexts, lattice_texts=True)
    assert together == wtexts
    assert toks[-1] == [] and sc[-1] == 0.0
    assert together[-1] == "0 1 0 0\n1 0\n"
    dec.close()


def test_graph_weights_add_onto_lattice_arcs():
    """fsa_search_test.cpp:395-430: every arc of the trivial graph shifted by
    delta: same lattice structure, label arcs shifted by delta (blank arcs
    unchanged), and both lattices equal the reference's."""
    from paper_2211_00484_b200.api import Decoder, FsaParams, Graph

    ref = H.ref()
    m = _small(777, 4)
    feats = ref.features(30_000, 5, 4)
    splits = np.array([0, 5], np.int32)
    enc = m.encoder(feats, splits)
    delta = 0.7
    V = 4
    labels = np.arange(1, V, dtype=np.int32)
    base = dict(num_states=1, arc_splits=np.array([0, V - 1], np.int32), dst=np.zeros(V - 1, np.int32),
                label=labels, weight=np.zeros(V - 1))
    dec = Decoder(H.api_weights(m.w))
    p = FsaParams(1e9, BIG, BIG)
    lats, texts = [], []
    for shift in (0.0, delta):
        g = Graph(dec, base["num_states"], base["arc_splits"], base["dst"], base["label"], base["weight"] + shift)
        dec.fsa_beam_search(enc, splits, g, p)
        lats.append(dec.fsa_lattice(0))
        texts.append(dec.fsa_lattice_text(0))
        rg = ref.graph_from_arcs(1, np.zeros(V - 1, np.int32), np.zeros(V - 1, np.int32), labels,
                                 np.zeros(V - 1) + shift, {0: 0.0})
        _, _, wt = m.fsa(feats, splits, rg, p.beam, p.max_states, p.max_contexts, lattice_texts=True)
        assert texts[-1] == wt[0]
    a, b = lats
    for k in ("src", "dst", "label"):
        assert np.array_equal(a[k], b[k])
    want = np.where(a["label"] == 0, 0.0, delta)
    np.testing.assert_allclose(b["score"] - a["score"], want, rtol=0, atol=1e-12)
    dec.close()
