"""FSA fast beam search on the GPU vs the oracle and the compiled reference.

Token sequences must be identical; best-path scores bit-equal (the device
log-softmax is the reference's index-order sum with glibc exp / log).  Graphs: the trivial graph (config 3), the seeded
synthetic trigram LG-style graph (config 4 shape), and small hand graphs with
parallel arcs / multiple states (the reference's fsa_search_test.cpp
fixtures re-expressed through the public search)."""
import functools

import numpy as np
import pytest

from oracle.py_oracle import synthetic_arpa
from tests import helpers as H

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def big():
    from paper_2211_00484_b200.api import Decoder

    m = H.model(V=500, seed=1, blank_bias=0.4)
    dec = Decoder(H.api_weights(m.w))
    yield m, dec
    dec.close()


@functools.lru_cache(maxsize=2)
def ngram_graph(V=500):
    return H.ref().graph_from_arpa(synthetic_arpa(V), V)


def _dev_graph(dec, g):
    from paper_2211_00484_b200.api import Graph

    return Graph(dec, g.num_states, g.arc_splits, g.dst, g.label, g.weight)


def _check(m, dec, dg, og, feats, enc, splits, beam, ms, mc, ref_graph=None):
    from paper_2211_00484_b200.api import FsaParams

    want, want_sc, _ = H.orc().fsa(m.w, enc, splits, og, beam, ms, mc)
    got, sc = dec.fsa_beam_search(enc, splits, dg, FsaParams(beam, ms, mc))
    assert got == want
    H.assert_scores_equal(sc, want_sc)
    if ref_graph is not None:
        rt, rs, _ = m.fsa(feats, splits, ref_graph, beam, ms, mc)
        assert rt == want
        np.testing.assert_allclose(rs, want_sc, rtol=0, atol=0)
    return got


def test_trivial_graph_config3_shape(big):
    """Config 3: trivial graph, beam 4, max_states 8, max_contexts 4."""
    from paper_2211_00484_b200.api import Graph

    m, dec = big
    tg = H.ref().graph_trivial(500)
    dg = Graph.trivial(dec)
    Ts = [50] * 12 + [0, 1, 13]
    feats, enc, splits = H.frames(m, Ts, seed0=4000)
    got = _check(m, dec, dg, tg.g, feats, enc, splits, 4.0, 8, 4, ref_graph=tg)
    assert got[12] == []
    st = dec.stats()
    assert st["arcs_expanded"] > 0 and st["lattice_arcs"] > 0


def test_trivial_graph_many_streams(big):
    from paper_2211_00484_b200.api import Graph

    m, dec = big
    tg = H.ref().graph_trivial(500)
    dg = Graph.trivial(dec)
    Ts = [int(x) for x in np.random.default_rng(3).integers(10, 40, 512)]
    feats, enc, splits = H.frames(m, Ts, seed0=9000)
    _check(m, dec, dg, tg.g, feats, enc, splits, 4.0, 8, 4)


@pytest.mark.parametrize("params", [(8.0, 64, 8), (8.0, 8, 4), (20.0, 64, 8)])
def test_ngram_graph(params):
    from paper_2211_00484_b200.api import Decoder

    m = H.model(V=500, seed=1, blank_bias=-1.4)
    dec = Decoder(H.api_weights(m.w))
    rg = ngram_graph()
    assert rg.g.num_arcs > 900_000
    dg = _dev_graph(dec, rg.g)
    Ts = [30] * 6 + [0, 7]
    feats, enc, splits = H.frames(m, Ts, seed0=600)
    _check(m, dec, dg, rg.g, feats, enc, splits, *params, ref_graph=rg if params[1] == 8 else None)
    dec.close()


def test_small_graphs_toy_models():
    """Multi-state graphs with parallel arcs and non-zero weights on toy
    vocabularies; exercises merges of duplicate (ctx, state) targets."""
    from paper_2211_00484_b200.api import Decoder

    rng = np.random.default_rng(7)
    for seed, V in [(11, 4), (12, 5), (13, 3)]:
        m = H.ref().model(V, 4, 8, 8, 8, seed, -0.5)
        dec = Decoder(H.api_weights(m.w))
        S = 3
        src, dst, lab, w = [], [], [], []
        for s in range(S):
            for _ in range(2 * V):
                src.append(s)
                dst.append(int(rng.integers(S)))
                lab.append(int(rng.integers(1, V)))
                w.append(float(rng.uniform(-1.0, 0.0)))
        rg = H.ref().graph_from_arcs(S, src, dst, lab, w, {0: 0.0})
        dg = _dev_graph(dec, rg.g)
        Ts = [2, 3, 5, 8, 0, 1]
        feats, enc, splits = H.frames(m, Ts, seed0=seed)
        for params in [(1e9, 64, 64), (2.0, 4, 2), (0.5, 2, 1), (0.0, 1, 1)]:
            _check(m, dec, dg, rg.g, feats, enc, splits, *params, ref_graph=rg)
        dec.close()


def test_fsa_invalid_params(big):
    from paper_2211_00484_b200.api import FsaParams, Graph, ValidationError

    m, dec = big
    dg = Graph.trivial(dec)
    _, enc, splits = H.frames(m, [4])
    for p in [FsaParams(-1.0, 8, 4), FsaParams(4.0, 0, 4), FsaParams(4.0, 8, 0)]:
        with pytest.raises(ValidationError):
            dec.fsa_beam_search(enc, splits, dg, p)
    with pytest.raises(ValidationError):
        Graph(dec, 1, np.array([0, 1], np.int32), np.zeros(1, np.int32), np.zeros(1, np.int32), np.zeros(1))
    with pytest.raises(ValidationError):
        Graph(dec, 1, np.array([0, 1], np.int32), np.zeros(1, np.int32), np.array([500], np.int32), np.zeros(1))


def test_graph_outlives_its_model():
    """A graph destroyed after its model (any order, as garbage collection
    goes) is detached, not a use-after-free; a second model refuses it."""
    from paper_2211_00484_b200.api import Decoder, FsaParams, Graph, ValidationError

    m = H.ref().model(6, 4, 8, 8, 8, 3, -0.5)
    dec, dec2 = Decoder(H.api_weights(m.w)), Decoder(H.api_weights(m.w))
    g = Graph.trivial(dec)
    g2 = Graph.trivial(dec)
    _, enc, splits = H.frames(m, [5, 3], seed0=11)
    with pytest.raises(ValidationError):
        dec2.fsa_beam_search(enc, splits, g, FsaParams(4.0, 8, 4))
    dec.close()
    del g  # after its model
    with pytest.raises(ValidationError):
        dec2.fsa_beam_search(enc, splits, g2, FsaParams(4.0, 8, 4))
    g2.__del__()
    dec2.close()


def test_lattice_pool_overflow_regrows_and_device_frames(big, monkeypatch):
    """A lattice pool far too small for the call: every stream's lattice
    overflows, best path is skipped for the incomplete lattices, the host
    regrows the pool and decodes again — same tokens / scores as a call with
    a large pool, for host and for device-resident frames."""
    import torch

    from paper_2211_00484_b200.api import FsaParams, Graph

    m, dec = big
    feats, enc, splits = H.frames(m, [60] * 40, seed0=61000)
    g = Graph.trivial(dec)
    want, want_sc = dec.fsa_beam_search(enc, splits, g, FsaParams(4.0, 8, 4))
    monkeypatch.setenv("RNNTG_LAT_CAP", "1024")
    got, sc = dec.fsa_beam_search(enc, splits, g, FsaParams(4.0, 8, 4))
    assert got == want and np.array_equal(sc, want_sc)
    d_enc = torch.from_numpy(enc).cuda()
    tok = torch.zeros(int(splits[-1]), dtype=torch.int32, device="cuda")
    dsc = torch.zeros(len(splits) - 1, dtype=torch.float64, device="cuda")
    osp, tok, dsc = dec.fsa_beam_search(d_enc, splits, g, FsaParams(4.0, 8, 4), tok, dsc)
    t = tok.cpu().numpy()
    assert [t[osp[i] : osp[i + 1]].tolist() for i in range(len(splits) - 1)] == want
    assert np.array_equal(dsc.cpu().numpy(), want_sc)
    monkeypatch.delenv("RNNTG_LAT_CAP")
    osp, tok, dsc = dec.fsa_beam_search(d_enc, splits, g, FsaParams(4.0, 8, 4), tok, dsc)
    assert np.array_equal(dsc.cpu().numpy(), want_sc)
