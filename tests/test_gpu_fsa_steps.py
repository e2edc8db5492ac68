"""The Algorithm-1 step API on the GPU (rnntg_fsa_stream_*; fsa_search.hpp:
95-297, the plug-in point of expand_arcs, 59-61) against the reference's
own init_streams / get_contexts / expand_arcs + prune_streams, driven
step by step with identical caller log-prob rows: the same contexts at every
step and byte-identical lattices, best sequences and scores at the end.
Plus the reference's step-API KATs that start from init_streams
(fsa_search_test.cpp:140-165 expansion, 309-338 invariants) and the stale
get_contexts error.  The whole toy-model decode through the step API equals
the reference's fsa_beam_search."""
import numpy as np
import pytest

from oracle.py_oracle import RefSteps
from tests import helpers as H

pytestmark = pytest.mark.gpu
BIG = 2**31 - 1


def _rows(ctx, t, V, salt):
    """Deterministic caller rows: a log-softmax of seeded normals per (frame,
    context) -- fsa_search_test.cpp's random_logprob_rows, made a function of
    the row's identity so both decoders see the same row."""
    out = np.empty((len(ctx), V))
    for r, c in enumerate(ctx):
        z = np.random.default_rng([salt, t, int(c)]).normal(size=V)
        mx = z.max()
        out[r] = z - (mx + np.log(np.exp(z - mx).sum()))
    return out


def _graph_pair(dec, ref, kind, V):
    from paper_2211_00484_b200.api import Graph

    if kind == "trivial":
        return Graph.trivial(dec), ref.graph_trivial(V)
    if kind == "merge":  # fsa_search_test.cpp:171: one arc 0 -> 1 labeled 2, weight -0.25
        src, dst, lab, w = [0], [1], [2], [-0.25]
        n = 2
    else:  # 3 states, parallel arcs, weights
        rng = np.random.default_rng(5)
        src, dst, lab, w = [], [], [], []
        for s_ in range(3):
            for c in range(1, V):
                for _ in range(1 + (c + s_) % 2):
                    src.append(s_)
                    dst.append(int(rng.integers(0, 3)))
                    lab.append(c)
                    w.append(float(-rng.uniform(0, 1)))
        n = 3
    order = np.argsort(np.asarray(src), kind="stable")
    src = np.asarray(src, np.int32)[order]
    dst = np.asarray(dst, np.int32)[order]
    lab = np.asarray(lab, np.int32)[order]
    w = np.asarray(w, np.float64)[order]
    splits = np.searchsorted(src, np.arange(n + 1)).astype(np.int32)
    return Graph(dec, n, splits, dst, lab, w), ref.graph_from_arcs(n, src, dst, lab, w, {n - 1: 0.0})


@pytest.mark.parametrize("kind,V,params", [
    ("trivial", 4, (1e9, BIG, BIG)),
    ("trivial", 6, (4.0, 8, 4)),
    ("trivial", 5, (0.5, 2, 1)),
    ("merge", 3, (1e9, BIG, BIG)),
    ("multi", 5, (20.0, 64, 8)),
    ("multi", 4, (2.0, 5, 2)),
])
def test_steps_match_reference(kind, V, params):
    from paper_2211_00484_b200.api import Decoder, FsaParams

    ref = H.ref()
    m = H.model(V=V, F=4, D=8, E=8, J=8, seed=11, blank_bias=0.0)
    dec = Decoder(H.api_weights(m.w))
    g, rg = _graph_pair(dec, ref, kind, V)
    nf = [6, 0, 3, 9, 1]
    dec.fsa_stream_begin(g, FsaParams(*params), nf)
    rs = RefSteps(ref, rg, params, V, nf)
    for t in range(max(nf)):
        gs, gc = dec.fsa_stream_contexts()
        ws, wc = rs.contexts()
        assert np.array_equal(gs, ws) and np.array_equal(gc, wc), t
        lp = _rows(gc, t, V, 77)
        dec.fsa_stream_step(lp)
        rs.step(lp)
    gs, gc = dec.fsa_stream_contexts()
    assert gs[-1] == 0  # every stream past its last frame
    toks, sc = dec.fsa_stream_end()
    wt, wsc, wtexts = rs.end()
    assert toks == wt
    H.assert_scores_equal(sc, wsc)
    assert [dec.fsa_lattice_text(i) for i in range(len(nf))] == wtexts
    dec.close()


def test_expansion_kat_from_init():
    """fsa_search_test.cpp:140-165: V = 2, trivial graph, unpruned; one
    step with rows [-0.7, -0.4]: a blank candidate (ctx 0) at -0.7 and a
    token candidate (ctx 1) at -0.4, each with its lattice arc."""
    from paper_2211_00484_b200.api import Decoder, FsaParams, Graph

    m = H.model(V=2, F=4, D=8, E=8, J=8, seed=3, blank_bias=0.0)
    dec = Decoder(H.api_weights(m.w))
    dec.fsa_stream_begin(Graph.trivial(dec), FsaParams(1e9, BIG, BIG), [1])
    rs, ctx = dec.fsa_stream_contexts()
    assert rs.tolist() == [0, 1] and ctx.tolist() == [0]
    dec.fsa_stream_step(np.array([[-0.7, -0.4]]))
    toks, sc = dec.fsa_stream_end()
    assert dec.fsa_lattice_text(0) == "0 1 0 -0.7\n0 2 1 -0.4\n1 3 0 0\n2 3 0 0\n3 0\n"
    assert toks == [[1]] and sc[0] == -0.4
    dec.close()


def test_stale_contexts_is_a_logic_error():
    """expand_arcs with stale get_contexts data is std::logic_error
    (fsa_search.hpp:164-180) -> RNNTG_INTERNAL."""
    from paper_2211_00484_b200.api import Decoder, FsaParams, Graph, LogicError

    m = H.model(V=3, F=4, D=8, E=8, J=8, seed=3, blank_bias=0.0)
    dec = Decoder(H.api_weights(m.w))
    dec.fsa_stream_begin(Graph.trivial(dec), FsaParams(1e9, BIG, BIG), [2])
    with pytest.raises(LogicError, match="stale get_contexts"):
        dec.fsa_stream_step(np.zeros((1, 3)))
    dec.close()


def test_toy_model_decode_through_steps_equals_fsa_beam_search():
    """The reference's own driver (fsa_search.hpp:326-387) re-run through the
    step API: each step's rows are the toy model's log-softmax of the
    joiner logits of (frame, context) -- computed by the GPU decoder's
    kernel-level entry points -- and the lattices equal fsa_beam_search's."""
    from paper_2211_00484_b200.api import Decoder, FsaParams, Graph, log_softmax_lse

    m = H.model(V=500, seed=1, blank_bias=0.4)
    feats, enc, splits = H.frames(m, [12, 0, 7], seed0=901)
    dec = Decoder(H.api_weights(m.w))
    g = Graph.trivial(dec)
    p = FsaParams(4.0, 8, 4)
    nf = np.diff(splits)
    dec.fsa_stream_begin(g, p, nf)
    for t in range(int(nf.max())):
        rs, ctx = dec.fsa_stream_contexts()
        rows_enc = np.concatenate([np.repeat(enc[splits[i] + t : splits[i] + t + 1], rs[i + 1] - rs[i], 0)
                                   for i in range(len(nf)) if rs[i + 1] > rs[i]] or [np.zeros((0, 512), np.float32)])
        logits = dec.joiner_logits(rows_enc, ctx) if len(ctx) else np.zeros((0, 500), np.float32)
        lse = log_softmax_lse(logits) if len(ctx) else np.zeros(0)
        dec.fsa_stream_step(logits.astype(np.float64) - lse[:, None])
    toks, sc = dec.fsa_stream_end()
    texts = [dec.fsa_lattice_text(i) for i in range(len(nf))]
    want, wsc, wtexts = m.fsa(feats, splits, H.ref().graph_trivial(500), 4.0, 8, 4, lattice_texts=True)
    assert toks == want
    H.assert_scores_equal(sc, wsc)
    assert texts == wtexts
    dec.close()
