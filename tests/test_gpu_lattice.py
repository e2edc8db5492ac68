"""FSA lattices from the GPU vs the reference's fsa_beam_search lattices
(SURVEY.md §8f row 2): identical node numbering, arc order, labels,
destinations and fp64 arc scores (bit-equal: the device log-softmax is the
reference's own arithmetic), hence byte-identical serialize_fsa_text /
serialize_lattice output (fsa.hpp:243-262, fsa_search.hpp:429-435)."""
import numpy as np
import pytest

from oracle.py_oracle import synthetic_arpa
from tests import helpers as H
from tests.test_oracle_vs_reference import _parse_lattice

pytestmark = pytest.mark.gpu


def _compare(dec, m, feats, enc, splits, rg, params):
    from paper_2211_00484_b200.api import FsaParams, Graph

    g = rg.g
    dg = Graph(dec, g.num_states, g.arc_splits, g.dst, g.label, g.weight)
    dec.fsa_beam_search(enc, splits, dg, FsaParams(*params))
    _, _, texts = m.fsa(feats, splits, rg, *params, lattice_texts=True)
    for s, text in enumerate(texts):
        arcs, finals = _parse_lattice(text)
        lat = dec.fsa_lattice(s)
        assert finals == {lat["num_nodes"] - 1: 0.0}
        assert len(arcs) == len(lat["src"])
        mine = list(zip(lat["src"].tolist(), lat["dst"].tolist(), lat["label"].tolist()))
        assert mine == [a[:3] for a in arcs]
        want = np.array([a[3] for a in arcs])
        H.assert_scores_equal(lat["score"], want)
        assert dec.fsa_lattice_text(s) == text
        T = int(splits[s + 1] - splits[s])
        assert dec.fsa_lattice_text(s, header=True) == f"# stream={s} frames={T}\n" + text


def test_trivial_graph_lattices_match_reference():
    from paper_2211_00484_b200.api import Decoder

    m = H.model(V=500, seed=1, blank_bias=0.4)
    dec = Decoder(H.api_weights(m.w))
    feats, enc, splits = H.frames(m, [25, 0, 9, 25, 1], seed0=71)
    _compare(dec, m, feats, enc, splits, H.ref().graph_trivial(500), (4.0, 8, 4))
    dec.close()


def test_ngram_graph_lattices_match_reference():
    from paper_2211_00484_b200.api import Decoder

    m = H.model(V=500, seed=1, blank_bias=-1.4)
    dec = Decoder(H.api_weights(m.w))
    rg = H.ref().graph_from_arpa(synthetic_arpa(500, 300, 600), 500)
    feats, enc, splits = H.frames(m, [12, 6], seed0=81)
    _compare(dec, m, feats, enc, splits, rg, (8.0, 64, 8))
    dec.close()
