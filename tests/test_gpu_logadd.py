"""lattice_to_best_seq(kLogAdd) on the GPU (
fsa_search.hpp:410-425, fsa.hpp:390-463, 533-540) against the reference's
own function on the reference's lattices of the same streams: identical
sequences, and bit-equal total log-probabilities of the chosen sequence
(the reference's sequence_total_logprob), for several seeds and n-best
sizes, ragged streams (including a zero-frame stream), the trivial graph
and an n-gram graph; the BASELINE config 3 / 4 shapes are in
test_gpu_configs.py."""
import numpy as np
import pytest

from oracle.py_oracle import synthetic_arpa
from tests import helpers as H

pytestmark = pytest.mark.gpu


def _check(dec, m, feats, enc, splits, g, rg, params, nbests=(100,), seeds=(0, 7)):
    from paper_2211_00484_b200.api import FsaParams

    dec.fsa_beam_search(enc, splits, g, FsaParams(*params))
    for nb in nbests:
        for seed in seeds:
            got, glp = dec.fsa_lattice_best(nbest=nb, seed=seed)
            want, wlp = m.fsa_logadd(feats, splits, rg, *params, nbest=nb, seed=seed)
            bad = [i for i, (a, b) in enumerate(zip(got, want)) if a != b]
            assert not bad, (nb, seed, bad[:8])
            H.assert_scores_equal(glp, wlp)


def test_logadd_trivial_graph():
    from paper_2211_00484_b200.api import Decoder, Graph

    m = H.model(V=500, seed=1, blank_bias=0.4)
    dec = Decoder(H.api_weights(m.w))
    feats, enc, splits = H.frames(m, [40, 0, 9, 40, 1, 25], seed0=171)
    _check(dec, m, feats, enc, splits, Graph.trivial(dec), H.ref().graph_trivial(500), (4.0, 8, 4),
           nbests=(1, 7, 100), seeds=(0, 7, 12345))
    dec.close()


def test_logadd_wide_beam_many_alignments():
    """A wide search (beam 12, 32 states, 16 contexts): many alignments per
    sequence, so the per-sequence totals sum over many paths."""
    from paper_2211_00484_b200.api import Decoder, Graph

    m = H.model(V=500, seed=2, blank_bias=0.2)
    dec = Decoder(H.api_weights(m.w))
    feats, enc, splits = H.frames(m, [30, 17, 30], seed0=271)
    _check(dec, m, feats, enc, splits, Graph.trivial(dec), H.ref().graph_trivial(500), (12.0, 32, 16))
    dec.close()


def test_logadd_ngram_graph():
    from paper_2211_00484_b200.api import Decoder, Graph

    m = H.model(V=500, seed=1, blank_bias=-1.4)
    rg = H.ref().graph_from_arpa(synthetic_arpa(500, 300, 600), 500)
    g0 = rg.g
    dec = Decoder(H.api_weights(m.w))
    g = Graph(dec, g0.num_states, g0.arc_splits, g0.dst, g0.label, g0.weight)
    feats, enc, splits = H.frames(m, [25, 12, 0, 25], seed0=371)
    _check(dec, m, feats, enc, splits, g, rg, (8.0, 64, 8))
    dec.close()


def test_logadd_validation():
    from paper_2211_00484_b200.api import Decoder, ValidationError

    m = H.model(V=500, seed=1, blank_bias=0.4)
    dec = Decoder(H.api_weights(m.w))
    with pytest.raises(ValidationError):
        dec.fsa_lattice_best()  # no FSA decode on this handle yet
    from paper_2211_00484_b200.api import FsaParams, Graph

    feats, enc, splits = H.frames(m, [5], seed0=5)
    dec.fsa_beam_search(enc, splits, Graph.trivial(dec), FsaParams(4.0, 8, 4))
    with pytest.raises(ValidationError, match="nbest_n must be >= 1"):
        dec.fsa_lattice_best(nbest=0)
    dec.close()
