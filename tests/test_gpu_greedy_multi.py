"""greedy_search with S > 1 symbols per frame (search.hpp:76-100), batched
over streams on the GPU, against the compiled reference's greedy_search on
identical inputs: tokens identical, and the frames stopped by the 10-symbol
safety cap (S unlimited) counted identically."""
import numpy as np
import pytest

from tests import helpers as H

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dec_model():
    from paper_2211_00484_b200.api import Decoder

    # blank bias 0: ~1 emission per frame, so S matters
    m = H.model(V=500, seed=5, blank_bias=0.0)
    dec = Decoder(H.api_weights(m.w))
    yield m, dec
    dec.close()


@pytest.mark.parametrize("S", [1, 2, 3, 7])
def test_greedy_multi_symbol_matches_reference(dec_model, S):
    m, dec = dec_model
    Ts = [int(x) for x in np.random.default_rng(S).integers(0, 40, 37)]
    feats, enc, splits = H.frames(m, Ts, seed0=4000 + S)
    want, _ = m.greedy_multi(feats, splits, S)
    got, capped = dec.greedy_search(enc, splits, S)
    assert got == want
    assert capped == 0
    assert max(len(y) - S * T for y, T in zip(got, Ts)) <= 0
    if S == 1:  # greedy_search(S=1) == greedy_search_batch
        assert got == dec.greedy_search_batch(enc, splits)


def test_greedy_unlimited_counts_capped_frames():
    from paper_2211_00484_b200.api import NO_SYMBOL_LIMIT, Decoder

    # strong negative blank bias: the model keeps emitting, the safety cap binds
    m = H.model(V=500, seed=6, blank_bias=-3.0)
    dec = Decoder(H.api_weights(m.w))
    try:
        Ts = [12, 0, 5, 20]
        feats, enc, splits = H.frames(m, Ts, seed0=5100)
        want, want_capped = m.greedy_multi(feats, splits, NO_SYMBOL_LIMIT)
        got, capped = dec.greedy_search(enc, splits, NO_SYMBOL_LIMIT)
        assert got == want
        assert capped == want_capped and capped > 0
    finally:
        dec.close()
