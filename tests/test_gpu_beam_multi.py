"""Modified beam search with S > 1 symbols per frame (beam_search,
search.hpp:206-277, any max_symbols) on the GPU against the compiled
reference's beam_search on identical inputs: tokens identical for max and
log-add merging, widths 1-8, length normalisation and the symbol cap."""
import numpy as np
import pytest

from tests import helpers as H

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dm():
    from paper_2211_00484_b200.api import Decoder

    m = H.model(V=500, seed=8, blank_bias=0.0)  # ~1 emission per frame: S matters
    dec = Decoder(H.api_weights(m.w))
    yield m, dec
    dec.close()


@pytest.mark.parametrize("S,beam,merge", [(2, 4, 0), (3, 4, 1), (2, 1, 0), (4, 8, 0), (2, 2, 1)])
def test_beam_multi_symbol_matches_reference(dm, S, beam, merge):
    from paper_2211_00484_b200.api import BeamParams

    m, dec = dm
    Ts = [int(x) for x in np.random.default_rng(S * 10 + beam).integers(0, 30, 19)]
    feats, enc, splits = H.frames(m, Ts, seed0=6000 + 7 * S + beam)
    want = m.beam(feats, splits, beam=beam, merge_op=merge, max_symbols=S)
    got, sc = dec.beam_search_batch(enc, splits, BeamParams(beam_size=beam, max_symbols=S, merge_op=merge))
    assert got == want
    assert np.all(np.isfinite(sc))


def test_beam_multi_length_norm_cap_and_unlimited(dm):
    from paper_2211_00484_b200.api import NO_SYMBOL_LIMIT, BeamParams

    m, dec = dm
    Ts = [25] * 9
    feats, enc, splits = H.frames(m, Ts, seed0=6500)
    for S, ln, cap in [(3, 1, 0), (2, 0, 5), (NO_SYMBOL_LIMIT, 0, 0)]:
        want = m.beam(feats, splits, beam=4, length_norm=ln, max_total=cap, max_symbols=S)
        got, _ = dec.beam_search_batch(
            enc, splits, BeamParams(beam_size=4, max_symbols=S, length_norm=bool(ln), max_total_symbols=cap)
        )
        assert got == want, (S, ln, cap)


def test_beam_multi_s1_path_unchanged(dm):
    """S = 1 keeps the specialised kernel: same results as before."""
    from paper_2211_00484_b200.api import BeamParams

    m, dec = dm
    Ts = [20] * 5
    feats, enc, splits = H.frames(m, Ts, seed0=6600)
    assert dec.beam_search_batch(enc, splits, BeamParams(beam_size=4, max_symbols=1))[0] == m.beam(
        feats, splits, beam=4, max_symbols=1
    )
