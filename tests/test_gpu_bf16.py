"""The bf16 tcgen05 joiner variant (reported separately; not token-exact).

It must run, agree with the exact path on most tokens (the north star asks
for its token-agreement rate), and leave the exact path untouched when
switched back."""
import numpy as np
import pytest

from tests import helpers as H

pytestmark = pytest.mark.gpu


def edit_distance(a, b):
    d = list(range(len(b) + 1))
    for i, x in enumerate(a, 1):
        prev, d[0] = d[0], i
        for j, y in enumerate(b, 1):
            cur = min(d[j] + 1, d[j - 1] + 1, prev + (x != y))
            prev, d[j] = d[j], cur
    return d[-1]


def agreement(ref, hyp):
    """1 - (token edit distance / reference tokens), pooled over streams."""
    errs = sum(edit_distance(r, h) for r, h in zip(ref, hyp))
    n = max(1, sum(len(r) for r in ref))
    return 1.0 - errs / n


def test_bf16_beam_runs_and_agrees():
    from paper_2211_00484_b200.api import BeamParams, Decoder

    m = H.model(V=500, seed=1, blank_bias=0.4)
    dec = Decoder(H.api_weights(m.w))
    Ts = [int(x) for x in np.random.default_rng(2).integers(20, 80, 300)]
    _, enc, splits = H.frames(m, Ts, seed0=123)
    exact, esc = dec.beam_search_batch(enc, splits, BeamParams(beam_size=4))
    dec.set_joiner_mode("bf16")
    fast, fsc = dec.beam_search_batch(enc, splits, BeamParams(beam_size=4))
    agree = agreement(exact, fast)
    print("bf16 token agreement", agree, "streams identical", np.mean([a == b for a, b in zip(exact, fast)]))
    assert agree > 0.5
    assert np.all(np.isfinite(fsc))
    np.testing.assert_allclose(fsc, esc, rtol=0.05)
    dec.set_joiner_mode("exact")
    again, asc = dec.beam_search_batch(enc, splits, BeamParams(beam_size=4))
    assert again == exact and np.array_equal(asc, esc)
    dec.close()
