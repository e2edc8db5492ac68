"""Small-batch modified beam search on thread-block clusters
(decode.cu beam_cluster_kernel: out_w column slices resident in 8 CTAs'
shared memory, rows reduced where their slices land, beam steps on CTA 0)
against the persistent kernel (RNNTG_BEAM_CLUSTER=0) and the oracle:
identical tokens, bit-equal scores, for ragged batches, every beam width,
both merge ops, length normalisation and the symbol cap, and at the
batch sizes where the cluster kernel takes over (up to 15 resident clusters
x min(14, 64 / beam) streams)."""
import numpy as np
import pytest

from tests import helpers as H

pytestmark = pytest.mark.gpu


def _both(m, enc, splits, params):
    from paper_2211_00484_b200.api import Decoder

    dc = Decoder(H.api_weights(m.w))
    dp = H.decoder_env(m, RNNTG_BEAM_CLUSTER="0")
    try:
        a = dc.beam_search_batch(enc, splits, params)
        b = dp.beam_search_batch(enc, splits, params)
    finally:
        dc.close()
        dp.close()
    return a, b


@pytest.mark.parametrize("beam,merge,lnorm,cap", [(4, 0, 0, 0), (1, 0, 0, 0), (2, 1, 0, 0), (8, 0, 1, 0),
                                                  (4, 1, 1, 7), (3, 0, 0, 0)])
def test_cluster_matches_persistent_and_oracle(beam, merge, lnorm, cap):
    from paper_2211_00484_b200.api import BeamParams

    m = H.model(V=500, seed=3, blank_bias=0.3)
    Ts = [37, 0, 12, 37, 5, 30, 1, 22]
    _, enc, splits = H.frames(m, Ts, seed0=611)
    params = BeamParams(beam_size=beam, merge_op=merge, length_norm=bool(lnorm), max_total_symbols=cap)
    (got, gsc), (want, wsc) = _both(m, enc, splits, params)
    assert got == want
    H.assert_scores_equal(gsc, wsc)
    ot, osc = H.orc().beam(m.w, enc, splits, beam=beam, merge_op=merge, length_norm=lnorm, max_total=cap)
    assert got == ot
    H.assert_scores_equal(gsc, osc)


@pytest.mark.parametrize("B,beam", [(15, 4), (150, 4), (180, 4), (210, 4), (120, 8)])
def test_cluster_batch_sizes(B, beam):
    """One stream per cluster; 10; 12; 14 per cluster (up to 56 joiner rows
    a frame: two h / GEMM passes); beam 8 at 8 per cluster (up to 64 rows:
    two full passes)."""
    from paper_2211_00484_b200.api import BeamParams

    m = H.model(V=500, seed=4, blank_bias=0.2)
    rng = np.random.default_rng(B)
    Ts = rng.integers(1, 24, B).tolist()
    _, enc, splits = H.frames(m, Ts, seed0=7000 + B)
    (got, gsc), (want, wsc) = _both(m, enc, splits, BeamParams(beam_size=beam))
    assert got == want
    H.assert_scores_equal(gsc, wsc)
