"""Small-batch greedy on thread-block clusters (cluster.cu: out_w column
slices resident in 8 CTAs' shared memory, h slices and slice maxima
exchanged by st.async on mbarriers, next-frame h rows built ahead and
rebuilt after an emission) against the compiled reference and against the
persistent single-CTA kernel, across the batch sizes where the cluster
kernel is chosen (<= 144 streams) and just beyond it, at a low and a high
emission rate (the rebuild path on most frames)."""
import os

import numpy as np
import pytest

from tests import helpers as H

pytestmark = pytest.mark.gpu


def _decoder(m, on):
    from paper_2211_00484_b200.api import Decoder

    old = os.environ.get("RNNTG_GREEDY_CLUSTER")
    os.environ["RNNTG_GREEDY_CLUSTER"] = "1" if on else "0"
    try:
        return Decoder(H.api_weights(m.w))
    finally:
        if old is None:
            del os.environ["RNNTG_GREEDY_CLUSTER"]
        else:
            os.environ["RNNTG_GREEDY_CLUSTER"] = old


@pytest.mark.parametrize("B,bias", [(1, 0.2), (7, 0.2), (8, 0.2), (19, 0.2), (144, 0.2), (150, 0.2), (8, -3.0),
                                    (40, -3.0)])
def test_greedy_cluster_matches_reference_and_plain_kernel(B, bias):
    m = H.model(V=500, seed=3, blank_bias=bias)
    Ts = [int(x) for x in np.random.default_rng(B).integers(0, 30, B)]
    feats, enc, splits = H.frames(m, Ts, seed0=7000 + B)
    want = m.greedy(feats, splits)
    on, off = _decoder(m, True), _decoder(m, False)
    try:
        assert on.greedy_search_batch(enc, splits) == want
        assert off.greedy_search_batch(enc, splits) == want
    finally:
        on.close()
        off.close()
