"""The fused encoder-projection path of the beam kernel (pe computed inside
the decode kernel; host frames streamed in per time slice by the copy engine
with stream-ordered counter writes) against the oracle and against the
separate K1 + decode path: tokens identical, scores bit-identical (pe is the
same sequential fp32 sum either way)."""
import os

import numpy as np
import pytest

from tests import helpers as H

pytestmark = pytest.mark.gpu


def _decoder(m, fused):
    # RNNTG_SLICED=0: host frames take the fused path, not the time-sliced one
    return H.decoder_env(m, RNNTG_FUSED_PE=str(fused), RNNTG_SLICED="0")


@pytest.mark.parametrize("T,B", [(77, 300), (32, 9), (1, 5), (100, 1)])
def test_fused_host_streaming_matches_oracle_and_k1_path(T, B):
    import torch

    from paper_2211_00484_b200.api import BeamParams

    m = H.model(V=500, seed=1, blank_bias=0.4)
    _, enc, splits = H.frames(m, [T] * B, seed0=31000 + T)
    want, want_sc = H.orc().beam(m.w, enc, splits, beam=4)
    fused, plain, forced = _decoder(m, 1), _decoder(m, 0), _decoder(m, 2)
    try:
        got, sc = fused.beam_search_batch(enc, splits, BeamParams(beam_size=4))  # host frames: streamed
        assert got == want
        np.testing.assert_allclose(sc, want_sc, rtol=1e-9, atol=0)
        got0, sc0 = plain.beam_search_batch(enc, splits, BeamParams(beam_size=4))  # chunked K1 + decode
        assert got0 == got and np.array_equal(sc0, sc)
        d_enc = torch.from_numpy(enc).cuda()
        tok = torch.zeros(max(1, int(splits[-1])), dtype=torch.int32, device="cuda")
        dsc = torch.zeros(B, dtype=torch.float64, device="cuda")
        osp, tok, dsc = forced.beam_search_batch(d_enc, splits, BeamParams(beam_size=4), tok, dsc)
        t = tok.cpu().numpy()
        assert [t[osp[i] : osp[i + 1]].tolist() for i in range(B)] == want
        assert np.array_equal(dsc.cpu().numpy(), sc)
    finally:
        fused.close()
        plain.close()
        forced.close()
