"""The reference toy encoder on the GPU, bit-exact
against rnnt::encoder_forward (model.hpp:224-238), then the feature-to-tokens
path end to end against the reference's own searches on features."""
import numpy as np
import pytest

from tests import helpers as H

pytestmark = pytest.mark.gpu


def test_encoder_bit_exact_and_feature_path():
    import torch

    from paper_2211_00484_b200.api import BeamParams, Decoder

    m = H.model(V=500, seed=1, blank_bias=0.4)
    dec = Decoder(H.api_weights(m.w))
    dec.set_encoder(m.w.p)
    Ts = [0, 37, 5, 120]
    feats, enc, splits = H.frames(m, Ts, seed0=55)
    got = dec.encoder_forward(feats, splits)
    assert np.array_equal(got.view(np.uint32), enc.view(np.uint32))
    d_feats = torch.from_numpy(feats).cuda()
    d_enc = torch.zeros(enc.shape, dtype=torch.float32, device="cuda")
    dec.encoder_forward(d_feats, splits, d_enc)
    assert np.array_equal(d_enc.cpu().numpy().view(np.uint32), enc.view(np.uint32))
    host, _ = dec.beam_search_batch(got, splits, BeamParams(beam_size=4))
    assert host == m.beam(feats, splits, beam=4)
    dec.close()
