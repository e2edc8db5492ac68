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


def test_host_features_time_sliced_matches_device_frames(monkeypatch):
    """Host features of a uniform batch (RNNTG_MEM_HOST_FEATURES, the C++
    drop-in's call): the encoder runs per time slice inside the sliced
    pipeline (copy, encoder, K1, decode overlapped).  Tokens identical and
    scores bit-equal to the unsliced device-frame path, and tokens equal to
    the reference's beam search on the same features."""
    import ctypes as C

    from paper_2211_00484_b200.api import BeamParams, Decoder, _BeamParams

    monkeypatch.setenv("RNNTG_BEAM_CLUSTER", "0")  # small B: else the cluster kernel takes the batch
    m = H.model(V=500, seed=2, blank_bias=0.4)
    dec = Decoder(H.api_weights(m.w))
    dec.set_encoder(m.w.p)
    B, T = 5, 70  # > the first 8-frame slice: slices 8, 16, 32, 14
    feats, enc, splits = H.frames(m, [T] * B, seed0=77)
    want, wsc = dec.beam_search_batch(enc, splits, BeamParams(beam_size=4))
    feats = np.ascontiguousarray(feats, np.float32)
    fs = np.ascontiguousarray(splits, np.int32)
    osp = np.zeros(B + 1, np.int32)
    tok = np.zeros(B * T, np.int32)
    sc = np.zeros(B, np.float64)
    bp = _BeamParams(4, 1, 0, 0, 0)
    i32p, f32p, f64p = C.POINTER(C.c_int32), C.POINTER(C.c_float), C.POINTER(C.c_double)
    rc = dec._lib.rnntg_beam_search_batch(dec.h, feats.ctypes.data_as(f32p), fs.ctypes.data_as(i32p), B, C.byref(bp),
                                          2, osp.ctypes.data_as(i32p), C.c_void_p(tok.ctypes.data),
                                          sc.ctypes.data_as(f64p))
    assert rc == 0
    got = [tok[osp[i] : osp[i + 1]].tolist() for i in range(B)]
    assert got == want
    assert np.array_equal(sc.view(np.uint64), np.asarray(wsc, np.float64).view(np.uint64))
    assert got == m.beam(feats, splits, beam=4)
    assert dec.stats()["kernel_launches"] >= 4 * 4  # 4 slices x (2 encoder layers + K1 + decode)
    dec.close()
