"""The time-sliced host-frame beam path (capi.cu run_sliced): frames copied
per time slice, K1 over row groups, the beam kernel resumed slice after slice
from hypothesis sets kept in HBM.  Tokens identical to the oracle, scores
bit-identical to the single-launch device-frame path (the slicing changes
launch boundaries only, never the arithmetic)."""
import numpy as np
import pytest

from tests import helpers as H

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize(
    "T,B,first,cap",
    [(77, 300, "3", "7"), (200, 1024, "16", "256"), (33, 9, "1", "1"), (17, 5, "16", "256"), (100, 1, "4", "32")],
)
def test_sliced_host_frames_match_oracle_and_device_path(T, B, first, cap):
    import torch

    from paper_2211_00484_b200.api import BeamParams

    m = H.model(V=500, seed=1, blank_bias=0.4)
    _, enc, splits = H.frames(m, [T] * B, seed0=52000 + T)
    sliced = H.decoder_env(m, RNNTG_SLICED="1", RNNTG_SLICE_FIRST=first, RNNTG_SLICE_MAX=cap)
    plain = H.decoder_env(m, RNNTG_SLICED="0")
    try:
        got, sc = sliced.beam_search_batch(enc, splits, BeamParams(beam_size=4))
        assert sliced.stats()["stream_frames"] == B * T
        if B <= 300:
            want, want_sc = H.orc().beam(m.w, enc, splits, beam=4)
            assert got == want
            H.assert_scores_equal(sc, want_sc)
        d_enc = torch.from_numpy(enc).cuda()
        tok = torch.zeros(max(1, int(splits[-1])), dtype=torch.int32, device="cuda")
        dsc = torch.zeros(B, dtype=torch.float64, device="cuda")
        osp, tok, dsc = plain.beam_search_batch(d_enc, splits, BeamParams(beam_size=4), tok, dsc)
        t = tok.cpu().numpy()
        assert [t[osp[i] : osp[i + 1]].tolist() for i in range(B)] == got
        assert np.array_equal(dsc.cpu().numpy(), sc)
    finally:
        sliced.close()
        plain.close()


def test_sliced_repeated_calls_and_beam_sizes():
    """Back-to-back calls on one handle reuse the slice events, the hypothesis
    state and the frame buffer; every beam capacity (1, 2, 4, 8) resumes."""
    from paper_2211_00484_b200.api import BeamParams

    m = H.model(V=500, seed=2, blank_bias=0.4)
    dec = H.decoder_env(m, RNNTG_SLICED="1", RNNTG_SLICE_FIRST="5", RNNTG_SLICE_MAX="11")
    try:
        for beam, T, B in [(1, 40, 20), (2, 60, 33), (8, 45, 17), (4, 40, 20)]:
            _, enc, splits = H.frames(m, [T] * B, seed0=53000 + beam)
            want, want_sc = H.orc().beam(m.w, enc, splits, beam=beam)
            got, sc = dec.beam_search_batch(enc, splits, BeamParams(beam_size=beam))
            assert got == want, beam
            H.assert_scores_equal(sc, want_sc)
    finally:
        dec.close()


def test_sliced_device_frames_opt_in():
    """RNNTG_SLICED=2 also slices device-resident frames (K1 per slice on the
    side stream): the same tokens and bit-identical scores as K1 + decode."""
    import torch

    from paper_2211_00484_b200.api import BeamParams

    m = H.model(V=500, seed=3, blank_bias=0.4)
    T, B = 90, 160
    _, enc, splits = H.frames(m, [T] * B, seed0=54000)
    d_enc = torch.from_numpy(enc).cuda()
    outs = []
    for env in ({"RNNTG_SLICED": "2", "RNNTG_SLICE_FIRST": "4", "RNNTG_SLICE_MAX": "16"}, {"RNNTG_SLICED": "0"}):
        dec = H.decoder_env(m, **env)
        try:
            tok = torch.zeros(B * T, dtype=torch.int32, device="cuda")
            dsc = torch.zeros(B, dtype=torch.float64, device="cuda")
            osp, tok, dsc = dec.beam_search_batch(d_enc, splits, BeamParams(beam_size=4), tok, dsc)
            t = tok.cpu().numpy()
            outs.append(([t[osp[i] : osp[i + 1]].tolist() for i in range(B)], dsc.cpu().numpy()))
        finally:
            dec.close()
    assert outs[0][0] == outs[1][0]
    assert np.array_equal(outs[0][1], outs[1][1])
    want, _ = H.orc().beam(m.w, enc[: 20 * T], splits[:21], beam=4)
    assert outs[0][0][:20] == want


def test_sliced_bench_scale_matches_single_launch_and_oracle_sample():
    """The bench shape (1024 streams x 1000 frames, default slices 8 ... 496):
    sliced host path == K1 + one decode launch on device frames (tokens and
    scores bit-identical), and the first 8 streams == the reference."""
    import torch

    from paper_2211_00484_b200.api import BeamParams

    m = H.model(V=500, seed=1, blank_bias=0.4)
    B, T, U = 1024, 1000, 8
    rng = np.random.default_rng(7)
    enc_u = np.tanh(rng.standard_normal((U, T, 512)).astype(np.float32) * 0.7)
    enc = np.ascontiguousarray(np.concatenate([enc_u] * (B // U)).reshape(B * T, 512))
    splits = (np.arange(B + 1) * T).astype(np.int32)
    sliced = H.decoder_env(m, RNNTG_SLICED="1")
    plain = H.decoder_env(m, RNNTG_SLICED="0")
    try:
        osp, tok, sc = sliced.beam_search_batch(torch.from_numpy(enc).pin_memory(), splits,
                                                BeamParams(beam_size=4), as_lists=False)
        d_enc = torch.from_numpy(enc).cuda()
        dtok = torch.zeros(B * T, dtype=torch.int32, device="cuda")
        dsc = torch.zeros(B, dtype=torch.float64, device="cuda")
        osp2, dtok, dsc = plain.beam_search_batch(d_enc, splits, BeamParams(beam_size=4), dtok, dsc)
        assert np.array_equal(osp, osp2)
        assert np.array_equal(tok, dtok.cpu().numpy()[: osp2[-1]])
        assert np.array_equal(sc, dsc.cpu().numpy())
        want, want_sc = H.orc().beam(m.w, enc[: U * T], splits[: U + 1], beam=4)
        assert [tok[osp[i] : osp[i + 1]].tolist() for i in range(U)] == want
        H.assert_scores_equal(sc[:U], want_sc)
    finally:
        sliced.close()
        plain.close()
