"""Token-exact parity on every BASELINE.json config at its stated shape,
against the compiled reference (oracle/_ref) run on the same inputs on this
host's cores (SURVEY.md §8(d) inputs: init_model weights (ModelConfig's default seed 0), DetRng features
through the reference encoder).

  config 1  greedy_search_batch S=1, B=8, T=200              (search.hpp:107-167)
  config 2  beam_search beam 4, B=256, T=500                 (search.hpp:206-277)
  config 3  fsa_beam_search trivial graph (4, 8, 4), B=512, T=500
  config 4  fsa_beam_search 1,003,931-arc trigram graph (8, 64, 8), B=256, T=500
            (blank bias -1.4; ~0.06 tokens/frame measured at seed 0)
  config 5  beam 4, B=1024, T=1000, frames from librnntg's own input path
            (host DetRng generator + GPU encoder, exactly bench.py's), a
            stratified 64-stream sample compared against the reference

Bars: tokens identical on every stream; beam scores bit-equal to the oracle
restatement's (the reference's beam_search returns tokens only); FSA
best-path scores bit-equal to the reference's and every stream's lattice
text (serialize_fsa_text) byte-identical.  Exact-score ties resolved by
the tie rules are counted by the device and reported.
"""
import os

import numpy as np
import pytest

from tests import helpers as H

pytestmark = pytest.mark.gpu

THREADS = os.cpu_count() or 1


def _assert_tokens(got, want, what):
    bad = [i for i, (a, b) in enumerate(zip(got, want)) if a != b]
    assert len(got) == len(want)
    assert not bad, f"{what}: {len(bad)} streams differ, first {bad[:8]}"


def _assert_texts(got, want, what):
    """serialize_fsa_text of every stream's lattice, byte for byte."""
    bad = [i for i, (a, b) in enumerate(zip(got, want)) if a != b]
    assert len(got) == len(want)
    assert not bad, f"{what}: {len(bad)} lattice texts differ, first {bad[:8]}"


def test_config2_beam_256x500():
    from paper_2211_00484_b200.api import BeamParams, Decoder

    m = H.model(V=500, seed=0, blank_bias=0.4)
    feats, enc, splits = H.frames(m, [500] * 256, seed0=20000)
    dec = Decoder(H.api_weights(m.w))
    try:
        got, sc = dec.beam_search_batch(enc, splits, BeamParams(beam_size=4))
        ties = dec.stats()["tie_breaks"]
    finally:
        dec.close()
    want = m.beam(feats, splits, beam=4, threads=THREADS)
    _assert_tokens(got, want, "config 2")
    _, osc = H.orc().beam(m.w, enc, splits, beam=4, threads=THREADS)
    H.assert_scores_equal(sc, osc)
    tpf = sum(map(len, want)) / splits[-1]
    assert 0.15 < tpf < 0.35, tpf  # the reference's emission rate (seed 0, blank bias 0.4)
    print(f"config 2: 256 streams identical, tokens/frame {tpf:.3f}, exact-score ties resolved {ties}")


def test_config3_fsa_trivial_512x500():
    from paper_2211_00484_b200.api import Decoder, FsaParams, Graph

    m = H.model(V=500, seed=0, blank_bias=0.4)
    feats, enc, splits = H.frames(m, [500] * 512, seed0=30000)
    rg = H.ref().graph_trivial(500)
    dec = Decoder(H.api_weights(m.w))
    try:
        got, sc = dec.fsa_beam_search(enc, splits, Graph.trivial(dec), FsaParams(4.0, 8, 4))
        texts = [dec.fsa_lattice_text(i) for i in range(512)]
    finally:
        dec.close()
    want, wsc, wtexts = m.fsa(feats, splits, rg, 4.0, 8, 4, threads=THREADS, lattice_texts=True)
    _assert_tokens(got, want, "config 3")
    H.assert_scores_equal(sc, wsc)
    _assert_texts(texts, wtexts, "config 3")


@pytest.mark.parametrize("cfg", [3, 4])
def test_config34_logadd_best_sequences(cfg):
    """lattice_to_best_seq(kLogAdd, nbest 100, seeds 0 and 7) of config 3 / 4
    at full shape on the GPU, every stream compared against the reference's
    own function on its own lattices: identical sequences, bit-equal
    sequence totals."""
    from oracle.py_oracle import synthetic_arpa
    from paper_2211_00484_b200.api import Decoder, FsaParams, Graph

    if cfg == 3:
        B, bias, seed0, params, step = 512, 0.4, 30000, (4.0, 8, 4), 1
    else:
        B, bias, seed0, params, step = 256, -1.4, 40000, (8.0, 64, 8), 1
    m = H.model(V=500, seed=0, blank_bias=bias)
    feats, enc, splits = H.frames(m, [500] * B, seed0=seed0)
    rg = H.ref().graph_trivial(500) if cfg == 3 else H.ref().graph_from_arpa(synthetic_arpa(500), 500)
    dec = Decoder(H.api_weights(m.w))
    try:
        g = Graph.trivial(dec) if cfg == 3 else Graph(dec, rg.g.num_states, rg.g.arc_splits, rg.g.dst, rg.g.label,
                                                      rg.g.weight)
        dec.fsa_beam_search(enc, splits, g, FsaParams(*params))
        got = {seed: dec.fsa_lattice_best(nbest=100, seed=seed) for seed in (0, 7)}
    finally:
        dec.close()
    pick = np.arange(0, B, step)
    T = 500
    f_pick = np.concatenate([feats[i * T : (i + 1) * T] for i in pick])
    s_pick = (np.arange(len(pick) + 1) * T).astype(np.int32)
    for seed in (0, 7):
        want, wlp = m.fsa_logadd(f_pick, s_pick, rg, *params, nbest=100, seed=seed, threads=THREADS)
        toks, lp = got[seed]
        _assert_tokens([toks[i] for i in pick], want, f"config {cfg} log-add seed {seed}")
        H.assert_scores_equal(lp[pick], wlp)


def test_config4_fsa_ngram_256x500():
    from oracle.py_oracle import synthetic_arpa
    from paper_2211_00484_b200.api import Decoder, FsaParams, Graph

    m = H.model(V=500, seed=0, blank_bias=-1.4)
    feats, enc, splits = H.frames(m, [500] * 256, seed0=40000)
    rg = H.ref().graph_from_arpa(synthetic_arpa(500), 500)
    g = rg.g
    assert g.num_arcs > 1_000_000
    dec = Decoder(H.api_weights(m.w))
    try:
        dg = Graph(dec, g.num_states, g.arc_splits, g.dst, g.label, g.weight)
        got, sc = dec.fsa_beam_search(enc, splits, dg, FsaParams(8.0, 64, 8))
        texts = [dec.fsa_lattice_text(i) for i in range(256)]
    finally:
        dec.close()
    want, wsc, wtexts = m.fsa(feats, splits, rg, 8.0, 64, 8, threads=THREADS, lattice_texts=True)
    _assert_tokens(got, want, "config 4")
    H.assert_scores_equal(sc, wsc)
    _assert_texts(texts, wtexts, "config 4")
    tpf = sum(map(len, want)) / splits[-1]
    assert tpf > 0.03, tpf


def test_config5_beam_1024x1000_bench_inputs_sample():
    """The bench workload itself: librnntg's input generators + GPU encoder,
    all 1024 streams decoded in one call on device-resident frames; every
    16th stream (64 streams) is decoded by the reference from the same
    DetRng features through its own encoder."""
    import torch

    from paper_2211_00484_b200.api import BeamParams, Decoder, ModelWeights, gaussian_features, init_model_weights

    B, T = 1024, 1000
    w = init_model_weights(500, 80, 512, 512, 512, seed=0, blank_bias=0.4)
    dec = Decoder(ModelWeights.from_dict(w))
    try:
        dec.set_encoder(w)
        feats = gaussian_features(7000, B, T, 80)
        splits = (np.arange(B + 1) * T).astype(np.int32)
        d_feats = torch.from_numpy(feats).cuda()
        d_enc = torch.empty((B * T, 512), dtype=torch.float32, device="cuda")
        dec.encoder_forward(d_feats, splits, d_enc)
        tok = torch.zeros(B * T, dtype=torch.int32, device="cuda")
        sc = torch.zeros(B, dtype=torch.float64, device="cuda")
        osp, tok, sc = dec.beam_search_batch(d_enc, splits, BeamParams(beam_size=4), tok, sc)
        torch.cuda.synchronize()
        t, s = tok.cpu().numpy(), sc.cpu().numpy()
        pick = np.arange(0, B, 16)
        got = [t[osp[i] : osp[i + 1]].tolist() for i in pick]
        got_sc = s[pick]
        enc_pick = np.concatenate([d_enc[i * T : (i + 1) * T].cpu().numpy() for i in pick])
    finally:
        dec.close()
    m = H.model(V=500, seed=0, blank_bias=0.4)
    assert np.array_equal(m.w.p["out_w"].view(np.uint32), w["out_w"].view(np.uint32))
    f_pick = np.concatenate([feats[i * T : (i + 1) * T] for i in pick])
    s_pick = (np.arange(len(pick) + 1) * T).astype(np.int32)
    # the GPU encoder's frames are the reference encoder's, bit for bit
    ref_enc = m.encoder(f_pick, s_pick, threads=THREADS)
    assert np.array_equal(ref_enc.view(np.uint32), enc_pick.view(np.uint32))
    want = m.beam(f_pick, s_pick, beam=4, threads=THREADS)
    _assert_tokens(got, want, "config 5 sample")
    _, osc = H.orc().beam(m.w, ref_enc, s_pick, beam=4, threads=THREADS)
    H.assert_scores_equal(got_sc, osc)
    tpf = sum(map(len, want)) / s_pick[-1]
    assert 0.15 < tpf < 0.35, tpf
