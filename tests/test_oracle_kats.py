"""Known-answer tests from the reference's own unit suite, re-expressed on the
oracle restatement, the compiled reference, and (gpu) the CUDA path.

  search_test.cpp:31-65   table_model greedy traces
  search_test.cpp:77-97   tie rules: blank wins, then the smaller token id
  search_test.cpp:169-187 batched greedy == per-utterance greedy
  search_test.cpp:189-199 width-1 beam == greedy
plus the committed golden vectors in tests/golden/decode_golden.json
(tools/make_golden.py)."""
import json
import os

import numpy as np
import pytest

from tests import helpers as H


def _table_model():
    """search_test.cpp:31-47: V=3, saturated diagonal encoder, identity
    joiner, zero decoder side -> token k wins on the one-hot of k."""
    m = H.ref().model(3, 3, 3, 8, 3, 0, 0.0)
    import ctypes as C

    for name in list(m.w.p):
        r, c = C.c_int32(), C.c_int32()
        ptr = m.ref.lib.ref_model_param(m.h, name.encode(), C.byref(r), C.byref(c))
        arr = np.ctypeslib.as_array(ptr, (r.value, c.value))
        arr[:] = 0.0
        if name in ("enc_w1", "enc_w2"):
            np.fill_diagonal(arr, 5.0)
        if name in ("j_we", "out_w"):
            np.fill_diagonal(arr, 1.0)
        m.w.p[name] = arr.copy()
    return m


def _one_hot(toks, dim=3):
    f = np.zeros((len(toks), dim), np.float32)
    for t, k in enumerate(toks):
        f[t, k] = 1.0
    return f


TRACES = [([1, 0, 2], [1, 2]), ([0, 0, 0], []), ([2, 2, 1, 0], [2, 2, 1])]


def _table_inputs(m):
    feats = np.concatenate([_one_hot(x) for x, _ in TRACES])
    splits = np.array([0, 3, 6, 10], np.int32)
    enc = m.encoder(feats, splits)
    return feats, enc, splits


def test_table_model_greedy_traces():
    m = _table_model()
    feats, enc, splits = _table_inputs(m)
    want = [y for _, y in TRACES]
    assert m.greedy(feats, splits) == want
    assert H.orc().greedy(m.w, enc, splits) == want
    for beam in (1, 4):
        got, _ = H.orc().beam(m.w, enc, splits, beam=beam)
        assert got == m.beam(feats, splits, beam=beam)


def _tied_models():
    import ctypes as C

    def param(m, name):
        r, c = C.c_int32(), C.c_int32()
        ptr = m.ref.lib.ref_model_param(m.h, name.encode(), C.byref(r), C.byref(c))
        return np.ctypeslib.as_array(ptr, (r.value, c.value))

    # All logits exactly equal -> blank (search_test.cpp:80-87).
    m1 = H.ref().model(3, 3, 8, 8, 8, 50, 0.0)
    ow, ob = param(m1, "out_w"), param(m1, "out_b")
    ow[1:] = ow[0]
    ob[:] = 0.25
    m1.w.p["out_w"], m1.w.p["out_b"] = ow.copy(), ob.copy()
    # Tokens 1 and 2 tied above blank -> token 1 (88-96).
    m2 = H.ref().model(3, 3, 8, 8, 8, 51, 0.0)
    ow, ob = param(m2, "out_w"), param(m2, "out_b")
    ow[2] = ow[1]
    ob[0, 0], ob[0, 1], ob[0, 2] = -10.0, 0.0, 0.0
    m2.w.p["out_w"], m2.w.p["out_b"] = ow.copy(), ob.copy()
    return m1, m2


def test_greedy_tie_rules():
    m1, m2 = _tied_models()
    rng = np.random.default_rng(43)
    f1 = rng.standard_normal((5, 3)).astype(np.float32)
    f2 = rng.standard_normal((4, 3)).astype(np.float32)
    s1, s2 = np.array([0, 5], np.int32), np.array([0, 4], np.int32)
    assert m1.greedy(f1, s1) == [[]]
    assert H.orc().greedy(m1.w, m1.encoder(f1, s1), s1) == [[]]
    assert m2.greedy(f2, s2) == [[1, 1, 1, 1]]
    assert H.orc().greedy(m2.w, m2.encoder(f2, s2), s2) == [[1, 1, 1, 1]]


def test_batched_equals_solo_and_width1_equals_greedy():
    m = H.ref().model(4, 4, 8, 8, 8, 301, -0.5)
    Ts = list(range(3, 11))
    feats, enc, splits = H.frames(m, Ts, seed0=59)
    batch = H.orc().greedy(m.w, enc, splits)
    for i in range(len(Ts)):
        sl = slice(splits[i], splits[i + 1])
        assert H.orc().greedy(m.w, enc[sl], np.array([0, Ts[i]], np.int32))[0] == batch[i]
    w1, _ = H.orc().beam(m.w, enc, splits, beam=1)
    assert w1 == batch


GOLD = os.path.join(H.GOLDEN, "decode_golden.json")


def _golden_cases():
    return json.load(open(GOLD))["cases"]


def _golden_inputs(case):
    m = H.ref().model(*case["model"])
    feats, enc, splits = H.frames(m, case["T"], seed0=case["seed0"])
    return m, feats, enc, splits


def test_oracle_reproduces_golden():
    from oracle.py_oracle import Graph

    for case in _golden_cases():
        m, feats, enc, splits = _golden_inputs(case)
        if case["method"] == "greedy":
            assert H.orc().greedy(m.w, enc, splits) == case["tokens"]
        elif case["method"] == "beam":
            got, sc = H.orc().beam(m.w, enc, splits, **case["params"])
            assert got == case["tokens"]
            np.testing.assert_array_equal(sc, np.array(case["scores"]))
        else:
            g = H.ref().graph_trivial(case["model"][0])
            got, sc, _ = H.orc().fsa(m.w, enc, splits, g.g, *case["params"])
            assert got == case["tokens"]
            np.testing.assert_array_equal(sc, np.array(case["scores"]))


@pytest.mark.gpu
def test_gpu_table_model_and_ties():
    from paper_2211_00484_b200.api import BeamParams, Decoder

    m = _table_model()
    _, enc, splits = _table_inputs(m)
    dec = Decoder(H.api_weights(m.w))
    assert dec.greedy_search_batch(enc, splits) == [y for _, y in TRACES]
    for beam in (1, 4):
        got, _ = dec.beam_search_batch(enc, splits, BeamParams(beam_size=beam))
        assert got == H.orc().beam(m.w, enc, splits, beam=beam)[0]
    dec.close()
    m1, m2 = _tied_models()
    rng = np.random.default_rng(43)
    for mm, T, want in [(m1, 5, [[]]), (m2, 4, [[1, 1, 1, 1]])]:
        f = rng.standard_normal((T, 3)).astype(np.float32)
        s = np.array([0, T], np.int32)
        d = Decoder(H.api_weights(mm.w))
        assert d.greedy_search_batch(mm.encoder(f, s), s) == want
        d.close()


@pytest.mark.gpu
def test_gpu_reproduces_golden():
    from paper_2211_00484_b200.api import BeamParams, Decoder, FsaParams, Graph

    for case in _golden_cases():
        m, feats, enc, splits = _golden_inputs(case)
        dec = Decoder(H.api_weights(m.w))
        if case["method"] == "greedy":
            assert dec.greedy_search_batch(enc, splits) == case["tokens"]
        elif case["method"] == "beam":
            p = case["params"]
            got, sc = dec.beam_search_batch(
                enc, splits, BeamParams(p["beam"], 1, p["merge_op"], bool(p["length_norm"]), p["max_total"])
            )
            assert got == case["tokens"]
            np.testing.assert_allclose(sc, case["scores"], rtol=1e-9)
        else:
            got, sc = dec.fsa_beam_search(enc, splits, Graph.trivial(dec), FsaParams(*case["params"]))
            assert got == case["tokens"]
            np.testing.assert_allclose(sc, case["scores"], rtol=1e-9)
        dec.close()
