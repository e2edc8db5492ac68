"""ctypes access to the CPU oracle and to the compiled reference.

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference leg.  The product package
(paper_2211_00484_b200) never imports this module.

* ``Oracle``     -> oracle/librnnt_oracle.so, the restatement (rnnt_oracle.cpp)
* ``Reference``  -> oracle/_ref/librnnt_ref.so, the unmodified reference
                    headers behind ref_capi.cpp
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "librnnt_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "librnnt_ref.so")

PARAM_NAMES = ("emb", "ctx_w", "ctx_b", "j_we", "j_wd", "j_b", "out_w", "out_b")
ENC_NAMES = ("enc_w1", "enc_b1", "enc_w2", "enc_b2")

_i32p = C.POINTER(C.c_int32)
_f32p = C.POINTER(C.c_float)
_f64p = C.POINTER(C.c_double)


def _p(a, t):
    return a.ctypes.data_as(t)


def build():
    """Build the oracle (and the reference wrapper when /root/reference exists)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


# --------------------------------------------------------------------------
# Model weights (reference init_model, model.hpp:129-169) as numpy arrays.
# --------------------------------------------------------------------------


@dataclass
class Weights:
    V: int
    F: int
    D: int
    E: int
    J: int
    p: dict  # name -> float32 ndarray (rows, cols)

    def desc_arrays(self):
        return [np.ascontiguousarray(self.p[n], dtype=np.float32) for n in PARAM_NAMES]


class _OrcModel(C.Structure):
    _fields_ = [("V", C.c_int32), ("D", C.c_int32), ("E", C.c_int32), ("J", C.c_int32)] + [
        (n, _f32p) for n in PARAM_NAMES
    ]


class _OrcGraph(C.Structure):
    _fields_ = [
        ("num_states", C.c_int32),
        ("num_arcs", C.c_int32),
        ("arc_splits", _i32p),
        ("dst", _i32p),
        ("label", _i32p),
        ("weight", _f64p),
    ]


class _OrcLattice(C.Structure):
    _fields_ = [
        ("num_nodes", C.c_int32),
        ("num_arcs", C.c_int32),
        ("src", _i32p),
        ("dst", _i32p),
        ("label", _i32p),
        ("score", _f64p),
    ]


@dataclass
class Graph:
    """CSR decoding graph (fsa.hpp:54-80)."""

    num_states: int
    arc_splits: np.ndarray  # int32 [S+1]
    dst: np.ndarray  # int32 [A]
    label: np.ndarray  # int32 [A]
    weight: np.ndarray  # float64 [A]
    finals: dict

    @property
    def num_arcs(self):
        return int(self.dst.shape[0])


def ragged(lists):
    splits = np.zeros(len(lists) + 1, dtype=np.int32)
    for i, x in enumerate(lists):
        splits[i + 1] = splits[i] + len(x)
    return splits


def unragged(splits, flat):
    return [list(map(int, flat[splits[i] : splits[i + 1]])) for i in range(len(splits) - 1)]


class Oracle:
    """The C restatement (rnnt_oracle.cpp)."""

    def __init__(self, path=ORACLE_SO):
        if not os.path.exists(path):
            build()
        self.lib = C.CDLL(path)
        L = self.lib
        L.orc_affine.argtypes = [_f32p, _f32p, _f32p, C.c_int32, C.c_int32, C.c_int32, _f32p]
        L.orc_tanhf.argtypes = [C.c_float]
        L.orc_tanhf.restype = C.c_float
        L.orc_encoder.argtypes = [_f32p] * 4 + [C.c_int32, C.c_int32, _f32p, C.c_int32, _f32p]
        L.orc_decoder_project.argtypes = [C.POINTER(_OrcModel), _i32p, C.c_int32, _f32p]
        L.orc_joiner_logits_from_proj.argtypes = [C.POINTER(_OrcModel), _f32p, _f32p, _f32p]
        L.orc_log_softmax.argtypes = [_f32p, C.c_int32, _f64p]
        L.orc_greedy_batch.argtypes = [C.POINTER(_OrcModel), _f32p, _i32p, C.c_int32, C.c_int, _i32p, _i32p]
        L.orc_beam_search.argtypes = [C.POINTER(_OrcModel), _f32p, _i32p, C.c_int32] + [C.c_int32] * 4 + [
            C.c_int,
            _i32p,
            _i32p,
            _f64p,
        ]
        L.orc_fsa_beam_search.argtypes = [
            C.POINTER(_OrcModel),
            _f32p,
            _i32p,
            C.c_int32,
            C.POINTER(_OrcGraph),
            C.c_double,
            C.c_int32,
            C.c_int32,
            C.c_int,
            _i32p,
            _i32p,
            _f64p,
            C.POINTER(_OrcLattice),
        ]
        L.orc_lattice_free.argtypes = [C.POINTER(_OrcLattice)]
        L.orc_last_error.restype = C.c_char_p

    def _model(self, w: Weights):
        arrs = w.desc_arrays()
        m = _OrcModel(w.V, w.D, w.E, w.J, *[_p(a, _f32p) for a in arrs])
        return m, arrs

    def _check(self, rc):
        if rc != 0:
            raise RuntimeError(f"oracle error {rc}: {self.lib.orc_last_error().decode()}")

    def affine(self, w, bias, x):
        w = np.ascontiguousarray(w, np.float32)
        x = np.ascontiguousarray(x, np.float32)
        M, K = x.shape
        N = w.shape[0]
        y = np.empty((M, N), np.float32)
        b = None if bias is None else np.ascontiguousarray(bias, np.float32)
        self.lib.orc_affine(_p(w, _f32p), None if b is None else _p(b, _f32p), _p(x, _f32p), M, N, K, _p(y, _f32p))
        return y

    def encoder(self, w: Weights, feats):
        feats = np.ascontiguousarray(feats, np.float32)
        T = feats.shape[0]
        out = np.empty((T, w.D), np.float32)
        e = [np.ascontiguousarray(w.p[n], np.float32) for n in ENC_NAMES]
        self.lib.orc_encoder(*[_p(a, _f32p) for a in e], w.F, w.D, _p(feats, _f32p), T, _p(out, _f32p))
        return out

    def decoder_project(self, w: Weights, ctxs):
        m, keep = self._model(w)
        ctxs = np.ascontiguousarray(ctxs, np.int32)
        pd = np.empty((len(ctxs), w.J), np.float32)
        self.lib.orc_decoder_project(C.byref(m), _p(ctxs, _i32p), len(ctxs), _p(pd, _f32p))
        return pd

    def joiner_logits(self, w: Weights, pe, pd):
        m, keep = self._model(w)
        pe = np.ascontiguousarray(pe, np.float32)
        pd = np.ascontiguousarray(pd, np.float32)
        out = np.empty((pe.shape[0], w.V), np.float32)
        for i in range(pe.shape[0]):
            self.lib.orc_joiner_logits_from_proj(
                C.byref(m), _p(pe[i], _f32p), _p(pd[i], _f32p), _p(out[i], _f32p)
            )
        return out

    def log_softmax(self, logits):
        logits = np.ascontiguousarray(logits, np.float32)
        out = np.empty(logits.shape, np.float64)
        for i in range(logits.shape[0]):
            self.lib.orc_log_softmax(_p(logits[i], _f32p), logits.shape[1], _p(out[i], _f64p))
        return out

    def greedy(self, w: Weights, enc, splits, threads=8):
        m, keep = self._model(w)
        enc = np.ascontiguousarray(enc, np.float32)
        splits = np.ascontiguousarray(splits, np.int32)
        B = len(splits) - 1
        osp = np.zeros(B + 1, np.int32)
        otk = np.zeros(max(1, int(splits[-1])), np.int32)
        self._check(
            self.lib.orc_greedy_batch(
                C.byref(m), _p(enc, _f32p), _p(splits, _i32p), B, threads, _p(osp, _i32p), _p(otk, _i32p)
            )
        )
        return unragged(osp, otk)

    def beam(self, w: Weights, enc, splits, beam=4, merge_op=0, length_norm=0, max_total=0, threads=8):
        m, keep = self._model(w)
        enc = np.ascontiguousarray(enc, np.float32)
        splits = np.ascontiguousarray(splits, np.int32)
        B = len(splits) - 1
        osp = np.zeros(B + 1, np.int32)
        otk = np.zeros(max(1, int(splits[-1])), np.int32)
        osc = np.zeros(B, np.float64)
        self._check(
            self.lib.orc_beam_search(
                C.byref(m),
                _p(enc, _f32p),
                _p(splits, _i32p),
                B,
                beam,
                merge_op,
                length_norm,
                max_total,
                threads,
                _p(osp, _i32p),
                _p(otk, _i32p),
                _p(osc, _f64p),
            )
        )
        return unragged(osp, otk), osc

    def fsa(self, w: Weights, enc, splits, g: Graph, beam, max_states, max_contexts, threads=8, lattices=False):
        m, keep = self._model(w)
        enc = np.ascontiguousarray(enc, np.float32)
        splits = np.ascontiguousarray(splits, np.int32)
        B = len(splits) - 1
        gg = _OrcGraph(
            g.num_states,
            g.num_arcs,
            _p(g.arc_splits, _i32p),
            _p(g.dst, _i32p),
            _p(g.label, _i32p),
            _p(g.weight, _f64p),
        )
        osp = np.zeros(B + 1, np.int32)
        otk = np.zeros(max(1, int(splits[-1])), np.int32)
        osc = np.zeros(B, np.float64)
        lats = (_OrcLattice * B)() if lattices else None
        self._check(
            self.lib.orc_fsa_beam_search(
                C.byref(m),
                _p(enc, _f32p),
                _p(splits, _i32p),
                B,
                C.byref(gg),
                beam,
                max_states,
                max_contexts,
                threads,
                _p(osp, _i32p),
                _p(otk, _i32p),
                _p(osc, _f64p),
                lats,
            )
        )
        out_lats = None
        if lattices:
            out_lats = []
            for i in range(B):
                L = lats[i]
                n = L.num_arcs
                out_lats.append(
                    dict(
                        num_nodes=L.num_nodes,
                        src=np.ctypeslib.as_array(L.src, (n,)).copy() if n else np.zeros(0, np.int32),
                        dst=np.ctypeslib.as_array(L.dst, (n,)).copy() if n else np.zeros(0, np.int32),
                        label=np.ctypeslib.as_array(L.label, (n,)).copy() if n else np.zeros(0, np.int32),
                        score=np.ctypeslib.as_array(L.score, (n,)).copy() if n else np.zeros(0, np.float64),
                    )
                )
                self.lib.orc_lattice_free(C.byref(L))
        return unragged(osp, otk), osc, out_lats


class Reference:
    """The unmodified reference (oracle/_ref/librnnt_ref.so)."""

    def __init__(self, path=REF_SO):
        if not os.path.exists(path):
            build()
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        self.lib = C.CDLL(path)
        L = self.lib
        L.ref_last_error.restype = C.c_char_p
        L.ref_model_new.restype = C.c_void_p
        L.ref_model_new.argtypes = [C.c_int32] * 5 + [C.c_uint64, C.c_double]
        L.ref_model_free.argtypes = [C.c_void_p]
        L.ref_model_param.restype = _f32p
        L.ref_model_param.argtypes = [C.c_void_p, C.c_char_p, _i32p, _i32p]
        L.ref_features.argtypes = [C.c_uint64, C.c_int32, C.c_int32, _f32p]
        L.ref_encoder_forward_batch.argtypes = [C.c_void_p, _f32p, _i32p, C.c_int32, C.c_int, _f32p]
        L.ref_decoder_project.argtypes = [C.c_void_p, _i32p, C.c_int32, _f32p]
        L.ref_joiner_logits.argtypes = [C.c_void_p, _f32p, _i32p, C.c_int32, _f32p]
        L.ref_log_softmax.argtypes = [_f32p, C.c_int32, _f64p]
        L.ref_greedy_search_batch.argtypes = [C.c_void_p, _f32p, _i32p, C.c_int32, C.c_int32, C.c_int, _i32p, _i32p]
        L.ref_greedy_search.argtypes = [C.c_void_p, _f32p, _i32p, C.c_int32, C.c_int32, C.c_int, _i32p, _i32p, C.POINTER(C.c_int64)]
        L.ref_beam_search_batch.argtypes = [C.c_void_p, _f32p, _i32p, C.c_int32] + [C.c_int32] * 5 + [
            C.c_int,
            _i32p,
            _i32p,
        ]
        L.ref_graph_trivial.restype = C.c_void_p
        L.ref_graph_trivial.argtypes = [C.c_int32]
        L.ref_graph_from_arpa.restype = C.c_void_p
        L.ref_graph_from_arpa.argtypes = [C.c_char_p, C.c_int32]
        L.ref_graph_from_text.restype = C.c_void_p
        L.ref_graph_from_text.argtypes = [C.c_char_p]
        L.ref_graph_from_arcs.restype = C.c_void_p
        L.ref_graph_from_arcs.argtypes = [C.c_int32, C.c_int32, _i32p, _i32p, _i32p, _f64p, C.c_int32, _i32p, _f64p]
        L.ref_graph_free.argtypes = [C.c_void_p]
        L.ref_graph_sizes.argtypes = [C.c_void_p, _i32p, _i32p, _i32p]
        L.ref_graph_export.argtypes = [C.c_void_p, _i32p, _i32p, _i32p, _i32p, _f64p, _i32p, _f64p]
        L.ref_graph_text.restype = C.c_void_p
        L.ref_graph_text.argtypes = [C.c_void_p]
        L.ref_free_string.argtypes = [C.c_void_p]
        L.ref_fsa_beam_search.argtypes = [
            C.c_void_p,
            _f32p,
            _i32p,
            C.c_int32,
            C.c_void_p,
            C.c_double,
            C.c_int32,
            C.c_int32,
            C.c_int,
            _i32p,
            _i32p,
            _f64p,
            C.POINTER(C.c_void_p),
        ]

        L.ref_steps_begin.argtypes = [C.c_void_p, C.c_int32, C.c_double, C.c_int32, C.c_int32, C.c_int32, _i32p]
        L.ref_steps_begin.restype = C.c_void_p
        L.ref_steps_contexts.argtypes = [C.c_void_p, _i32p, _i32p]
        L.ref_steps_step.argtypes = [C.c_void_p, _f64p, C.c_int32, C.c_int32]
        L.ref_steps_end.argtypes = [C.c_void_p, C.POINTER(C.c_void_p), _i32p, _i32p, _f64p]
        L.ref_steps_free.argtypes = [C.c_void_p]
        L.ref_fsa_logadd.argtypes = [
            C.c_void_p, _f32p, _i32p, C.c_int32, C.c_void_p, C.c_double, C.c_int32, C.c_int32, C.c_int,
            C.c_int32, C.c_uint64, _i32p, _i32p, _f64p,
        ]

    def _check(self, rc):
        if rc != 0:
            raise RuntimeError(f"reference error {rc}: {self.lib.ref_last_error().decode()}")

    # ---- model ----
    def model(self, V=500, F=80, D=512, E=512, J=512, seed=1, blank_bias=0.0):
        h = self.lib.ref_model_new(V, F, D, E, J, seed, blank_bias)
        if not h:
            raise RuntimeError(self.lib.ref_last_error().decode())
        p = {}
        for n in PARAM_NAMES + ENC_NAMES:
            r, c = C.c_int32(), C.c_int32()
            ptr = self.lib.ref_model_param(h, n.encode(), C.byref(r), C.byref(c))
            p[n] = np.ctypeslib.as_array(ptr, (r.value, c.value)).copy()
        return RefModel(self, h, Weights(V, F, D, E, J, p))

    def features(self, seed, T, F):
        out = np.empty((T, F), np.float32)
        self.lib.ref_features(seed, T, F, _p(out, _f32p))
        return out

    def log_softmax(self, logits):
        logits = np.ascontiguousarray(logits, np.float32)
        out = np.empty(logits.shape, np.float64)
        for i in range(logits.shape[0]):
            self.lib.ref_log_softmax(_p(logits[i], _f32p), logits.shape[1], _p(out[i], _f64p))
        return out

    # ---- graphs ----
    def _export(self, h):
        S, A, NF = C.c_int32(), C.c_int32(), C.c_int32()
        self.lib.ref_graph_sizes(h, C.byref(S), C.byref(A), C.byref(NF))
        sp = np.zeros(S.value + 1, np.int32)
        src = np.zeros(max(1, A.value), np.int32)
        dst = np.zeros(max(1, A.value), np.int32)
        lab = np.zeros(max(1, A.value), np.int32)
        sc = np.zeros(max(1, A.value), np.float64)
        fs = np.zeros(max(1, NF.value), np.int32)
        fw = np.zeros(max(1, NF.value), np.float64)
        self.lib.ref_graph_export(
            h, _p(sp, _i32p), _p(src, _i32p), _p(dst, _i32p), _p(lab, _i32p), _p(sc, _f64p), _p(fs, _i32p), _p(fw, _f64p)
        )
        A = A.value
        return Graph(
            S.value,
            sp,
            dst[:A].copy(),
            lab[:A].copy(),
            sc[:A].copy(),
            {int(fs[i]): float(fw[i]) for i in range(NF.value)},
        )

    def graph_trivial(self, V):
        h = self.lib.ref_graph_trivial(V)
        return RefGraph(self, h, self._export(h))

    def graph_from_arpa(self, text: str, V: int):
        h = self.lib.ref_graph_from_arpa(text.encode(), V)
        if not h:
            raise RuntimeError(self.lib.ref_last_error().decode())
        return RefGraph(self, h, self._export(h))

    def graph_from_arcs(self, num_states, src, dst, label, score, finals):
        src = np.ascontiguousarray(src, np.int32)
        dst = np.ascontiguousarray(dst, np.int32)
        label = np.ascontiguousarray(label, np.int32)
        score = np.ascontiguousarray(score, np.float64)
        fs = np.ascontiguousarray(list(finals.keys()) or [0], np.int32)
        fw = np.ascontiguousarray(list(finals.values()) or [0.0], np.float64)
        h = self.lib.ref_graph_from_arcs(
            num_states,
            len(src),
            _p(src, _i32p),
            _p(dst, _i32p),
            _p(label, _i32p),
            _p(score, _f64p),
            len(finals),
            _p(fs, _i32p),
            _p(fw, _f64p),
        )
        if not h:
            raise RuntimeError(self.lib.ref_last_error().decode())
        return RefGraph(self, h, self._export(h))


class RefGraph:
    def __init__(self, ref, h, g: Graph):
        self.ref, self.h, self.g = ref, h, g

    def text(self):
        p = self.ref.lib.ref_graph_text(self.h)
        s = C.cast(p, C.c_char_p).value.decode()
        self.ref.lib.ref_free_string(p)
        return s

    def __del__(self):
        try:
            self.ref.lib.ref_graph_free(self.h)
        except Exception:
            pass


class RefModel:
    def __init__(self, ref: Reference, h, w: Weights):
        self.ref, self.h, self.w = ref, h, w

    def __del__(self):
        try:
            self.ref.lib.ref_model_free(self.h)
        except Exception:
            pass

    def encoder(self, feats, splits, threads=8):
        feats = np.ascontiguousarray(feats, np.float32)
        splits = np.ascontiguousarray(splits, np.int32)
        out = np.empty((int(splits[-1]), self.w.D), np.float32)
        self.ref._check(
            self.ref.lib.ref_encoder_forward_batch(
                self.h, _p(feats, _f32p), _p(splits, _i32p), len(splits) - 1, threads, _p(out, _f32p)
            )
        )
        return out

    def decoder_project(self, ctxs):
        ctxs = np.ascontiguousarray(ctxs, np.int32)
        pd = np.empty((len(ctxs), self.w.J), np.float32)
        self.ref._check(self.ref.lib.ref_decoder_project(self.h, _p(ctxs, _i32p), len(ctxs), _p(pd, _f32p)))
        return pd

    def joiner_logits(self, enc_rows, ctxs):
        enc_rows = np.ascontiguousarray(enc_rows, np.float32)
        ctxs = np.ascontiguousarray(ctxs, np.int32)
        out = np.empty((len(ctxs), self.w.V), np.float32)
        self.ref._check(
            self.ref.lib.ref_joiner_logits(self.h, _p(enc_rows, _f32p), _p(ctxs, _i32p), len(ctxs), _p(out, _f32p))
        )
        return out

    def greedy(self, feats, splits, threads=8, max_symbols=1):
        feats = np.ascontiguousarray(feats, np.float32)
        splits = np.ascontiguousarray(splits, np.int32)
        B = len(splits) - 1
        osp = np.zeros(B + 1, np.int32)
        otk = np.zeros(max(1, int(splits[-1])), np.int32)
        self.ref._check(
            self.ref.lib.ref_greedy_search_batch(
                self.h, _p(feats, _f32p), _p(splits, _i32p), B, max_symbols, threads, _p(osp, _i32p), _p(otk, _i32p)
            )
        )
        return unragged(osp, otk)

    def greedy_multi(self, feats, splits, max_symbols, threads=8):
        """Reference greedy_search (any S) per utterance: (token lists, capped frames)."""
        feats = np.ascontiguousarray(feats, np.float32)
        splits = np.ascontiguousarray(splits, np.int32)
        B = len(splits) - 1
        cap = 10 if max_symbols == 2147483647 else max_symbols
        osp = np.zeros(B + 1, np.int32)
        otk = np.zeros(max(1, int(splits[-1]) * cap), np.int32)
        capped = C.c_int64(0)
        self.ref._check(
            self.ref.lib.ref_greedy_search(
                self.h, _p(feats, _f32p), _p(splits, _i32p), B, max_symbols, threads, _p(osp, _i32p),
                _p(otk, _i32p), C.byref(capped)
            )
        )
        return unragged(osp, otk), int(capped.value)

    def beam(self, feats, splits, beam=4, merge_op=0, length_norm=0, max_total=0, threads=8, max_symbols=1):
        feats = np.ascontiguousarray(feats, np.float32)
        splits = np.ascontiguousarray(splits, np.int32)
        B = len(splits) - 1
        osp = np.zeros(B + 1, np.int32)
        otk = np.zeros(max(1, int(splits[-1]) * max(1, min(max_symbols, 10))), np.int32)
        self.ref._check(
            self.ref.lib.ref_beam_search_batch(
                self.h,
                _p(feats, _f32p),
                _p(splits, _i32p),
                B,
                beam,
                max_symbols,
                merge_op,
                length_norm,
                max_total,
                threads,
                _p(osp, _i32p),
                _p(otk, _i32p),
            )
        )
        return unragged(osp, otk)

    def fsa(self, feats, splits, graph: RefGraph, beam, max_states, max_contexts, threads=8, lattice_texts=False):
        feats = np.ascontiguousarray(feats, np.float32)
        splits = np.ascontiguousarray(splits, np.int32)
        B = len(splits) - 1
        osp = np.zeros(B + 1, np.int32)
        otk = np.zeros(max(1, int(splits[-1])), np.int32)
        osc = np.zeros(B, np.float64)
        texts = (C.c_void_p * B)() if lattice_texts else None
        self.ref._check(
            self.ref.lib.ref_fsa_beam_search(
                self.h,
                _p(feats, _f32p),
                _p(splits, _i32p),
                B,
                graph.h,
                beam,
                max_states,
                max_contexts,
                threads,
                _p(osp, _i32p),
                _p(otk, _i32p),
                _p(osc, _f64p),
                texts,
            )
        )
        out_texts = None
        if lattice_texts:
            out_texts = []
            for i in range(B):
                out_texts.append(C.cast(texts[i], C.c_char_p).value.decode())
                self.ref.lib.ref_free_string(texts[i])
        return unragged(osp, otk), osc, out_texts


def _refmodel_fsa_logadd(self, feats, splits, graph, beam, max_states, max_contexts, nbest=100, seed=0,
                         threads=8):
    """lattice_to_best_seq(kLogAdd, nbest, seed) of each stream's reference
    lattice, and that sequence's total log-probability."""
    feats = np.ascontiguousarray(feats, np.float32)
    splits = np.ascontiguousarray(splits, np.int32)
    B = len(splits) - 1
    osp = np.zeros(B + 1, np.int32)
    otk = np.zeros(max(1, int(splits[-1])), np.int32)
    olp = np.zeros(max(1, B), np.float64)
    self.ref._check(
        self.ref.lib.ref_fsa_logadd(self.h, _p(feats, _f32p), _p(splits, _i32p), B, graph.h, beam, max_states,
                                    max_contexts, threads, nbest, seed, _p(osp, _i32p), _p(otk, _i32p),
                                    _p(olp, _f64p)))
    return unragged(osp, otk), olp[:B]


RefModel.fsa_logadd = _refmodel_fsa_logadd


class RefSteps:
    """The reference's Algorithm-1 step API (init_streams / get_contexts /
    expand_arcs + prune_streams / finish), driven like fsa_beam_search."""

    def __init__(self, ref: "Reference", graph: "RefGraph", params, V, num_frames):
        self.ref, self.V = ref, V
        nf = np.ascontiguousarray(num_frames, np.int32)
        self.B, self.total = len(nf), int(nf.sum())
        self.h = ref.lib.ref_steps_begin(graph.h, len(nf), params[0], params[1], params[2], V, _p(nf, _i32p))
        if not self.h:
            raise RuntimeError(ref.lib.ref_last_error().decode())

    def contexts(self):
        rs = np.zeros(self.B + 1, np.int32)
        ctx = np.zeros(max(1, self.B * 64 * 2), np.int32)
        self.ref._check(self.ref.lib.ref_steps_contexts(self.h, _p(rs, _i32p), _p(ctx, _i32p)))
        return rs, ctx[: rs[-1]].copy()

    def step(self, logprobs):
        lp = np.ascontiguousarray(logprobs, np.float64).reshape(-1, self.V)
        self.ref._check(self.ref.lib.ref_steps_step(self.h, _p(lp, _f64p), lp.shape[0], self.V))

    def end(self):
        texts = (C.c_void_p * self.B)()
        osp = np.zeros(self.B + 1, np.int32)
        otk = np.zeros(max(1, self.total), np.int32)
        osc = np.zeros(max(1, self.B), np.float64)
        self.ref._check(self.ref.lib.ref_steps_end(self.h, texts, _p(osp, _i32p), _p(otk, _i32p), _p(osc, _f64p)))
        out = []
        for i in range(self.B):
            out.append(C.cast(texts[i], C.c_char_p).value.decode())
            self.ref.lib.ref_free_string(texts[i])
        return unragged(osp, otk), osc[: self.B], out

    def __del__(self):
        if getattr(self, "h", None):
            self.ref.lib.ref_steps_free(self.h)
            self.h = None


def synthetic_arpa(V=500, n_bigrams=1500, n_trigrams=3000, seed=7):
    """Seeded synthetic trigram ARPA over tokens w1..w{V-1} (SURVEY.md §8d,
    config 4).  Uses numpy's PCG64, which is platform-deterministic; words
    map to labels by ``ref_graph_from_arpa`` ("w<k>" -> k)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    words = [f"w{k}" for k in range(1, V)]
    uni = [("<s>",), ("</s>",)] + [(w,) for w in words]
    big = set()
    while len(big) < n_bigrams:
        a = words[rng.integers(len(words))] if rng.random() > 0.1 else "<s>"
        b = words[rng.integers(len(words))]
        big.add((a, b))
    big = sorted(big)
    tri = set()
    while len(tri) < n_trigrams:
        a, b = big[rng.integers(len(big))]
        c = words[rng.integers(len(words))]
        tri.add((a, b, c))
    tri = sorted(tri)
    lines = ["\\data\\", f"ngram 1={len(uni)}", f"ngram 2={len(big)}", f"ngram 3={len(tri)}", "", "\\1-grams:"]
    for g in uni:
        lp = -99.0 if g == ("<s>",) else rng.uniform(-3.0, -0.5)
        bow = rng.uniform(-0.8, -0.05)
        lines.append(f"{lp:.4f}\t{g[0]}\t{bow:.4f}" if g != ("</s>",) else f"{lp:.4f}\t{g[0]}")
    lines += ["", "\\2-grams:"]
    for g in big:
        lines.append(f"{rng.uniform(-3.0, -0.5):.4f}\t{' '.join(g)}\t{rng.uniform(-0.8, -0.05):.4f}")
    lines += ["", "\\3-grams:"]
    for g in tri:
        lines.append(f"{rng.uniform(-3.0, -0.5):.4f}\t{' '.join(g)}")
    lines += ["", "\\end\\", ""]
    return "\n".join(lines)
