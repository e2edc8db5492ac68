"""ctypes mirror of the reference decoder API over librnntg.so.

Reference (rnnt-kit) -> here:
  greedy_search_batch(m, batch, 1)         search.hpp:107-167  -> Decoder.greedy_search_batch
  beam_search(m, f, SearchParams)          search.hpp:206-277  -> Decoder.beam_search / beam_search_batch
  fsa_beam_search + lattice_to_best_seq    fsa_search.hpp:326-426 -> Decoder.fsa_beam_search
  Fsa (CSR arcs)                           fsa.hpp:54-80       -> Graph

Inputs are encoder frames (the reference runs its toy encoder inside each
search; the north-star boundary starts at the encoder output).  Errors map to
the reference's exception types: ValidationError (bad arguments) and
LogicError (internal inconsistency).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

from . import build as _build

_HERE = os.path.dirname(os.path.abspath(__file__))
# RNNTG_LIB: development only, A/B timing of an alternate build of the same library
lib_path = os.environ.get("RNNTG_LIB") or _build.LIB

PARAM_NAMES = ("emb", "ctx_w", "ctx_b", "j_we", "j_wd", "j_b", "out_w", "out_b")

OK, INVALID_ARGUMENT, INTERNAL, CUDA_ERROR, UNSUPPORTED = range(5)
MEM_HOST, MEM_DEVICE = 0, 1
NO_SYMBOL_LIMIT = 2147483647  # RNNTG_NO_SYMBOL_LIMIT (search.hpp:30 kNoSymbolLimit)
MERGE_MAX, MERGE_LOG_ADD = 0, 1
CUDA_STREAM_LEGACY = 0x1  # cudaStreamLegacy (driver_types.h)


class RnntgError(RuntimeError):
    """CUDA or capability error from librnntg."""


class ValidationError(RnntgError, ValueError):
    """The reference's rnnt::ValidationError (common.hpp:38-40)."""


class LogicError(RnntgError):
    """The reference's std::logic_error."""


class UnsupportedError(RnntgError):
    """Valid for the reference, beyond a documented device cap."""


class _Desc(C.Structure):
    _fields_ = [
        ("vocab_size", C.c_int32),
        ("enc_dim", C.c_int32),
        ("emb_dim", C.c_int32),
        ("joiner_dim", C.c_int32),
        ("context_size", C.c_int32),
    ] + [(n, C.POINTER(C.c_float)) for n in PARAM_NAMES]


class _EncDesc(C.Structure):
    _fields_ = [("feat_dim", C.c_int32)] + [
        (n, C.POINTER(C.c_float)) for n in ("enc_w1", "enc_b1", "enc_w2", "enc_b2")
    ]


class _BeamParams(C.Structure):
    _fields_ = [
        ("beam_size", C.c_int32),
        ("max_symbols", C.c_int32),
        ("merge_op", C.c_int32),
        ("length_norm", C.c_int32),
        ("max_total_symbols", C.c_int32),
    ]


class _FsaParams(C.Structure):
    _fields_ = [("beam", C.c_double), ("max_states", C.c_int32), ("max_contexts", C.c_int32)]


class _Stats(C.Structure):
    _fields_ = [
        ("stream_frames", C.c_int64),
        ("joiner_rows", C.c_int64),
        ("arcs_expanded", C.c_int64),
        ("lattice_arcs", C.c_int64),
        ("tie_breaks", C.c_int64),
        ("kernel_launches", C.c_int64),
        ("gpu_ms", C.c_float),
        ("decode_ms", C.c_float),
        ("phase_cycles", C.c_int64 * 4),
        ("joiner_rows_computed", C.c_int64),
        ("gather_cycles", C.c_int64),
        ("gemm_wait_cycles", C.c_int64),
        ("capped_frames", C.c_int64),
    ]


_lib = None


def _load():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(lib_path):
        # Build in-tree (nvcc cross-compiles without a GPU); never fall back.
        _build.build()
    lib = C.CDLL(lib_path)
    vp, i32, i32p, f32p, f64p = C.c_void_p, C.c_int32, C.POINTER(C.c_int32), C.c_void_p, C.c_void_p
    lib.rnntg_last_error.restype = C.c_char_p
    lib.rnntg_version.restype = C.c_char_p
    lib.rnntg_model_create.argtypes = [C.POINTER(_Desc), i32, C.POINTER(vp)]
    lib.rnntg_model_destroy.argtypes = [vp]
    lib.rnntg_set_stream.argtypes = [vp, vp]
    lib.rnntg_set_joiner_mode.argtypes = [vp, i32]
    lib.rnntg_get_stats.argtypes = [vp, C.POINTER(_Stats)]
    lib.rnntg_greedy_search_batch.argtypes = [vp, f32p, i32p, i32, i32, i32, i32p, vp]
    lib.rnntg_greedy_search.argtypes = [vp, f32p, i32p, i32, i32, i32, i32p, vp, C.POINTER(C.c_int64)]
    lib.rnntg_beam_search_batch.argtypes = [vp, f32p, i32p, i32, C.POINTER(_BeamParams), i32, i32p, vp, f64p]
    lib.rnntg_graph_create.argtypes = [vp, i32, i32p, i32, i32p, i32p, f64p, C.POINTER(vp)]
    lib.rnntg_graph_destroy.argtypes = [vp]
    lib.rnntg_fsa_beam_search.argtypes = [vp, f32p, i32p, i32, vp, C.POINTER(_FsaParams), i32, i32p, vp, f64p]
    lib.rnntg_fsa_lattice.argtypes = [vp, i32, C.POINTER(C.c_int32), C.POINTER(C.c_int32), i32, vp, vp, vp, vp]
    lib.rnntg_fsa_lattice.restype = C.c_int
    lib.rnntg_fsa_lattice_text.argtypes = [vp, i32, i32, C.c_char_p, C.c_int64, C.POINTER(C.c_int64)]
    lib.rnntg_fsa_lattice_best.argtypes = [vp, i32, i32, C.c_uint64, i32p, vp, vp]
    lib.rnntg_fsa_stream_begin.argtypes = [vp, vp, C.POINTER(_FsaParams), i32, i32p]
    lib.rnntg_fsa_stream_contexts.argtypes = [vp, i32p, i32, i32p]
    lib.rnntg_fsa_stream_step.argtypes = [vp, vp, i32]
    lib.rnntg_fsa_stream_end.argtypes = [vp, i32p, vp, vp]
    lib.rnntg_model_set_encoder.argtypes = [vp, C.POINTER(_EncDesc)]
    lib.rnntg_encoder_forward.argtypes = [vp, f32p, i32p, i32, i32, vp]
    lib.rnntg_debug_decoder_projection.argtypes = [vp, i32p, i32, f32p]
    lib.rnntg_debug_joiner_logits.argtypes = [vp, f32p, i32p, i32, f32p]
    lib.rnntg_debug_tanhf_chunk_hashes.argtypes = [i32, i32, i32, C.POINTER(C.c_uint64)]
    lib.rnntg_debug_log_softmax_lse.argtypes = [i32, f32p, i32, i32, vp]
    lib.rnntg_debug_f64_math.argtypes = [i32, i32, vp, C.c_int64, vp]
    lib.rnntg_init_model_weights.argtypes = [vp, vp]
    lib.rnntg_gaussian_features.argtypes = [C.c_uint64, i32, i32, i32, i32, vp]
    for f in (
        "rnntg_model_create",
        "rnntg_model_destroy",
        "rnntg_set_stream",
        "rnntg_set_joiner_mode",
        "rnntg_get_stats",
        "rnntg_greedy_search_batch",
        "rnntg_beam_search_batch",
        "rnntg_graph_create",
        "rnntg_graph_destroy",
        "rnntg_fsa_beam_search",
        "rnntg_fsa_lattice_text",
        "rnntg_fsa_lattice_best",
        "rnntg_fsa_stream_begin",
        "rnntg_fsa_stream_contexts",
        "rnntg_fsa_stream_step",
        "rnntg_fsa_stream_end",
        "rnntg_model_set_encoder",
        "rnntg_encoder_forward",
        "rnntg_debug_decoder_projection",
        "rnntg_debug_joiner_logits",
        "rnntg_debug_tanhf_chunk_hashes",
        "rnntg_debug_log_softmax_lse",
        "rnntg_debug_f64_math",
        "rnntg_init_model_weights",
        "rnntg_gaussian_features",
    ):
        getattr(lib, f).restype = C.c_int
    _lib = lib
    return lib


def _check(rc):
    if rc == OK:
        return
    msg = _load().rnntg_last_error().decode()
    raise {INVALID_ARGUMENT: ValidationError, INTERNAL: LogicError, UNSUPPORTED: UnsupportedError}.get(
        rc, RnntgError
    )(msg)


def _ptr(a):
    return C.c_void_p(a.ctypes.data)


def _i32p(a):
    return a.ctypes.data_as(C.POINTER(C.c_int32))


@dataclass
class ModelWeights:
    """Stateless-transducer weights in param_views naming (model.hpp:75-82)."""

    V: int
    D: int
    E: int
    J: int
    p: dict

    @staticmethod
    def from_dict(p: dict) -> "ModelWeights":
        V, E = p["emb"].shape
        J, D = p["j_we"].shape
        return ModelWeights(V, D, E, J, {n: np.ascontiguousarray(p[n], np.float32) for n in PARAM_NAMES})


@dataclass
class BeamParams:
    """SearchParams (search.hpp:44-50) at max_symbols = 1."""

    beam_size: int = 4
    max_symbols: int = 1
    merge_op: int = MERGE_MAX
    length_norm: bool = False
    max_total_symbols: int = 0


@dataclass
class FsaParams:
    """FsaSearchParams (fsa_search.hpp:33-37)."""

    beam: float = 20.0
    max_states: int = 64
    max_contexts: int = 8


def _frames(enc, frame_splits):
    """(pointer, mem kind, keepalive) for host numpy / torch tensors."""
    splits = np.ascontiguousarray(frame_splits, np.int32)
    if hasattr(enc, "data_ptr"):  # torch tensor
        if enc.dtype.__str__() != "torch.float32" or not enc.is_contiguous():
            raise ValidationError("enc must be a contiguous float32 tensor")
        mem = MEM_DEVICE if enc.is_cuda else MEM_HOST
        return C.c_void_p(enc.data_ptr()), mem, splits, enc
    a = np.ascontiguousarray(enc, np.float32)
    return _ptr(a), MEM_HOST, splits, a


def _ragged(splits, flat):
    return [flat[splits[i] : splits[i + 1]].tolist() for i in range(len(splits) - 1)]


class Graph:
    """Device copy of a CSR decoding graph (fsa.hpp:54-80)."""

    def __init__(self, decoder: "Decoder", num_states, arc_splits, dst, label, weight):
        lib = _load()
        self._lib = lib
        self.num_states = int(num_states)
        arc_splits = np.ascontiguousarray(arc_splits, np.int32)
        dst = np.ascontiguousarray(dst, np.int32)
        label = np.ascontiguousarray(label, np.int32)
        weight = np.ascontiguousarray(weight, np.float64)
        self.num_arcs = int(dst.shape[0])
        h = C.c_void_p()
        _check(
            lib.rnntg_graph_create(
                decoder.h,
                self.num_states,
                _i32p(arc_splits),
                self.num_arcs,
                _i32p(dst),
                _i32p(label),
                _ptr(weight),
                C.byref(h),
            )
        )
        self.h = h

    @staticmethod
    def trivial(decoder: "Decoder") -> "Graph":
        """trivial_graph (fsa.hpp:266-273): one state, self-loops 1..V-1, score 0."""
        V = decoder.V
        return Graph(
            decoder,
            1,
            np.array([0, V - 1], np.int32),
            np.zeros(V - 1, np.int32),
            np.arange(1, V, dtype=np.int32),
            np.zeros(V - 1, np.float64),
        )

    def __del__(self):
        if getattr(self, "h", None):
            self._lib.rnntg_graph_destroy(self.h)
            self.h = None


class Decoder:
    """A model resident on one GPU (rnntg_model_t)."""

    def __init__(self, weights: ModelWeights, device: int = 0):
        lib = _load()
        self._lib = lib
        self.w = weights
        self.V, self.D, self.E, self.J = weights.V, weights.D, weights.E, weights.J
        arrs = [np.ascontiguousarray(weights.p[n], np.float32) for n in PARAM_NAMES]
        desc = _Desc(
            weights.V,
            weights.D,
            weights.E,
            weights.J,
            2,
            *[a.ctypes.data_as(C.POINTER(C.c_float)) for a in arrs],
        )
        h = C.c_void_p()
        _check(lib.rnntg_model_create(C.byref(desc), device, C.byref(h)))
        self.h = h
        self.device = device
        self._last_fsa_splits = None

    def close(self):
        if getattr(self, "h", None):
            self._lib.rnntg_model_destroy(self.h)
            self.h = None

    def __del__(self):
        self.close()

    def set_encoder(self, p: dict):
        """Uploads the reference toy encoder (enc_w1/enc_b1/enc_w2/enc_b2)."""
        self._enc_keep = [np.ascontiguousarray(p[n], np.float32) for n in ("enc_w1", "enc_b1", "enc_w2", "enc_b2")]
        desc = _EncDesc(
            int(self._enc_keep[0].shape[1]), *[a.ctypes.data_as(C.POINTER(C.c_float)) for a in self._enc_keep]
        )
        _check(self._lib.rnntg_model_set_encoder(self.h, C.byref(desc)))
        self.F = int(self._enc_keep[0].shape[1])

    def encoder_forward(self, feats, frame_splits, out=None):
        """encoder_forward (model.hpp:224-238) on the GPU, bit-exact.  Host
        numpy in -> numpy out; CUDA tensor in -> `out` (CUDA tensor) filled."""
        p, mem, splits, keep = _frames(feats, frame_splits)
        B = len(splits) - 1
        if mem == MEM_DEVICE:
            _check(self._lib.rnntg_encoder_forward(self.h, p, _i32p(splits), B, mem, C.c_void_p(out.data_ptr())))
            return out
        enc = np.zeros((int(splits[-1]), self.D), np.float32)
        _check(self._lib.rnntg_encoder_forward(self.h, p, _i32p(splits), B, mem, _ptr(enc)))
        return enc

    def set_joiner_mode(self, mode: str):
        """"exact" (default, bit-exact fp32 on CUDA cores) or "bf16" (tcgen05
        tensor cores, bf16 operands, fp32 accumulation; not token-exact)."""
        _check(self._lib.rnntg_set_joiner_mode(self.h, {"exact": 0, "bf16": 1}[mode]))

    def set_stream(self, stream_handle: int | None):
        """Run this handle's work on `stream_handle` (a cudaStream_t as an
        int, e.g. torch.cuda.current_stream().cuda_stream).  None selects the
        handle's own stream.  torch's default stream reports handle 0, which
        is the legacy default stream: it is passed as cudaStreamLegacy so the
        decode stays ordered with the caller's work (the C ABI reads NULL as
        "the handle's own stream")."""
        if stream_handle is None:
            h = 0
        else:
            h = int(stream_handle) or CUDA_STREAM_LEGACY
        _check(self._lib.rnntg_set_stream(self.h, C.c_void_p(h)))

    def stats(self) -> dict:
        s = _Stats()
        _check(self._lib.rnntg_get_stats(self.h, C.byref(s)))
        d = {f: getattr(s, f) for f, _ in _Stats._fields_}
        d["phase_cycles"] = list(d["phase_cycles"])
        return d

    # ---- searches ----
    def greedy_search_batch(self, enc, frame_splits, max_symbols=1, out_tokens=None):
        p, mem, splits, keep = _frames(enc, frame_splits)
        B = len(splits) - 1
        osp = np.zeros(B + 1, np.int32)
        if mem == MEM_DEVICE:
            if out_tokens is None or not out_tokens.is_cuda:
                raise ValidationError("device frames need a device out_tokens tensor")
            tok, tokp = out_tokens, C.c_void_p(out_tokens.data_ptr())
        else:
            tok = np.zeros(max(1, int(splits[-1])), np.int32)
            tokp = _ptr(tok)
        _check(self._lib.rnntg_greedy_search_batch(self.h, p, _i32p(splits), B, max_symbols, mem, _i32p(osp), tokp))
        if mem == MEM_DEVICE:
            return osp, tok
        return _ragged(osp, tok)

    def greedy_search(self, enc, frame_splits, max_symbols=1):
        """greedy_search (search.hpp:76-100) for every stream, any S
        (NO_SYMBOL_LIMIT = unlimited, capped at 10 per frame).  Returns
        (token lists, frames stopped by the cap)."""
        p, mem, splits, keep = _frames(enc, frame_splits)
        B = len(splits) - 1
        cap = 10 if max_symbols == NO_SYMBOL_LIMIT else max_symbols
        osp = np.zeros(B + 1, np.int32)
        tok = np.zeros(max(1, int(splits[-1]) * max(1, cap)), np.int32)
        capped = C.c_int64(0)
        if mem == MEM_DEVICE:
            raise ValueError("greedy_search: host frames only in this binding")
        _check(self._lib.rnntg_greedy_search(self.h, p, _i32p(splits), B, max_symbols, mem, _i32p(osp), _ptr(tok),
                                             C.byref(capped)))
        return _ragged(osp, tok), int(capped.value)

    def beam_search_batch(self, enc, frame_splits, params: BeamParams = BeamParams(), out_tokens=None, out_scores=None,
                          as_lists=True):
        """Host frames: (token lists, scores), or with as_lists=False the flat
        form the C ABI returns, (out_splits, tokens, scores) as numpy arrays
        (no per-stream Python lists).  Device frames: (out_splits, out_tokens,
        out_scores) written into the caller's device tensors."""
        p, mem, splits, keep = _frames(enc, frame_splits)
        B = len(splits) - 1
        osp = np.zeros(B + 1, np.int32)
        bp = _BeamParams(
            params.beam_size, params.max_symbols, params.merge_op, int(params.length_norm), params.max_total_symbols
        )
        if mem == MEM_DEVICE:
            if out_tokens is None or out_scores is None or not (out_tokens.is_cuda and out_scores.is_cuda):
                raise ValidationError("device frames need device out_tokens and out_scores tensors")
            tokp, scp = C.c_void_p(out_tokens.data_ptr()), C.c_void_p(out_scores.data_ptr())
        else:
            cap = 10 if params.max_symbols == NO_SYMBOL_LIMIT else max(1, params.max_symbols)
            tok = np.empty(max(1, int(splits[-1]) * cap), np.int32)  # capacity; only osp[-1] are written
            sc = np.zeros(max(1, B), np.float64)
            tokp, scp = _ptr(tok), _ptr(sc)
        _check(self._lib.rnntg_beam_search_batch(self.h, p, _i32p(splits), B, C.byref(bp), mem, _i32p(osp), tokp, scp))
        if mem == MEM_DEVICE:
            return osp, out_tokens, out_scores
        if not as_lists:
            return osp, tok[: osp[-1]], sc[:B]
        return _ragged(osp, tok), sc[:B].copy()

    def beam_search(self, enc_one, params: BeamParams = BeamParams()):
        """Per-utterance form of the reference's beam_search (returns ys)."""
        enc_one = np.ascontiguousarray(enc_one, np.float32)
        ys, _ = self.beam_search_batch(enc_one, [0, enc_one.shape[0]], params)
        return ys[0]

    def fsa_beam_search(self, enc, frame_splits, graph: Graph, params: FsaParams = FsaParams(), out_tokens=None,
                        out_scores=None):
        """Host frames: (token lists, best-path scores).  Device frames:
        the caller's device tensors out_tokens (>= frame_splits[-1] int32)
        and out_scores (B float64) are filled and (out_splits, out_tokens,
        out_scores) returned, as beam_search_batch does."""
        p, mem, splits, keep = _frames(enc, frame_splits)
        B = len(splits) - 1
        osp = np.zeros(B + 1, np.int32)
        fp = _FsaParams(float(params.beam), int(params.max_states), int(params.max_contexts))
        if mem == MEM_DEVICE:
            if out_tokens is None or out_scores is None or not (out_tokens.is_cuda and out_scores.is_cuda):
                raise ValidationError("device frames need device out_tokens and out_scores tensors")
            tokp, scp = C.c_void_p(out_tokens.data_ptr()), C.c_void_p(out_scores.data_ptr())
        else:
            tok = np.zeros(max(1, int(splits[-1])), np.int32)
            sc = np.zeros(max(1, B), np.float64)
            tokp, scp = _ptr(tok), _ptr(sc)
        _check(
            self._lib.rnntg_fsa_beam_search(
                self.h, p, _i32p(splits), B, graph.h, C.byref(fp), mem, _i32p(osp), tokp, scp
            )
        )
        self._last_fsa_splits = np.array(splits, np.int32)
        if mem == MEM_DEVICE:
            return osp, out_tokens, out_scores
        return _ragged(osp, tok), sc[:B].copy()

    def fsa_lattice(self, stream: int) -> dict:
        """Lattice of `stream` from the last fsa_beam_search, in the
        reference's Fsa layout (build_lattice + make_fsa order)."""
        nn, na = C.c_int32(), C.c_int32()
        _check(self._lib.rnntg_fsa_lattice(self.h, stream, C.byref(nn), C.byref(na), 0, None, None, None, None))
        n = na.value
        src, dst, lab = (np.zeros(max(1, n), np.int32) for _ in range(3))
        sc = np.zeros(max(1, n), np.float64)
        _check(
            self._lib.rnntg_fsa_lattice(
                self.h, stream, C.byref(nn), C.byref(na), n, _ptr(src), _ptr(dst), _ptr(lab), _ptr(sc)
            )
        )
        return dict(num_nodes=nn.value, src=src[:n], dst=dst[:n], label=lab[:n], score=sc[:n])

    # ---- the Algorithm-1 step API (fsa_search.hpp:95-297) ----
    def fsa_stream_begin(self, graph: Graph, params: FsaParams, num_frames):
        """init_streams over len(num_frames) streams sharing `graph`."""
        nf = np.ascontiguousarray(num_frames, np.int32)
        fp = _FsaParams(float(params.beam), int(params.max_states), int(params.max_contexts))
        _check(self._lib.rnntg_fsa_stream_begin(self.h, graph.h, C.byref(fp), len(nf), _i32p(nf)))
        self._step_graph = graph  # the device graph must outlive the decode (DecodeStream::graph)
        self._step_B = len(nf)
        self._last_fsa_splits = np.concatenate([[0], np.cumsum(nf)]).astype(np.int32)

    def fsa_stream_contexts(self):
        """get_contexts: (row_splits [B+1], packed contexts a*V+b per row)."""
        rs = np.zeros(self._step_B + 1, np.int32)
        _check(self._lib.rnntg_fsa_stream_contexts(self.h, _i32p(rs), 0, None))
        ctx = np.zeros(max(1, int(rs[-1])), np.int32)
        _check(self._lib.rnntg_fsa_stream_contexts(self.h, _i32p(rs), len(ctx), _i32p(ctx)))
        return rs, ctx[: rs[-1]]

    def fsa_stream_step(self, logprobs):
        """expand_arcs + prune_streams with the caller's log-prob rows [rows][V]."""
        if hasattr(logprobs, "is_cuda") and logprobs.is_cuda:
            _check(self._lib.rnntg_fsa_stream_step(self.h, C.c_void_p(logprobs.data_ptr()), MEM_DEVICE))
            return
        lp = np.ascontiguousarray(logprobs, np.float64)
        _check(self._lib.rnntg_fsa_stream_step(self.h, _ptr(lp) if lp.size else None, MEM_HOST))

    def fsa_stream_end(self):
        """finish_stream + lattice_to_best_seq(kMax): (token lists, best-path scores)."""
        B = self._step_B
        osp = np.zeros(B + 1, np.int32)
        tok = np.zeros(max(1, int(self._last_fsa_splits[-1])), np.int32)
        sc = np.zeros(max(1, B), np.float64)
        _check(self._lib.rnntg_fsa_stream_end(self.h, _i32p(osp), _ptr(tok), _ptr(sc)))
        return _ragged(osp, tok), sc[:B].copy()

    def fsa_lattice_best(self, nbest: int = 100, seed: int = 0, merge_op: int = MERGE_LOG_ADD):
        """lattice_to_best_seq(lattice, kLogAdd, nbest, seed) of every stream
        of the last fsa_beam_search (fsa_search.hpp:410-425), on the GPU:
        (token lists, total log-probabilities of the chosen sequences)."""
        B = len(self._last_fsa_splits) - 1 if self._last_fsa_splits is not None else 0
        osp = np.zeros(B + 1, np.int32)
        tok = np.zeros(max(1, int(self._last_fsa_splits[-1]) if B else 1), np.int32)
        lp = np.zeros(max(1, B), np.float64)
        _check(self._lib.rnntg_fsa_lattice_best(self.h, merge_op, nbest, seed, _i32p(osp), _ptr(tok), _ptr(lp)))
        return _ragged(osp, tok), lp[:B].copy()

    def fsa_lattice_text(self, stream: int, header: bool = False) -> str:
        """serialize_fsa_text (or, with header, serialize_lattice) of
        `stream`'s lattice from the last fsa_beam_search."""
        n = C.c_int64()
        _check(self._lib.rnntg_fsa_lattice_text(self.h, stream, int(header), None, 0, C.byref(n)))
        buf = C.create_string_buffer(n.value + 1)
        _check(self._lib.rnntg_fsa_lattice_text(self.h, stream, int(header), buf, n.value + 1, C.byref(n)))
        return buf.value.decode()

    # ---- kernel-level parity ----
    def decoder_projection(self, ctxs):
        ctxs = np.ascontiguousarray(ctxs, np.int32)
        out = np.zeros((len(ctxs), self.J), np.float32)
        _check(self._lib.rnntg_debug_decoder_projection(self.h, _i32p(ctxs), len(ctxs), _ptr(out)))
        return out

    def joiner_logits(self, enc_rows, ctxs):
        enc_rows = np.ascontiguousarray(enc_rows, np.float32)
        ctxs = np.ascontiguousarray(ctxs, np.int32)
        out = np.zeros((len(ctxs), self.V), np.float32)
        _check(self._lib.rnntg_debug_joiner_logits(self.h, _ptr(enc_rows), _i32p(ctxs), len(ctxs), _ptr(out)))
        return out


class _ModelConfig(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("vocab_size", "feat_dim", "enc_dim", "emb_dim", "joiner_dim")] + [
        ("seed", C.c_uint64)
    ]


_WEIGHT_ORDER = ("enc_w1", "enc_b1", "enc_w2", "enc_b2") + PARAM_NAMES


class _WeightPtrs(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in _WEIGHT_ORDER]


def init_model_weights(vocab_size=500, feat_dim=80, enc_dim=512, emb_dim=512, joiner_dim=512, seed=1,
                       blank_bias=0.0) -> dict:
    """The reference's init_model weights (model.hpp:129-169), bit for bit,
    as param_views-named float32 arrays (encoder included); `blank_bias` is
    added to out_b[0] in float, as the north-star configs do."""
    V, F, D, E, J = vocab_size, feat_dim, enc_dim, emb_dim, joiner_dim
    shapes = {"enc_w1": (D, F), "enc_b1": (1, D), "enc_w2": (D, D), "enc_b2": (1, D), "emb": (V, E),
              "ctx_w": (E, 2 * E), "ctx_b": (1, E), "j_we": (J, D), "j_wd": (J, E), "j_b": (1, J),
              "out_w": (V, J), "out_b": (1, V)}
    p = {n: np.zeros(shapes[n], np.float32) for n in _WEIGHT_ORDER}
    ptrs = _WeightPtrs(*[p[n].ctypes.data for n in _WEIGHT_ORDER])
    _check(_load().rnntg_init_model_weights(C.byref(_ModelConfig(V, F, D, E, J, seed)), C.byref(ptrs)))
    p["out_b"][0, 0] = np.float32(p["out_b"][0, 0] + np.float32(blank_bias))
    return p


def gaussian_features(seed0, B, T, feat_dim=80, threads=0, out=None):
    """Per-stream synthetic features [B*T, feat_dim]: stream i is
    DetRng(seed0 + i).gaussian(), bit-identical to the
    reference's generator.  `out` may be a (pinned) host buffer to fill."""
    if B < 0 or T < 0 or feat_dim < 1:
        raise ValidationError("bad feature shape")
    if out is None:
        out = np.empty((B * T, feat_dim), np.float32)
    ptr = out.data_ptr() if hasattr(out, "data_ptr") else out.ctypes.data
    _check(_load().rnntg_gaussian_features(C.c_uint64(seed0), B, T, feat_dim, threads, C.c_void_p(ptr)))
    return out


def tanhf_chunk_hashes(first_chunk=0, num_chunks=256, device=0):
    out = (C.c_uint64 * num_chunks)()
    _check(_load().rnntg_debug_tanhf_chunk_hashes(device, first_chunk, num_chunks, out))
    return [int(x) for x in out]


def exported_symbols():
    """Names declared in include/rnntg.h (for the ABI export test)."""
    import re

    hdr = open(os.path.join(_HERE, "..", "include", "rnntg.h")).read()
    return sorted(set(re.findall(r"\b(rnntg_[a-z_0-9]+)\s*\(", hdr)))


def log_softmax_lse(logits, device=0):
    """Device log-softmax normalisers of fp32 rows [n][V] (model.hpp:115-125)."""
    x = np.ascontiguousarray(logits, np.float32)
    n, V = x.shape
    out = np.zeros(max(1, n), np.float64)
    _check(_load().rnntg_debug_log_softmax_lse(device, _ptr(x), n, V, _ptr(out)))
    return out[:n]


F64_OPS = {"exp": 0, "log": 1, "log1p": 2, "exp_g": 3}


def f64_math(op, x, device=0):
    """Device glibc exp / log / log1p ports (glibc_f64.h) over x."""
    a = np.ascontiguousarray(x, np.float64)
    y = np.zeros(max(1, a.size), np.float64)
    _check(_load().rnntg_debug_f64_math(device, F64_OPS[op], _ptr(a), a.size, _ptr(y)))
    return y[: a.size]
