#!/usr/bin/env python3
"""Small decodes of every kernel family, for compute-sanitizer
(tests/test_gpu_sanitize.py runs it under memcheck, racecheck, synccheck):

  encoder (K1-style exact GEMM), greedy (persistent kernel and the
  thread-block-cluster kernel), modified beam search (single launch, the
  time-sliced resumable launches, S > 1 sub-steps, the bf16 tcgen05
  joiner), FSA fast beam search (trivial and a multi-state graph) with its
  lattice export, and the exact log-softmax / glibc fp64 entry points.

    python tools/sanitize_smoke.py [V=64] [B=3] [T=12]
    python tools/sanitize_smoke.py cluster [T=4]

`cluster`: the V = 500 (Vp = 512) cluster kernels only -- the small-batch
modified beam search (st.async h / logit slices, mbarrier phases) and the
greedy cluster kernel -- on two streams.

No torch: host buffers through the C ABI only."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2211_00484_b200.api import (  # noqa: E402
    BeamParams, Decoder, FsaParams, Graph, ModelWeights, f64_math, gaussian_features, init_model_weights,
    log_softmax_lse)


def cluster_kernels(T):
    w = init_model_weights(500, 80, 512, 512, 512, seed=0, blank_bias=0.4)
    dec = Decoder(ModelWeights.from_dict(w))
    dec.set_encoder(w)
    enc = dec.encoder_forward(gaussian_features(7100, 2, T, 80), np.array([0, T, 2 * T], np.int32))
    rag = np.array([0, T, T + max(1, T // 2)], np.int32)
    enc_r = np.ascontiguousarray(enc[: rag[-1]])
    dec.beam_search_batch(enc_r, rag, BeamParams(beam_size=4))  # beam_cluster_kernel
    dec.greedy_search_batch(enc_r, rag)                          # greedy_cluster_kernel
    dec.close()
    print("sanitize smoke ok", flush=True)


def main():
    if len(sys.argv) > 1 and sys.argv[1] == "cluster":
        return cluster_kernels(int(sys.argv[2]) if len(sys.argv) > 2 else 4)
    V = int(sys.argv[1]) if len(sys.argv) > 1 else 64
    B = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    T = int(sys.argv[3]) if len(sys.argv) > 3 else 12
    w = init_model_weights(V, 80, 512, 512, 512, seed=0, blank_bias=0.4)
    dec = Decoder(ModelWeights.from_dict(w))
    dec.set_encoder(w)
    feats = gaussian_features(7000, B, T, 80)
    uni = (np.arange(B + 1) * T).astype(np.int32)
    enc = dec.encoder_forward(feats, uni)
    lens = [T, 0, max(1, T // 3)][:B] + [T] * max(0, B - 3)
    rag = np.zeros(B + 1, np.int32)
    rag[1:] = np.cumsum(lens)
    enc_r = np.ascontiguousarray(enc[: rag[-1]])
    dec.greedy_search_batch(enc, uni)                        # cluster kernel (small B)
    dec.greedy_search(enc_r, rag, max_symbols=3)             # persistent greedy, S > 1
    dec.beam_search_batch(enc, uni, BeamParams(beam_size=4))  # uniform host frames: time slices
    dec.beam_search_batch(enc_r, rag, BeamParams(beam_size=4, merge_op=1))  # single launch, log-add
    dec.beam_search_batch(enc_r, rag, BeamParams(beam_size=2, max_symbols=2))  # sub-steps
    dec.set_joiner_mode("bf16")
    dec.beam_search_batch(enc_r, rag, BeamParams(beam_size=4))
    dec.set_joiner_mode("exact")
    dec.fsa_beam_search(enc_r, rag, Graph.trivial(dec), FsaParams(4.0, 8, 4))
    # a 3-state graph with parallel arcs
    src, dst, lab = [], [], []
    for s in range(3):
        for c in range(1, V):
            if (c + s) % 3 == 0:
                src.append(s)
                dst.append((s + c) % 3)
                lab.append(c)
    order = np.argsort(np.asarray(src, np.int64), kind="stable")
    src = np.asarray(src, np.int32)[order]
    splits = np.searchsorted(src, np.arange(4)).astype(np.int32)
    g = Graph(dec, 3, splits, np.asarray(dst, np.int32)[order], np.asarray(lab, np.int32)[order],
              -0.1 * np.arange(len(src), dtype=np.float64) / len(src))
    dec.fsa_beam_search(enc_r, rag, g, FsaParams(6.0, 16, 6))
    dec.fsa_lattice_text(0, header=True)
    dec.fsa_lattice_best(nbest=20, seed=3)
    # the step API, caller rows
    dec.fsa_stream_begin(g, FsaParams(6.0, 16, 6), lens)
    for t in range(max(lens)):
        rs, ctx = dec.fsa_stream_contexts()
        z = np.random.default_rng(t).normal(size=(len(ctx), V))
        dec.fsa_stream_step(z - np.log(np.exp(z).sum(1, keepdims=True)))
    dec.fsa_stream_end()
    log_softmax_lse(np.random.default_rng(0).normal(0, 3, (5, V)).astype(np.float32))
    f64_math("log1p", np.linspace(-0.5, 2.0, 100))
    dec.close()
    print("sanitize smoke ok", flush=True)


if __name__ == "__main__":
    main()
