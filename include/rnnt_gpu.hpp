// rnnt_gpu.hpp — header-only C++ drop-in for the reference decoder API
// (rnnt-kit) on top of the rnntg C ABI (rnntg.h).
//
// Include AFTER the reference headers (it uses rnnt::ToyTransducer, Mat,
// SearchParams, Fsa, FsaSearchParams and the reference exception types) and
// link librnntg.so.  Each function keeps the reference signature plus a
// leading rnnt::gpu::Context& (the device-resident model):
//
//   rnnt::greedy_search_batch(m, batch, 1)      search.hpp:107-167
//     -> rnnt::gpu::greedy_search_batch(ctx, m, batch, 1)
//   rnnt::beam_search(m, features, params)      search.hpp:206-277
//     -> rnnt::gpu::beam_search(ctx, m, features, params)
//        (+ beam_search_batch: one call for a whole batch of utterances)
//   rnnt::fsa_beam_search + lattice_to_best_seq(kMax)   fsa_search.hpp:326-409
//     -> rnnt::gpu::fsa_best_sequences(ctx, m, batch, graph, params)
//
// Like the reference, each search takes acoustic features.  The encoder
// (encoder_forward, model.hpp:224-238) runs on the GPU, bit-exact with the
// reference's (RNNTG_MEM_HOST_FEATURES: features in, device-resident frames,
// host results), so a call costs one H2D copy of the features and no host
// compute; callers that already hold encoder frames use the C ABI directly.
// Decoding graphs are uploaded once per Context and reused for every call
// with the same graph content.
// Errors map back to the reference's types: RNNTG_INVALID_ARGUMENT ->
// rnnt::ValidationError, RNNTG_INTERNAL -> std::logic_error, anything else ->
// std::runtime_error.
#ifndef RNNT_GPU_HPP_
#define RNNT_GPU_HPP_

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "rnntg.h"

namespace rnnt {
namespace gpu {

inline void check(rnntg_status st) {
  if (st == RNNTG_OK) return;
  const std::string msg = rnntg_last_error();
  if (st == RNNTG_INVALID_ARGUMENT) throw ValidationError(msg);
  if (st == RNNTG_INTERNAL) throw std::logic_error(msg);
  throw std::runtime_error("rnntg: " + msg);
}

// A model resident on one GPU.  Weights are taken from the reference model
// in param_views naming (model.hpp:75-82).
class Context {
 public:
  explicit Context(const ToyTransducer& m, int32_t device = 0) {
    check_model_shapes(m);
    rnntg_model_desc d{};
    d.vocab_size = m.cfg.vocab_size;
    d.enc_dim = m.cfg.enc_dim;
    d.emb_dim = m.cfg.emb_dim;
    d.joiner_dim = m.cfg.joiner_dim;
    d.context_size = m.cfg.context_size;
    d.emb = m.emb.data.data();
    d.ctx_w = m.ctx_w.data.data();
    d.ctx_b = m.ctx_b.data.data();
    d.j_we = m.j_we.data.data();
    d.j_wd = m.j_wd.data.data();
    d.j_b = m.j_b.data.data();
    d.out_w = m.out_w.data.data();
    d.out_b = m.out_b.data.data();
    check(rnntg_model_create(&d, device, &h_));
    vocab_ = m.cfg.vocab_size;
    rnntg_encoder_desc e{};
    e.feat_dim = m.cfg.feat_dim;
    e.enc_w1 = m.enc_w1.data.data();
    e.enc_b1 = m.enc_b1.data.data();
    e.enc_w2 = m.enc_w2.data.data();
    e.enc_b2 = m.enc_b2.data.data();
    const rnntg_status st = rnntg_model_set_encoder(h_, &e);
    if (st != RNNTG_OK) {
      rnntg_model_destroy(h_);
      check(st);
    }
  }
  ~Context() {
    for (Cached& c : graphs_) rnntg_graph_destroy(c.handle);
    rnntg_host_free(stage_);
    rnntg_model_destroy(h_);
  }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  rnntg_model_t handle() const { return h_; }
  int32_t vocab_size() const { return vocab_; }

  // Pinned staging for a call's features, kept across calls (grown, never
  // shrunk): no page faults on a fresh buffer, one fast asynchronous DMA.
  float* staging(size_t floats) {
    if (floats > stage_cap_) {
      check(rnntg_host_free(stage_));
      stage_ = nullptr;
      stage_cap_ = 0;
      const size_t cap = std::max(floats, stage_cap_ + stage_cap_ / 2);
      void* p = nullptr;
      check(rnntg_host_alloc(cap * sizeof(float), &p));
      stage_ = static_cast<float*>(p);
      stage_cap_ = cap;
    }
    return stage_;
  }

  // The device copy of `graph` (fsa.hpp:54-80), uploaded on first use and
  // reused by content (a 64-bit hash of the CSR, confirmed by Fsa equality).
  rnntg_graph_t graph(const Fsa& graph) {
    const uint64_t key = hash(graph);
    for (Cached& c : graphs_)
      if (c.key == key && *c.copy == graph) return c.handle;
    std::vector<int32_t> dst, label;
    std::vector<double> w;
    dst.reserve(graph.arcs.size());
    label.reserve(graph.arcs.size());
    w.reserve(graph.arcs.size());
    for (const Arc& a : graph.arcs) {
      dst.push_back(a.dst);
      label.push_back(a.label);
      w.push_back(a.score);
    }
    rnntg_graph_t g = nullptr;
    check(rnntg_graph_create(h_, graph.num_states, graph.arc_splits.data(),
                             static_cast<int32_t>(graph.arcs.size()), dst.data(), label.data(), w.data(), &g));
    graphs_.push_back({key, std::make_unique<Fsa>(graph), g});
    return g;
  }

 private:
  struct Cached {
    uint64_t key;
    std::unique_ptr<Fsa> copy;
    rnntg_graph_t handle;
  };
  static uint64_t hash(const Fsa& g) {
    uint64_t x = 0xcbf29ce484222325ull ^ static_cast<uint64_t>(g.num_states);
    auto mix = [&x](uint64_t v) { x = (x ^ v) * 0x100000001b3ull; };
    for (int32_t v : g.arc_splits) mix(static_cast<uint32_t>(v));
    for (const Arc& a : g.arcs) {
      uint64_t b;
      std::memcpy(&b, &a.score, 8);
      mix((static_cast<uint64_t>(static_cast<uint32_t>(a.dst)) << 32) | static_cast<uint32_t>(a.label));
      mix(b);
    }
    return x;
  }
  rnntg_model_t h_ = nullptr;
  int32_t vocab_ = 0;
  std::vector<Cached> graphs_;
  float* stage_ = nullptr;
  size_t stage_cap_ = 0;
};

namespace detail {

// The batch's features, concatenated into the Context's pinned staging
// buffer (streams copied by up to 16 threads for large batches), with the
// reference encoder's validation (model.hpp:226-228); the GPU runs the
// encoder itself.
struct Frames {
  const float* enc = nullptr;  // features [sum T][F] (RNNTG_MEM_HOST_FEATURES), pinned
  std::vector<int32_t> splits;
};

inline Frames encode(Context& ctx, const ToyTransducer& m, const std::vector<Mat<float>>& batch) {
  check_model_shapes(m);
  Frames f;
  f.splits.reserve(batch.size() + 1);
  f.splits.push_back(0);
  std::vector<size_t> off(batch.size() + 1, 0);
  for (size_t i = 0; i < batch.size(); ++i) {
    const Mat<float>& x = batch[i];
    if (x.cols != m.cfg.feat_dim) throw ValidationError("features must have feat_dim columns");
    f.splits.push_back(f.splits.back() + x.rows);
    off[i + 1] = off[i] + x.data.size();
  }
  float* dst = ctx.staging(std::max<size_t>(1, off.back()));
  if (off.back() == 0) dst[0] = 0.0f;
  const size_t nb = batch.size();
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  const size_t nth = off.back() * sizeof(float) < (8u << 20) ? 1 : std::min<size_t>({16, hw, nb});
  auto copy = [&](size_t w) {
    for (size_t i = w; i < nb; i += nth)
      if (!batch[i].data.empty()) std::memcpy(dst + off[i], batch[i].data.data(), batch[i].data.size() * sizeof(float));
  };
  if (nth <= 1) {
    copy(0);
  } else {
    std::vector<std::thread> th;
    th.reserve(nth - 1);
    for (size_t w = 1; w < nth; ++w) th.emplace_back(copy, w);
    copy(0);
    for (std::thread& t : th) t.join();
  }
  f.enc = dst;
  return f;
}

inline std::vector<std::vector<int32_t>> unpack(const std::vector<int32_t>& splits,
                                                const std::vector<int32_t>& toks) {
  std::vector<std::vector<int32_t>> out(splits.size() - 1);
  for (size_t i = 0; i + 1 < splits.size(); ++i)
    out[i].assign(toks.begin() + splits[i], toks.begin() + splits[i + 1]);
  return out;
}

}  // namespace detail

inline std::vector<std::vector<int32_t>> greedy_search_batch(
    Context& ctx, const ToyTransducer& m, const std::vector<Mat<float>>& batch,
    int32_t max_symbols = 1) {
  if (max_symbols != 1)
    throw ValidationError("greedy_search_batch supports max_symbols = 1 only");
  detail::Frames f = detail::encode(ctx, m, batch);
  const int32_t B = static_cast<int32_t>(batch.size());
  std::vector<int32_t> splits(B + 1), toks(std::max<int32_t>(1, f.splits.back()));
  check(rnntg_greedy_search_batch(ctx.handle(), f.enc, f.splits.data(), B, max_symbols,
                                  RNNTG_MEM_HOST_FEATURES, splits.data(), toks.data()));
  return detail::unpack(splits, toks);
}

// greedy_search (search.hpp:76-100) with the reference's signature, any S
// (kNoSymbolLimit = unlimited, 10 per frame at most), and its batched form.
inline std::vector<std::vector<int32_t>> greedy_search_batched(
    Context& ctx, const ToyTransducer& m, const std::vector<Mat<float>>& batch,
    int32_t max_symbols, int64_t* capped_frames = nullptr) {
  if (max_symbols < 1) throw ValidationError("max_symbols must be >= 1");
  detail::Frames f = detail::encode(ctx, m, batch);
  const int32_t B = static_cast<int32_t>(batch.size());
  const int64_t cap = max_symbols == kNoSymbolLimit ? kMaxSymbolsPerFrameSafety : max_symbols;
  std::vector<int32_t> splits(B + 1), toks(std::max<int64_t>(1, f.splits.back() * cap));
  int64_t capped = 0;
  check(rnntg_greedy_search(ctx.handle(), f.enc, f.splits.data(), B, max_symbols,
                            RNNTG_MEM_HOST_FEATURES, splits.data(), toks.data(), &capped));
  if (capped_frames) *capped_frames = capped;
  return detail::unpack(splits, toks);
}

inline std::vector<int32_t> greedy_search(Context& ctx, const ToyTransducer& m,
                                          const Mat<float>& features, int32_t max_symbols,
                                          int64_t* capped_frames = nullptr) {
  return greedy_search_batched(ctx, m, {features}, max_symbols, capped_frames)[0];
}

inline std::vector<std::vector<int32_t>> beam_search_batch(
    Context& ctx, const ToyTransducer& m, const std::vector<Mat<float>>& batch,
    const SearchParams& params, std::vector<double>* scores = nullptr) {
  if (params.max_symbols < 1) throw ValidationError("max_symbols must be >= 1");
  if (params.beam_size < 1) throw ValidationError("beam_size must be >= 1");
  detail::Frames f = detail::encode(ctx, m, batch);
  const int32_t B = static_cast<int32_t>(batch.size());
  rnntg_beam_params p{params.beam_size, params.max_symbols,
                      params.merge_op == MergeOp::kLogAdd ? RNNTG_MERGE_LOG_ADD : RNNTG_MERGE_MAX,
                      params.length_norm ? 1 : 0, params.max_total_symbols};
  const int64_t cap = params.max_symbols == kNoSymbolLimit ? kMaxSymbolsPerFrameSafety : params.max_symbols;
  std::vector<int32_t> splits(B + 1), toks(std::max<int64_t>(1, f.splits.back() * cap));
  std::vector<double> sc(std::max<int32_t>(1, B));
  check(rnntg_beam_search_batch(ctx.handle(), f.enc, f.splits.data(), B, &p,
                                RNNTG_MEM_HOST_FEATURES, splits.data(), toks.data(), sc.data()));
  if (scores) scores->assign(sc.begin(), sc.begin() + B);
  return detail::unpack(splits, toks);
}

inline std::vector<int32_t> beam_search(Context& ctx, const ToyTransducer& m,
                                        const Mat<float>& features,
                                        const SearchParams& params) {
  return beam_search_batch(ctx, m, {features}, params)[0];
}

// fsa_beam_search followed by lattice_to_best_seq(kMax) for every stream,
// with one graph shared by all streams (the CLI's usage, rnnt_main.cpp:297).
inline std::vector<std::vector<int32_t>> fsa_best_sequences(
    Context& ctx, const ToyTransducer& m, const std::vector<Mat<float>>& batch,
    const Fsa& graph, const FsaSearchParams& params,
    std::vector<double>* scores = nullptr) {
  rnntg_graph_t g = ctx.graph(graph);
  detail::Frames f = detail::encode(ctx, m, batch);
  const int32_t B = static_cast<int32_t>(batch.size());
  rnntg_fsa_params p{params.beam, params.max_states, params.max_contexts};
  std::vector<int32_t> splits(B + 1), toks(std::max<int32_t>(1, f.splits.back()));
  std::vector<double> sc(std::max<int32_t>(1, B));
  check(rnntg_fsa_beam_search(ctx.handle(), f.enc, f.splits.data(), B, g, &p,
                              RNNTG_MEM_HOST_FEATURES, splits.data(), toks.data(), sc.data()));
  if (scores) scores->assign(sc.begin(), sc.begin() + B);
  return detail::unpack(splits, toks);
}

// fsa_beam_search followed by lattice_to_best_seq(method, nbest_n, seed)
// for every stream (fsa_search.hpp:394-426; the CLI's decode with --merge,
// rnnt_main.cpp:302): kMax is the search's own best path, kLogAdd runs the
// n-best sampling / dedup / per-sequence totals on the GPU lattices.
inline std::vector<std::vector<int32_t>> fsa_best_sequences(
    Context& ctx, const ToyTransducer& m, const std::vector<Mat<float>>& batch,
    const Fsa& graph, const FsaSearchParams& params, MergeOp method, int32_t nbest_n = 100,
    uint64_t seed = 0) {
  if (method == MergeOp::kMax) return fsa_best_sequences(ctx, m, batch, graph, params);
  if (nbest_n < 1) throw ValidationError("nbest_n must be >= 1");
  fsa_best_sequences(ctx, m, batch, graph, params);
  const int32_t B = static_cast<int32_t>(batch.size());
  int64_t total = 0;
  for (const Mat<float>& x : batch) total += x.rows;
  std::vector<int32_t> splits(B + 1), toks(std::max<int64_t>(1, total));
  check(rnntg_fsa_lattice_best(ctx.handle(), RNNTG_MERGE_LOG_ADD, nbest_n, seed, splits.data(), toks.data(),
                               nullptr));
  return detail::unpack(splits, toks);
}

// fsa_beam_search (fsa_search.hpp:326-387) with the reference's signature
// and return type: one lattice per stream, node numbering and arc order as
// build_lattice + make_fsa produce them.  Streams sharing a graph (by
// content) are decoded in one device call.
inline std::vector<Fsa> fsa_beam_search(Context& ctx, const ToyTransducer& m,
                                        const std::vector<Mat<float>>& batch,
                                        const std::vector<Fsa>& graphs,
                                        const FsaSearchParams& params) {
  if (batch.size() != graphs.size())
    throw ValidationError("fsa_beam_search: |batch| != |graphs|");
  std::vector<Fsa> out(batch.size());
  std::vector<bool> done(batch.size(), false);
  for (size_t i = 0; i < batch.size(); ++i) {
    if (done[i]) continue;
    std::vector<size_t> idx;
    std::vector<Mat<float>> sub;
    for (size_t j = i; j < batch.size(); ++j)
      if (!done[j] && (j == i || graphs[j] == graphs[i])) {
        idx.push_back(j);
        sub.push_back(batch[j]);
        done[j] = true;
      }
    fsa_best_sequences(ctx, m, sub, graphs[i], params);
    for (size_t k = 0; k < idx.size(); ++k) {
      int32_t nn = 0, na = 0;
      check(rnntg_fsa_lattice(ctx.handle(), static_cast<int32_t>(k), &nn, &na, 0, nullptr, nullptr,
                              nullptr, nullptr));
      std::vector<int32_t> src(na), dst(na), lab(na);
      std::vector<double> sc(na);
      check(rnntg_fsa_lattice(ctx.handle(), static_cast<int32_t>(k), &nn, &na, na, src.data(),
                              dst.data(), lab.data(), sc.data()));
      std::vector<Arc> arcs(na);
      for (int32_t a = 0; a < na; ++a) arcs[a] = {src[a], dst[a], lab[a], sc[a]};
      out[idx[k]] = make_fsa(nn, std::move(arcs), {{nn - 1, 0.0}});
    }
  }
  return out;
}

// The Algorithm-1 step API (fsa_search.hpp:95-297) on the GPU, with the
// reference's types: construct = init_streams over one graph shared by all
// streams; get_contexts() as rnnt::get_contexts; expand_and_prune(logprobs)
// as expand_arcs + prune_streams (the caller's model output enters here,
// 59-61); finish() = finish_stream + build_lattice for every stream (equal
// to the reference's lattices), optionally with lattice_to_best_seq(kMax)
// and best_path scores.  num_frames[i] is the frames stream i consumes (the
// driver's DecodeStream::num_frames).  `graph` must outlive the object.
class FsaStreams {
 public:
  FsaStreams(Context& ctx, const Fsa& graph, const FsaSearchParams& p, const std::vector<int32_t>& num_frames)
      : ctx_(ctx), B_(static_cast<int32_t>(num_frames.size())), frames_(num_frames) {
    rnntg_fsa_params fp{p.beam, p.max_states, p.max_contexts};
    check(rnntg_fsa_stream_begin(ctx.handle(), ctx.graph(graph), &fp, B_, num_frames.data()));
  }
  std::pair<RaggedShape, Mat<int32_t>> get_contexts() {
    std::vector<int32_t> splits(B_ + 1);
    check(rnntg_fsa_stream_contexts(ctx_.handle(), splits.data(), 0, nullptr));
    std::vector<int32_t> packed(std::max(1, splits[B_]));
    check(rnntg_fsa_stream_contexts(ctx_.handle(), splits.data(), splits[B_], packed.data()));
    std::vector<int32_t> counts(B_);
    for (int32_t i = 0; i < B_; ++i) counts[i] = splits[i + 1] - splits[i];
    Mat<int32_t> ctx(splits[B_], 2);
    for (int32_t r = 0; r < splits[B_]; ++r) {
      auto [a, b] = unpack_context(packed[r], vocab());
      ctx.at(r, 0) = a;
      ctx.at(r, 1) = b;
    }
    rows_ = splits[B_];
    return {build_ragged(counts), std::move(ctx)};
  }
  void expand_and_prune(const Mat<double>& logprobs) {
    if (logprobs.rows != rows_) throw std::logic_error("expand_arcs: log-prob rows != context count");
    if (rows_ > 0 && logprobs.cols != vocab()) throw std::logic_error("expand_arcs: log-prob columns != vocab size");
    check(rnntg_fsa_stream_step(ctx_.handle(), logprobs.data.data(), RNNTG_MEM_HOST));
  }
  std::vector<Fsa> finish(std::vector<std::vector<int32_t>>* best = nullptr, std::vector<double>* scores = nullptr) {
    int64_t total = 0;
    for (int32_t n : frames_) total += n;
    std::vector<int32_t> splits(B_ + 1), toks(std::max<int64_t>(1, total));
    std::vector<double> sc(std::max(1, B_));
    check(rnntg_fsa_stream_end(ctx_.handle(), splits.data(), toks.data(), sc.data()));
    if (best) *best = detail::unpack(splits, toks);
    if (scores) scores->assign(sc.begin(), sc.begin() + B_);
    std::vector<Fsa> out(B_);
    for (int32_t k = 0; k < B_; ++k) {
      int32_t nn = 0, na = 0;
      check(rnntg_fsa_lattice(ctx_.handle(), k, &nn, &na, 0, nullptr, nullptr, nullptr, nullptr));
      std::vector<int32_t> src(na), dst(na), lab(na);
      std::vector<double> w(na);
      check(rnntg_fsa_lattice(ctx_.handle(), k, &nn, &na, na, src.data(), dst.data(), lab.data(), w.data()));
      std::vector<Arc> arcs(na);
      for (int32_t a = 0; a < na; ++a) arcs[a] = {src[a], dst[a], lab[a], w[a]};
      out[k] = make_fsa(nn, std::move(arcs), {{nn - 1, 0.0}});
    }
    return out;
  }

 private:
  int32_t vocab() const { return ctx_.vocab_size(); }
  Context& ctx_;
  int32_t B_;
  std::vector<int32_t> frames_;
  int32_t rows_ = 0;
};

}  // namespace gpu
}  // namespace rnnt

#endif  // RNNT_GPU_HPP_
