// C-ABI wrapper around the UNMODIFIED reference headers (rnnt-kit), compiled
// from /root/reference/proj/include by oracle/Makefile into
// oracle/_ref/librnnt_ref.so.  TEST INFRASTRUCTURE ONLY: used by tests/ as the
// parity checker and by bench.py's cpu_baseline / --impl reference leg as the
// timed CPU reference.  Nothing in the product path links or loads it.
//
// Every entry point calls the reference's own public API:
//   init_model / encoder_forward           model.hpp:129-169, 224-238
//   greedy_search_batch                    search.hpp:107-167
//   beam_search                            search.hpp:206-277
//   fsa_beam_search + lattice_to_best_seq  fsa_search.hpp:326-426
//   best_path                              fsa.hpp:345-376
//   trivial_graph / ngram_graph_from_arpa  fsa.hpp:266-273, arpa.hpp:170-288
//   parse/serialize_fsa_text               fsa.hpp:140-262
// Thread fan-out mirrors the reference CLI's parallel_for
// (tools/rnnt_main.cpp:131-158): an atomic index over independent streams.
#include <atomic>
#include <cstdint>
#include <cstring>
#include <exception>
#include <map>
#include <string>
#include <thread>
#include <vector>

#include "rnnt/arpa.hpp"
#include "rnnt/common.hpp"
#include "rnnt/fsa.hpp"
#include "rnnt/fsa_search.hpp"
#include "rnnt/model.hpp"
#include "rnnt/ragged.hpp"
#include "rnnt/search.hpp"

namespace {

thread_local std::string g_err;

int fail(const std::exception& e) {
  g_err = e.what();
  if (dynamic_cast<const rnnt::ValidationError*>(&e)) return 1;
  if (dynamic_cast<const rnnt::ParseError*>(&e)) return 3;
  return 2;
}

template <typename F>
void parallel_for(int64_t n, int threads, F&& fn) {
  if (threads <= 1 || n <= 1) {
    for (int64_t i = 0; i < n; ++i) fn(i);
    return;
  }
  std::atomic<int64_t> next{0};
  std::vector<std::thread> pool;
  std::exception_ptr first;
  std::atomic<bool> failed{false};
  for (int t = 0; t < threads; ++t)
    pool.emplace_back([&] {
      while (!failed.load()) {
        int64_t i = next.fetch_add(1);
        if (i >= n) break;
        try {
          fn(i);
        } catch (...) {
          if (!failed.exchange(true)) first = std::current_exception();
        }
      }
    });
  for (auto& t : pool) t.join();
  if (first) std::rethrow_exception(first);
}

std::vector<rnnt::Mat<float>> split_frames(const float* data,
                                           const int32_t* splits, int32_t B,
                                           int32_t dim) {
  std::vector<rnnt::Mat<float>> out(B);
  for (int32_t i = 0; i < B; ++i) {
    int32_t T = splits[i + 1] - splits[i];
    out[i] = rnnt::Mat<float>(T, dim);
    std::memcpy(out[i].data.data(), data + static_cast<size_t>(splits[i]) * dim,
                sizeof(float) * static_cast<size_t>(T) * dim);
  }
  return out;
}

void write_ragged(const std::vector<std::vector<int32_t>>& ys,
                  int32_t* out_splits, int32_t* out_tokens) {
  out_splits[0] = 0;
  for (size_t i = 0; i < ys.size(); ++i) {
    std::memcpy(out_tokens + out_splits[i], ys[i].data(),
                sizeof(int32_t) * ys[i].size());
    out_splits[i + 1] = out_splits[i] + static_cast<int32_t>(ys[i].size());
  }
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

void* ref_model_new(int32_t V, int32_t feat_dim, int32_t enc_dim,
                    int32_t emb_dim, int32_t joiner_dim, uint64_t seed,
                    double blank_bias) {
  try {
    rnnt::ModelConfig cfg;
    cfg.vocab_size = V;
    cfg.feat_dim = feat_dim;
    cfg.enc_dim = enc_dim;
    cfg.emb_dim = emb_dim;
    cfg.joiner_dim = joiner_dim;
    cfg.seed = seed;
    auto* m = new rnnt::ToyTransducer(rnnt::init_model(cfg));
    m->out_b.at(0, 0) += static_cast<float>(blank_bias);
    return m;
  } catch (const std::exception& e) {
    fail(e);
    return nullptr;
  }
}

void ref_model_free(void* m) { delete static_cast<rnnt::ToyTransducer*>(m); }

// Pointer to the named parameter (param_views naming, model.hpp:75-82).
float* ref_model_param(void* mp, const char* name, int32_t* rows,
                       int32_t* cols) {
  auto* m = static_cast<rnnt::ToyTransducer*>(mp);
  for (auto& [n, mat] : m->param_views())
    if (n == name) {
      *rows = mat->rows;
      *cols = mat->cols;
      return mat->data.data();
    }
  return nullptr;
}

// Features ~ N(0,1) from DetRng(seed).gaussian() (common.hpp:108-121).
void ref_features(uint64_t seed, int32_t T, int32_t feat_dim, float* out) {
  rnnt::DetRng rng(seed);
  for (int64_t i = 0; i < static_cast<int64_t>(T) * feat_dim; ++i)
    out[i] = static_cast<float>(rng.gaussian());
}

int ref_encoder_forward(void* mp, const float* feats, int32_t T,
                        float* out) {
  try {
    auto* m = static_cast<rnnt::ToyTransducer*>(mp);
    rnnt::Mat<float> f(T, m->cfg.feat_dim);
    std::memcpy(f.data.data(), feats, sizeof(float) * f.data.size());
    rnnt::Mat<float> enc = rnnt::encoder_forward(*m, f);
    std::memcpy(out, enc.data.data(), sizeof(float) * enc.data.size());
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int ref_encoder_forward_batch(void* mp, const float* feats,
                              const int32_t* splits, int32_t B, int threads,
                              float* out) {
  try {
    auto* m = static_cast<rnnt::ToyTransducer*>(mp);
    const int32_t F = m->cfg.feat_dim, D = m->cfg.enc_dim;
    parallel_for(B, threads, [&](int64_t i) {
      int32_t T = splits[i + 1] - splits[i];
      rnnt::Mat<float> f(T, F);
      std::memcpy(f.data.data(), feats + static_cast<size_t>(splits[i]) * F,
                  sizeof(float) * f.data.size());
      rnnt::Mat<float> enc = rnnt::encoder_forward(*m, f);
      std::memcpy(out + static_cast<size_t>(splits[i]) * D, enc.data.data(),
                  sizeof(float) * enc.data.size());
    });
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// Reference joiner pieces, for kernel-level bit checks.
int ref_decoder_project(void* mp, const int32_t* ctxs, int32_t n, float* pd) {
  try {
    auto* m = static_cast<rnnt::ToyTransducer*>(mp);
    std::vector<int32_t> c(ctxs, ctxs + n);
    rnnt::Mat<float> dec = rnnt::decoder_forward(*m, c);
    for (int32_t i = 0; i < n; ++i)
      rnnt::joiner_project_dec(*m, dec.row(i),
                               pd + static_cast<size_t>(i) * m->cfg.joiner_dim);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int ref_joiner_logits(void* mp, const float* enc_rows, const int32_t* ctxs,
                      int32_t n, float* logits) {
  try {
    auto* m = static_cast<rnnt::ToyTransducer*>(mp);
    const int32_t D = m->cfg.enc_dim, V = m->cfg.vocab_size;
    for (int32_t i = 0; i < n; ++i) {
      rnnt::Mat<float> dec = rnnt::decoder_forward(*m, {ctxs[i]});
      rnnt::joiner_logits(*m, enc_rows + static_cast<size_t>(i) * D, dec.row(0),
                          logits + static_cast<size_t>(i) * V);
    }
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int ref_log_softmax(const float* logits, int32_t n, double* out) {
  rnnt::detail::log_softmax_row(logits, n, out);
  return 0;
}

// greedy_search_batch over `threads` contiguous shards (batching transparency,
// search_test.cpp:169-187, makes the shard split invisible in the results).
int ref_greedy_search_batch(void* mp, const float* feats,
                            const int32_t* splits, int32_t B, int32_t max_sym,
                            int threads, int32_t* out_splits,
                            int32_t* out_tokens) {
  try {
    auto* m = static_cast<rnnt::ToyTransducer*>(mp);
    auto batch = split_frames(feats, splits, B, m->cfg.feat_dim);
    std::vector<std::vector<int32_t>> ys(B);
    int nshard = std::max(1, std::min<int>(threads, B));
    parallel_for(nshard, nshard, [&](int64_t s) {
      int64_t lo = B * s / nshard, hi = B * (s + 1) / nshard;
      std::vector<rnnt::Mat<float>> part(batch.begin() + lo, batch.begin() + hi);
      auto got = rnnt::greedy_search_batch(*m, part, max_sym);
      for (int64_t i = lo; i < hi; ++i) ys[i] = std::move(got[i - lo]);
    });
    write_ragged(ys, out_splits, out_tokens);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// greedy_search (search.hpp:76-100, any S) per utterance under parallel_for;
// capped_frames summed over utterances.
int ref_greedy_search(void* mp, const float* feats, const int32_t* splits, int32_t B,
                      int32_t max_symbols, int threads, int32_t* out_splits,
                      int32_t* out_tokens, int64_t* capped_frames) {
  try {
    auto* m = static_cast<rnnt::ToyTransducer*>(mp);
    auto batch = split_frames(feats, splits, B, m->cfg.feat_dim);
    std::vector<std::vector<int32_t>> ys(B);
    std::vector<int64_t> capped(B, 0);
    parallel_for(B, std::max(1, threads), [&](int64_t i) {
      ys[i] = rnnt::greedy_search(*m, batch[i], max_symbols, &capped[i]);
    });
    write_ragged(ys, out_splits, out_tokens);
    if (capped_frames) {
      *capped_frames = 0;
      for (int64_t c : capped) *capped_frames += c;
    }
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// beam_search per utterance under parallel_for (rnnt_main.cpp:274-287).
int ref_beam_search_batch(void* mp, const float* feats, const int32_t* splits,
                          int32_t B, int32_t beam_size, int32_t max_symbols,
                          int32_t merge_op, int32_t length_norm,
                          int32_t max_total_symbols, int threads,
                          int32_t* out_splits, int32_t* out_tokens) {
  try {
    auto* m = static_cast<rnnt::ToyTransducer*>(mp);
    auto batch = split_frames(feats, splits, B, m->cfg.feat_dim);
    rnnt::SearchParams p;
    p.beam_size = beam_size;
    p.max_symbols = max_symbols;
    p.merge_op = merge_op ? rnnt::MergeOp::kLogAdd : rnnt::MergeOp::kMax;
    p.length_norm = length_norm != 0;
    p.max_total_symbols = max_total_symbols;
    std::vector<std::vector<int32_t>> ys(B);
    parallel_for(B, threads,
                 [&](int64_t i) { ys[i] = rnnt::beam_search(*m, batch[i], p); });
    write_ragged(ys, out_splits, out_tokens);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// ---- graphs ----

void* ref_graph_trivial(int32_t V) {
  try {
    return new rnnt::Fsa(rnnt::trivial_graph(V));
  } catch (const std::exception& e) {
    fail(e);
    return nullptr;
  }
}

// ARPA words "w<k>" map to token k (1..V-1).
void* ref_graph_from_arpa(const char* text, int32_t V) {
  try {
    std::map<std::string, int32_t> tm;
    for (int32_t k = 1; k < V; ++k) tm["w" + std::to_string(k)] = k;
    return new rnnt::Fsa(rnnt::ngram_graph_from_arpa(text, tm));
  } catch (const std::exception& e) {
    fail(e);
    return nullptr;
  }
}

void* ref_graph_from_text(const char* text) {
  try {
    return new rnnt::Fsa(rnnt::parse_fsa_text(text));
  } catch (const std::exception& e) {
    fail(e);
    return nullptr;
  }
}

// arcs = (src,dst,label,score) in CSR order; finals listed separately.
void* ref_graph_from_arcs(int32_t num_states, int32_t num_arcs,
                          const int32_t* src, const int32_t* dst,
                          const int32_t* label, const double* score,
                          int32_t num_finals, const int32_t* final_states,
                          const double* final_scores) {
  try {
    std::vector<rnnt::Arc> arcs(num_arcs);
    for (int32_t i = 0; i < num_arcs; ++i)
      arcs[i] = {src[i], dst[i], label[i], score[i]};
    std::map<rnnt::StateId, double> finals;
    for (int32_t i = 0; i < num_finals; ++i)
      finals[final_states[i]] = final_scores[i];
    return new rnnt::Fsa(rnnt::make_fsa(num_states, std::move(arcs), finals));
  } catch (const std::exception& e) {
    fail(e);
    return nullptr;
  }
}

void ref_graph_free(void* g) { delete static_cast<rnnt::Fsa*>(g); }

void ref_graph_sizes(void* gp, int32_t* num_states, int32_t* num_arcs,
                     int32_t* num_finals) {
  auto* g = static_cast<rnnt::Fsa*>(gp);
  *num_states = g->num_states;
  *num_arcs = static_cast<int32_t>(g->arcs.size());
  *num_finals = static_cast<int32_t>(g->finals.size());
}

void ref_graph_export(void* gp, int32_t* arc_splits, int32_t* src,
                      int32_t* dst, int32_t* label, double* score,
                      int32_t* final_states, double* final_scores) {
  auto* g = static_cast<rnnt::Fsa*>(gp);
  for (size_t i = 0; i < g->arc_splits.size(); ++i)
    arc_splits[i] = g->arc_splits[i];
  for (size_t i = 0; i < g->arcs.size(); ++i) {
    src[i] = g->arcs[i].src;
    dst[i] = g->arcs[i].dst;
    label[i] = g->arcs[i].label;
    score[i] = g->arcs[i].score;
  }
  int32_t k = 0;
  for (auto& [s, w] : g->finals) {
    final_states[k] = s;
    final_scores[k] = w;
    ++k;
  }
}

// Caller frees with ref_free_string.
char* ref_graph_text(void* gp) {
  std::string s = rnnt::serialize_fsa_text(*static_cast<rnnt::Fsa*>(gp));
  return strdup(s.c_str());
}

void ref_free_string(char* s) { free(s); }

// ---- FSA beam search ----
//
// fsa_beam_search over `threads` shards; each shard decodes its streams one
// at a time with a single graph copy (batching transparency,
// fsa_search_test.cpp:364-393).  Per stream: lattice_to_best_seq(kMax) tokens
// and best_path(...).score (or -inf for an empty lattice).  If lattice_texts
// is non-null, each entry receives serialize_fsa_text(lattice) (free with
// ref_free_string).
int ref_fsa_beam_search(void* mp, const float* feats, const int32_t* splits,
                        int32_t B, void* gp, double beam, int32_t max_states,
                        int32_t max_contexts, int threads, int32_t* out_splits,
                        int32_t* out_tokens, double* out_scores,
                        char** lattice_texts) {
  try {
    auto* m = static_cast<rnnt::ToyTransducer*>(mp);
    const rnnt::Fsa& g = *static_cast<rnnt::Fsa*>(gp);
    auto batch = split_frames(feats, splits, B, m->cfg.feat_dim);
    rnnt::FsaSearchParams p;
    p.beam = beam;
    p.max_states = max_states;
    p.max_contexts = max_contexts;
    std::vector<std::vector<int32_t>> ys(B);
    int nshard = std::max(1, std::min<int>(threads, B));
    parallel_for(nshard, nshard, [&](int64_t s) {
      std::vector<rnnt::Fsa> one{g};
      int64_t lo = B * s / nshard, hi = B * (s + 1) / nshard;
      for (int64_t i = lo; i < hi; ++i) {
        auto lats = rnnt::fsa_beam_search(*m, {batch[i]}, one, p);
        ys[i] = rnnt::lattice_to_best_seq(lats[0], rnnt::MergeOp::kMax);
        double sc = rnnt::kNegInf;
        try {
          sc = rnnt::best_path(lats[0]).score;
        } catch (const rnnt::ValidationError&) {
        }
        out_scores[i] = sc;
        if (lattice_texts)
          lattice_texts[i] = strdup(rnnt::serialize_fsa_text(lats[0]).c_str());
      }
    });
    write_ragged(ys, out_splits, out_tokens);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// fsa_beam_search + lattice_to_best_seq(kLogAdd, nbest_n, seed) per stream
// (the CLI's `--merge log_add` decode, rnnt_main.cpp:302), sharded like
// ref_fsa_beam_search.  out_logprob[i] = sequence_total_logprob(lattice,
// seq) of the returned sequence (-inf for an empty lattice).
int ref_fsa_logadd(void* mp, const float* feats, const int32_t* splits, int32_t B, void* gp,
                   double beam, int32_t max_states, int32_t max_contexts, int threads,
                   int32_t nbest_n, uint64_t seed, int32_t* out_splits, int32_t* out_tokens,
                   double* out_logprob) {
  try {
    auto* m = static_cast<rnnt::ToyTransducer*>(mp);
    const rnnt::Fsa& g = *static_cast<rnnt::Fsa*>(gp);
    auto batch = split_frames(feats, splits, B, m->cfg.feat_dim);
    rnnt::FsaSearchParams p;
    p.beam = beam;
    p.max_states = max_states;
    p.max_contexts = max_contexts;
    std::vector<std::vector<int32_t>> ys(B);
    int nshard = std::max(1, std::min<int>(threads, B));
    parallel_for(nshard, nshard, [&](int64_t s) {
      std::vector<rnnt::Fsa> one{g};
      int64_t lo = B * s / nshard, hi = B * (s + 1) / nshard;
      for (int64_t i = lo; i < hi; ++i) {
        auto lats = rnnt::fsa_beam_search(*m, {batch[i]}, one, p);
        ys[i] = rnnt::lattice_to_best_seq(lats[0], rnnt::MergeOp::kLogAdd, nbest_n, seed);
        double lp = rnnt::kNegInf;
        if (rnnt::total_logprob(lats[0]) != rnnt::kNegInf) lp = rnnt::sequence_total_logprob(lats[0], ys[i]);
        out_logprob[i] = lp;
      }
    });
    write_ragged(ys, out_splits, out_tokens);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// ---- the Algorithm-1 step API (fsa_search.hpp:95-297), driven like the
// reference's fsa_beam_search (326-387): num_frames per stream, streams
// finished (finish_stream) when they reach it; for the GPU step-API tests.
struct RefSteps {
  std::vector<rnnt::Fsa> graphs;  // DecodeStream::graph points in here
  std::vector<rnnt::DecodeStream> streams;
  rnnt::RaggedShape shape;
};

void* ref_steps_begin(void* gp, int32_t B, double beam, int32_t max_states, int32_t max_contexts, int32_t V,
                      const int32_t* num_frames) {
  try {
    auto* r = new RefSteps();
    r->graphs.assign(B, *static_cast<rnnt::Fsa*>(gp));
    rnnt::FsaSearchParams p;
    p.beam = beam;
    p.max_states = max_states;
    p.max_contexts = max_contexts;
    r->streams = rnnt::init_streams(r->graphs, p, V);
    for (int32_t i = 0; i < B; ++i) {
      r->streams[i].num_frames = num_frames[i];
      if (num_frames[i] == 0) rnnt::detail::finish_stream(r->streams[i]);
    }
    return r;
  } catch (const std::exception& e) {
    fail(e);
    return nullptr;
  }
}

// get_contexts: row splits [B+1] and packed contexts a*V+b.
int ref_steps_contexts(void* hp, int32_t* out_row_splits, int32_t* out_ctx) {
  try {
    auto* r = static_cast<RefSteps*>(hp);
    auto [shape, ctx] = rnnt::get_contexts(r->streams);
    r->shape = shape;
    for (size_t i = 0; i < shape.row_splits.size(); ++i) out_row_splits[i] = shape.row_splits[i];
    const int32_t V = r->streams.empty() ? 2 : r->streams[0].vocab_size;
    for (int32_t k = 0; k < ctx.rows; ++k) out_ctx[k] = ctx.at(k, 0) * V + ctx.at(k, 1);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// expand_arcs + prune_streams with the caller's rows, then finish_stream
// for the streams that reached their last frame.
int ref_steps_step(void* hp, const double* logprobs, int32_t rows, int32_t V) {
  try {
    auto* r = static_cast<RefSteps*>(hp);
    rnnt::Mat<double> lp(rows, V);
    for (int32_t k = 0; k < rows * V; ++k) lp.data[k] = logprobs[k];
    rnnt::expand_arcs(r->streams, r->shape, lp);
    rnnt::prune_streams(r->streams);
    for (rnnt::DecodeStream& s : r->streams)
      if (!s.done && s.t == s.num_frames) rnnt::detail::finish_stream(s);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// Per stream: serialize_fsa_text of its lattice, lattice_to_best_seq(kMax)
// tokens and best_path score (-inf without a complete path).
int ref_steps_end(void* hp, char** texts, int32_t* out_splits, int32_t* out_tokens, double* out_scores) {
  try {
    auto* r = static_cast<RefSteps*>(hp);
    std::vector<std::vector<int32_t>> ys;
    for (size_t i = 0; i < r->streams.size(); ++i) {
      rnnt::Fsa lat = rnnt::detail::build_lattice(r->streams[i]);
      texts[i] = strdup(rnnt::serialize_fsa_text(lat).c_str());
      ys.push_back(rnnt::lattice_to_best_seq(lat, rnnt::MergeOp::kMax));
      double sc = rnnt::kNegInf;
      try {
        sc = rnnt::best_path(lat).score;
      } catch (const rnnt::ValidationError&) {
      }
      out_scores[i] = sc;
    }
    write_ragged(ys, out_splits, out_tokens);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

void ref_steps_free(void* hp) { delete static_cast<RefSteps*>(hp); }

}  // extern "C"
