// CPU restatement of the reference decoding path.  TEST INFRASTRUCTURE ONLY
// (see rnnt_oracle.h).  Built by oracle/Makefile with the reference's own
// flags (-O3 -DNDEBUG, no -march, -ffp-contract=off) so the float
// arithmetic is the same scalar mul/add sequence as the reference build.
#include "rnnt_oracle.h"

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <exception>
#include <limits>
#include <stdexcept>
#include <string>
#include <thread>
#include <unordered_map>
#include <utility>
#include <vector>

namespace {

constexpr double kNegInf = -std::numeric_limits<double>::infinity();
thread_local std::string g_err;

// Spread independent streams over threads (the reference CLI's parallel_for,
// tools/rnnt_main.cpp:131-158).
template <typename F>
void for_streams(int32_t n, int threads, F&& fn) {
  if (threads <= 1 || n <= 1) {
    for (int32_t i = 0; i < n; ++i) fn(i);
    return;
  }
  std::atomic<int32_t> next{0};
  std::vector<std::thread> pool;
  for (int t = 0; t < threads; ++t)
    pool.emplace_back([&] {
      for (int32_t i; (i = next.fetch_add(1)) < n;) fn(i);
    });
  for (auto& th : pool) th.join();
}

// log_add, common.hpp:48-54.
double log_add(double a, double b) {
  if (a == kNegInf) return b;
  if (b == kNegInf) return a;
  double hi = a > b ? a : b, lo = a > b ? b : a;
  return hi + std::log1p(std::exp(lo - hi));
}

// Per-model cache of decoder-side joiner projections.  A pure function of
// the packed context (model.hpp:240; search.hpp:126-141), so caching never
// changes values.
class PdCache {
 public:
  explicit PdCache(const orc_model* m) : m_(m) {}
  const float* get(int32_t ctx) {
    auto it = map_.find(ctx);
    if (it != map_.end()) return it->second.data();
    std::vector<float> pd(m_->J);
    orc_decoder_project(m_, &ctx, 1, pd.data());
    return map_.emplace(ctx, std::move(pd)).first->second.data();
  }

 private:
  const orc_model* m_;
  std::unordered_map<int32_t, std::vector<float>> map_;
};

// Argmax with the first maximum winning (search.hpp:59-66).
int32_t first_argmax(const float* x, int32_t n) {
  int32_t best = 0;
  for (int32_t i = 1; i < n; ++i)
    if (x[i] > x[best]) best = i;
  return best;
}

}  // namespace

extern "C" {

const char* orc_last_error(void) { return g_err.c_str(); }

float orc_tanhf(float x) { return std::tanh(x); }

// detail::affine / joiner_project_*: model.hpp:100-108, 263-281.  The
// accumulator starts at the bias (or 0.0f) and adds w*x in index order.
void orc_affine(const float* w, const float* bias, const float* x, int32_t M,
                int32_t N, int32_t K, float* y) {
  for (int32_t m = 0; m < M; ++m) {
    const float* xr = x + static_cast<size_t>(m) * K;
    for (int32_t n = 0; n < N; ++n) {
      const float* wr = w + static_cast<size_t>(n) * K;
      float acc = bias ? bias[n] : 0.0f;
      for (int32_t k = 0; k < K; ++k) acc += wr[k] * xr[k];
      y[static_cast<size_t>(m) * N + n] = acc;
    }
  }
}

// encoder_forward, model.hpp:224-238: two affine+tanh layers per frame.
void orc_encoder(const float* w1, const float* b1, const float* w2,
                 const float* b2, int32_t F, int32_t D, const float* feats,
                 int32_t T, float* enc) {
  std::vector<float> h(D);
  for (int32_t t = 0; t < T; ++t) {
    orc_affine(w1, b1, feats + static_cast<size_t>(t) * F, 1, D, F, h.data());
    for (float& v : h) v = std::tanh(v);
    float* o = enc + static_cast<size_t>(t) * D;
    orc_affine(w2, b2, h.data(), 1, D, D, o);
    for (int32_t i = 0; i < D; ++i) o[i] = std::tanh(o[i]);
  }
}

// decoder_forward (model.hpp:241-259) then joiner_project_dec (273-281):
// pd = j_wd . tanh(ctx_b + ctx_w . [emb[a] ; emb[b]]), context = a*V + b.
void orc_decoder_project(const orc_model* m, const int32_t* ctxs, int32_t n,
                         float* pd) {
  const int32_t E = m->E;
  std::vector<float> cat(2 * E), dec(E);
  for (int32_t i = 0; i < n; ++i) {
    const int32_t a = ctxs[i] / m->V, b = ctxs[i] % m->V;
    std::memcpy(cat.data(), m->emb + static_cast<size_t>(a) * E,
                sizeof(float) * E);
    std::memcpy(cat.data() + E, m->emb + static_cast<size_t>(b) * E,
                sizeof(float) * E);
    orc_affine(m->ctx_w, m->ctx_b, cat.data(), 1, E, 2 * E, dec.data());
    for (float& v : dec) v = std::tanh(v);
    orc_affine(m->j_wd, nullptr, dec.data(), 1, m->J, E,
               pd + static_cast<size_t>(i) * m->J);
  }
}

// joiner_logits_from_proj, model.hpp:284-292:
// h = tanh((pe + pd) + j_b); logits = out_b + out_w . h.
void orc_joiner_logits_from_proj(const orc_model* m, const float* pe,
                                 const float* pd, float* logits) {
  std::vector<float> h(m->J);
  for (int32_t i = 0; i < m->J; ++i) h[i] = std::tanh(pe[i] + pd[i] + m->j_b[i]);
  orc_affine(m->out_w, m->out_b, h.data(), 1, m->V, m->J, logits);
}

// detail::log_softmax_row, model.hpp:115-125: float max, double sum of
// exp(double(l) - max) in index order, lp = double(l) - (max + log(sum)).
void orc_log_softmax(const float* logits, int32_t n, double* out) {
  float mx = logits[0];
  for (int32_t i = 1; i < n; ++i) mx = std::max(mx, logits[i]);
  double sum = 0.0;
  for (int32_t i = 0; i < n; ++i)
    sum += std::exp(static_cast<double>(logits[i]) - mx);
  const double lse = static_cast<double>(mx) + std::log(sum);
  for (int32_t i = 0; i < n; ++i) out[i] = static_cast<double>(logits[i]) - lse;
}

// greedy_search_batch with S = 1, search.hpp:107-167.  Per frame the stream's
// context comes from its last two tokens, the joiner row decides by the
// first-max argmax of the raw float logits, and non-blank winners append.
int orc_greedy_batch(const orc_model* m, const float* enc,
                     const int32_t* frame_splits, int32_t B, int threads,
                     int32_t* out_splits, int32_t* out_tokens) {
  std::vector<std::vector<int32_t>> ys(B);
  for_streams(B, threads, [&](int32_t s) {
    PdCache cache(m);
    std::vector<float> pe(m->J), logits(m->V);
    for (int32_t t = frame_splits[s]; t < frame_splits[s + 1]; ++t) {
      orc_affine(m->j_we, nullptr, enc + static_cast<size_t>(t) * m->D, 1,
                 m->J, m->D, pe.data());
      const std::vector<int32_t>& y = ys[s];
      const size_t L = y.size();
      const int32_t ctx = (L >= 2 ? y[L - 2] : 0) * m->V + (L >= 1 ? y[L - 1] : 0);
      orc_joiner_logits_from_proj(m, pe.data(), cache.get(ctx), logits.data());
      const int32_t k = first_argmax(logits.data(), m->V);
      if (k != 0) ys[s].push_back(k);
    }
  });
  out_splits[0] = 0;
  for (int32_t s = 0; s < B; ++s) {
    std::copy(ys[s].begin(), ys[s].end(), out_tokens + out_splits[s]);
    out_splits[s + 1] = out_splits[s] + static_cast<int32_t>(ys[s].size());
  }
  return 0;
}

}  // extern "C"

namespace {

struct Hyp {
  std::vector<int32_t> ys;
  double score;
};

// detail::hyp_better, search.hpp:172-178: score desc, then shorter, then
// lexicographically smaller.
bool hyp_before(const std::vector<int32_t>& ya, double sa,
                const std::vector<int32_t>& yb, double sb) {
  if (sa != sb) return sa > sb;
  if (ya.size() != yb.size()) return ya.size() < yb.size();
  return ya < yb;
}

// One stream of beam_search at max_symbols = 1 (search.hpp:206-277).  Per
// frame: every hypothesis contributes its blank continuation to the frame
// set and its V-1 extensions to the level set; the level set is cut to the
// beam (prune_to_beam, 189-198), merged into the frame set by full-sequence
// equality (merge_into, 180-187), and the frame set is cut to the beam.
std::pair<std::vector<int32_t>, double> beam_one(const orc_model* m,
                                                 const float* enc, int32_t T,
                                                 int32_t beam, bool log_merge,
                                                 bool length_norm,
                                                 int32_t max_total) {
  const int32_t V = m->V;
  PdCache cache(m);
  std::vector<Hyp> hyps{{{}, 0.0}};
  std::vector<float> pe(m->J), logits(V);
  std::vector<double> lp(V);

  auto merge = [&](std::vector<Hyp>& set, const std::vector<int32_t>& ys,
                   double sc) {
    for (Hyp& h : set)
      if (h.ys == ys) {
        h.score = log_merge ? log_add(h.score, sc) : std::max(h.score, sc);
        return;
      }
    set.push_back({ys, sc});
  };
  auto cut = [&](std::vector<Hyp>& set) {
    if (static_cast<int32_t>(set.size()) <= beam) return;
    std::sort(set.begin(), set.end(), [](const Hyp& a, const Hyp& b) {
      return hyp_before(a.ys, a.score, b.ys, b.score);
    });
    set.resize(beam);
  };

  struct Ext {
    int32_t hyp, tok;
    double score;
  };
  for (int32_t t = 0; t < T; ++t) {
    orc_affine(m->j_we, nullptr, enc + static_cast<size_t>(t) * m->D, 1, m->J,
               m->D, pe.data());
    std::vector<Hyp> frame;
    std::vector<Ext> ext;
    for (int32_t h = 0; h < static_cast<int32_t>(hyps.size()); ++h) {
      const std::vector<int32_t>& y = hyps[h].ys;
      const size_t L = y.size();
      const int32_t ctx = (L >= 2 ? y[L - 2] : 0) * V + (L >= 1 ? y[L - 1] : 0);
      orc_joiner_logits_from_proj(m, pe.data(), cache.get(ctx), logits.data());
      orc_log_softmax(logits.data(), V, lp.data());
      merge(frame, y, hyps[h].score + lp[0]);
      if (max_total > 0 && static_cast<int32_t>(L) >= max_total) continue;
      for (int32_t k = 1; k < V; ++k) ext.push_back({h, k, hyps[h].score + lp[k]});
    }
    // Extensions are pairwise distinct sequences (distinct parents or
    // distinct last tokens), so stage one is a plain top-beam cut.
    auto ext_before = [&](const Ext& a, const Ext& b) {
      if (a.score != b.score) return a.score > b.score;
      if (a.hyp == b.hyp) return a.tok < b.tok;  // same length, same prefix
      const auto& ya = hyps[a.hyp].ys;
      const auto& yb = hyps[b.hyp].ys;
      if (ya.size() != yb.size()) return ya.size() < yb.size();
      return ya < yb;
    };
    if (static_cast<int32_t>(ext.size()) > beam) {
      std::partial_sort(ext.begin(), ext.begin() + beam, ext.end(), ext_before);
      ext.resize(beam);
    }
    for (const Ext& e : ext) {
      std::vector<int32_t> y = hyps[e.hyp].ys;
      y.push_back(e.tok);
      merge(frame, y, e.score);
    }
    cut(frame);
    hyps = std::move(frame);
  }

  // Final choice, search.hpp:261-276.
  size_t best = 0;
  auto key = [&](const Hyp& h) {
    return length_norm ? h.score / std::max<size_t>(1, h.ys.size()) : h.score;
  };
  for (size_t i = 1; i < hyps.size(); ++i)
    if (hyp_before(hyps[i].ys, key(hyps[i]), hyps[best].ys, key(hyps[best])))
      best = i;
  return {hyps[best].ys, hyps[best].score};
}

// ---------------- FSA search (fsa_search.hpp) ----------------

struct Tuple {   // StreamState, fsa_search.hpp:41-46
  int32_t ctx, state;
  double score;
  int32_t node;
};
struct Piece {   // LatticePiece, fsa_search.hpp:50-55
  int32_t src, dst, label;
  double score;
};
struct Key {
  int32_t ctx, state;
  bool operator<(const Key& o) const {
    return ctx != o.ctx ? ctx < o.ctx : state < o.state;
  }
  bool operator==(const Key& o) const { return ctx == o.ctx && state == o.state; }
};

struct FsaResult {
  std::vector<int32_t> ys;
  double score;
  std::vector<Piece> arcs;  // make_fsa order, super-final hops included
  int32_t num_nodes;        // including super-final
};

// best_path, fsa.hpp:345-376, on a lattice whose node ids are already a
// topological order (nodes are numbered frame by frame,
// fsa_search.hpp:280-282): backward tropical suffix maxima, then a forward
// trace that stops at the final node when possible and otherwise takes the
// first arc (CSR order) that attains the remaining suffix score.
void lattice_best(FsaResult& r, int32_t super) {
  const int32_t N = r.num_nodes;
  std::vector<int32_t> split(N + 1, 0);
  for (const Piece& p : r.arcs) split[p.src + 1]++;
  for (int32_t i = 0; i < N; ++i) split[i + 1] += split[i];
  std::vector<double> best(N, kNegInf);
  for (int32_t s = N - 1; s >= 0; --s) {
    double b = s == super ? 0.0 : kNegInf;
    for (int32_t a = split[s]; a < split[s + 1]; ++a)
      b = std::max(b, r.arcs[a].score + best[r.arcs[a].dst]);
    best[s] = b;
  }
  r.ys.clear();
  if (best[0] == kNegInf) {
    r.score = kNegInf;
    return;
  }
  int32_t s = 0;
  double remaining = best[0], total = 0.0;
  while (true) {
    if (s == super && remaining == 0.0) {
      total += 0.0;
      break;
    }
    int32_t chosen = -1;
    for (int32_t a = split[s]; a < split[s + 1]; ++a)
      if (r.arcs[a].score + best[r.arcs[a].dst] == remaining) {
        chosen = a;
        break;
      }
    if (chosen < 0) throw std::logic_error("lattice trace failed");
    const Piece& p = r.arcs[chosen];
    if (p.label != 0) r.ys.push_back(p.label);
    total += p.score;
    remaining = best[p.dst];
    s = p.dst;
  }
  r.score = total;
}

// One stream of fsa_beam_search (fsa_search.hpp:326-387) with
// lattice_to_best_seq(kMax) (394-409).
FsaResult fsa_one(const orc_model* m, const float* enc, int32_t T,
                  const orc_graph* g, double beam, int32_t max_states,
                  int32_t max_contexts) {
  const int32_t V = m->V;
  PdCache cache(m);
  std::vector<Tuple> active{{0, 0, 0.0, 0}};  // init_streams, 95-120
  std::vector<Piece> arcs;
  std::vector<int32_t> finals;
  int32_t num_nodes = 1;
  bool done = false;
  if (T == 0) {  // finish_stream at frame 0 (fsa_search.hpp:343)
    finals.push_back(0);
    done = true;
  }
  std::vector<float> pe(m->J), logits(V);
  for (int32_t t = 0; t < T && !done; ++t) {
    orc_affine(m->j_we, nullptr, enc + static_cast<size_t>(t) * m->D, 1, m->J,
               m->D, pe.data());
    // get_contexts (124-154): distinct contexts in ascending order, since
    // active is sorted by (context, state).
    std::vector<int32_t> ctxs;
    for (const Tuple& a : active)
      if (ctxs.empty() || ctxs.back() != a.ctx) ctxs.push_back(a.ctx);
    std::vector<std::vector<double>> lp(ctxs.size(), std::vector<double>(V));
    for (size_t r = 0; r < ctxs.size(); ++r) {
      orc_joiner_logits_from_proj(m, pe.data(), cache.get(ctxs[r]),
                                  logits.data());
      orc_log_softmax(logits.data(), V, lp[r].data());
    }
    // expand_arcs (161-223): raw candidates in generation order; the
    // candidate score of a key is the max over its raw candidates.
    struct Raw {
      Key key;
      Piece piece;
      double score;
    };
    std::vector<Raw> raw;
    for (const Tuple& a : active) {
      const size_t r =
          std::lower_bound(ctxs.begin(), ctxs.end(), a.ctx) - ctxs.begin();
      const double* row = lp[r].data();
      raw.push_back({{a.ctx, a.state}, {a.node, 0, 0, row[0]}, a.score + row[0]});
      for (int32_t e = g->arc_splits[a.state]; e < g->arc_splits[a.state + 1];
           ++e) {
        const int32_t lab = g->label[e];
        const double arc_score = g->weight[e] + row[lab];
        raw.push_back({{(a.ctx % V) * V + lab, g->dst[e]},
                       {a.node, 0, lab, arc_score},
                       a.score + arc_score});
      }
    }
    if (raw.empty()) {  // prune_streams, 233-238: the stream dies
      active.clear();
      done = true;
      break;
    }
    std::vector<std::pair<Key, double>> cand;
    {
      std::vector<std::pair<Key, double>> tmp;
      tmp.reserve(raw.size());
      for (const Raw& x : raw) tmp.push_back({x.key, x.score});
      std::stable_sort(tmp.begin(), tmp.end(),
                       [](const auto& a, const auto& b) { return a.first < b.first; });
      for (const auto& x : tmp) {
        if (!cand.empty() && cand.back().first == x.first)
          cand.back().second = std::max(cand.back().second, x.second);
        else
          cand.push_back(x);
      }
    }
    // prune_streams (240-283).
    std::vector<std::pair<Key, double>> order = cand;
    std::sort(order.begin(), order.end(), [](const auto& a, const auto& b) {
      if (a.second != b.second) return a.second > b.second;
      return a.first < b.first;
    });
    const double floor = order.front().second - beam;
    std::vector<std::pair<Key, double>> pass1;
    for (const auto& c : order) {
      if (c.second < floor) continue;
      pass1.push_back(c);
      if (static_cast<int32_t>(pass1.size()) == max_states) break;
    }
    std::vector<int32_t> kept;
    for (const auto& c : pass1)
      if (std::find(kept.begin(), kept.end(), c.first.ctx) == kept.end() &&
          static_cast<int32_t>(kept.size()) < max_contexts)
        kept.push_back(c.first.ctx);
    std::vector<Tuple> next;
    for (const auto& c : pass1)
      if (std::find(kept.begin(), kept.end(), c.first.ctx) != kept.end())
        next.push_back({c.first.ctx, c.first.state, c.second, -1});
    std::sort(next.begin(), next.end(), [](const Tuple& a, const Tuple& b) {
      return Key{a.ctx, a.state} < Key{b.ctx, b.state};
    });
    for (Tuple& n : next) n.node = num_nodes++;
    for (const Raw& x : raw) {
      auto it = std::lower_bound(next.begin(), next.end(), x.key,
                                 [](const Tuple& a, const Key& k) {
                                   return Key{a.ctx, a.state} < k;
                                 });
      if (it == next.end() || !(Key{it->ctx, it->state} == x.key)) continue;
      Piece p = x.piece;
      p.dst = it->node;
      arcs.push_back(p);
    }
    active = std::move(next);
    if (t + 1 == T) {
      for (const Tuple& a : active) finals.push_back(a.node);
      done = true;
    }
  }
  // build_lattice (309-317) + make_fsa's stable sort by src (fsa.hpp:100-101).
  FsaResult r;
  const int32_t super = num_nodes;
  for (int32_t f : finals) arcs.push_back({f, super, 0, 0.0});
  std::stable_sort(arcs.begin(), arcs.end(),
                   [](const Piece& a, const Piece& b) { return a.src < b.src; });
  r.arcs = std::move(arcs);
  r.num_nodes = num_nodes + 1;
  lattice_best(r, super);
  return r;
}

}  // namespace

extern "C" {

int orc_beam_search(const orc_model* m, const float* enc,
                    const int32_t* frame_splits, int32_t B, int32_t beam_size,
                    int32_t merge_op, int32_t length_norm,
                    int32_t max_total_symbols, int threads,
                    int32_t* out_splits, int32_t* out_tokens,
                    double* out_scores) {
  if (beam_size < 1) {
    g_err = "beam_size must be >= 1";
    return 1;
  }
  std::vector<std::vector<int32_t>> ys(B);
  for_streams(B, threads, [&](int32_t s) {
    auto r = beam_one(m, enc + static_cast<size_t>(frame_splits[s]) * m->D,
                      frame_splits[s + 1] - frame_splits[s], beam_size,
                      merge_op != 0, length_norm != 0, max_total_symbols);
    ys[s] = std::move(r.first);
    out_scores[s] = r.second;
  });
  out_splits[0] = 0;
  for (int32_t s = 0; s < B; ++s) {
    std::copy(ys[s].begin(), ys[s].end(), out_tokens + out_splits[s]);
    out_splits[s + 1] = out_splits[s] + static_cast<int32_t>(ys[s].size());
  }
  return 0;
}

int orc_fsa_beam_search(const orc_model* m, const float* enc,
                        const int32_t* frame_splits, int32_t B,
                        const orc_graph* g, double beam, int32_t max_states,
                        int32_t max_contexts, int threads, int32_t* out_splits,
                        int32_t* out_tokens, double* out_scores,
                        orc_lattice* lattices) {
  if (!(beam >= 0.0) || max_states < 1 || max_contexts < 1) {
    g_err = "invalid fsa search params";
    return 1;
  }
  for (int32_t e = 0; e < g->num_arcs; ++e)
    if (g->label[e] <= 0 || g->label[e] >= m->V) {
      g_err = "decoding graph label outside (0, V)";
      return 1;
    }
  std::vector<FsaResult> res(B);
  try {
    for_streams(B, threads, [&](int32_t s) {
      res[s] = fsa_one(m, enc + static_cast<size_t>(frame_splits[s]) * m->D,
                       frame_splits[s + 1] - frame_splits[s], g, beam,
                       max_states, max_contexts);
    });
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
  out_splits[0] = 0;
  for (int32_t s = 0; s < B; ++s) {
    std::copy(res[s].ys.begin(), res[s].ys.end(), out_tokens + out_splits[s]);
    out_splits[s + 1] = out_splits[s] + static_cast<int32_t>(res[s].ys.size());
    out_scores[s] = res[s].score;
    if (lattices) {
      orc_lattice& L = lattices[s];
      const auto& a = res[s].arcs;
      L.num_nodes = res[s].num_nodes;
      L.num_arcs = static_cast<int32_t>(a.size());
      L.src = static_cast<int32_t*>(malloc(sizeof(int32_t) * (a.size() + 1)));
      L.dst = static_cast<int32_t*>(malloc(sizeof(int32_t) * (a.size() + 1)));
      L.label = static_cast<int32_t*>(malloc(sizeof(int32_t) * (a.size() + 1)));
      L.score = static_cast<double*>(malloc(sizeof(double) * (a.size() + 1)));
      for (size_t i = 0; i < a.size(); ++i) {
        L.src[i] = a[i].src;
        L.dst[i] = a[i].dst;
        L.label[i] = a[i].label;
        L.score[i] = a[i].score;
      }
    }
  }
  return 0;
}

// Exhaustive-sweep support for the device tanhf port: per 2^24-input chunk,
// sum over inputs u of mix((u << 32) | bits(glibc tanhf(u))), NaN outputs
// canonicalised (same definition as the device kernel in csrc/debug.cu).
static unsigned long long orc_mix(unsigned long long x) {
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdull;
  x ^= x >> 33;
  x *= 0xc4ceb9fe1a85ec53ull;
  x ^= x >> 33;
  return x;
}

void orc_tanhf_chunk_hashes(int32_t first_chunk, int32_t num_chunks,
                            int threads, uint64_t* out) {
  for_streams(num_chunks, threads, [&](int32_t c) {
    const uint32_t base = static_cast<uint32_t>(first_chunk + c) << 24;
    unsigned long long acc = 0;
    for (uint32_t j = 0; j < (1u << 24); ++j) {
      const uint32_t u = base + j;
      float x;
      std::memcpy(&x, &u, 4);
      const float y = std::tanh(x);
      uint32_t bits;
      std::memcpy(&bits, &y, 4);
      if ((bits & 0x7fffffffu) > 0x7f800000u) bits = 0x7fc00000u;
      acc += orc_mix((static_cast<unsigned long long>(u) << 32) | bits);
    }
    out[c] = acc;
  });
}

void orc_lattice_free(orc_lattice* l) {
  free(l->src);
  free(l->dst);
  free(l->label);
  free(l->score);
  l->src = l->dst = l->label = nullptr;
  l->score = nullptr;
}

}  // extern "C"
