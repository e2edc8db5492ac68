// Drop-in check: the same caller code decodes through the reference
// (rnnt::greedy_search_batch / beam_search / fsa_beam_search +
// lattice_to_best_seq) and through rnnt::gpu (include/rnnt_gpu.hpp over
// librnntg.so); outputs must be identical.  Built against the reference
// headers by tests/cpp/Makefile; run on the GPU by tests/test_cpp_shim.py.
#include <cmath>
#include <cstdio>
#include <random>
#include <vector>

#include "rnnt/fsa_search.hpp"
#include "rnnt/model.hpp"
#include "rnnt/search.hpp"
#include "rnnt_gpu.hpp"

int main() {
  using namespace rnnt;
  ModelConfig cfg;
  cfg.vocab_size = 500;
  cfg.feat_dim = 80;
  cfg.enc_dim = cfg.emb_dim = cfg.joiner_dim = 512;
  cfg.seed = 3;
  ToyTransducer m = init_model(cfg);
  m.out_b.at(0, 0) += 0.4f;
  std::vector<Mat<float>> batch;
  for (int i = 0; i < 6; ++i) {
    DetRng rng(900 + i);
    Mat<float> f(10 + 7 * i, cfg.feat_dim);
    for (float& v : f.data) v = static_cast<float>(rng.gaussian());
    batch.push_back(f);
  }
  gpu::Context ctx(m, 0);
  int bad = 0;
  if (gpu::greedy_search_batch(ctx, m, batch) != greedy_search_batch(m, batch)) {
    std::printf("greedy mismatch\n");
    ++bad;
  }
  SearchParams sp;
  sp.beam_size = 4;
  auto gb = gpu::beam_search_batch(ctx, m, batch, sp);
  for (size_t i = 0; i < batch.size(); ++i)
    if (gb[i] != beam_search(m, batch[i], sp)) {
      std::printf("beam mismatch %zu\n", i);
      ++bad;
    }
  Fsa g = trivial_graph(cfg.vocab_size);
  FsaSearchParams fp;
  fp.beam = 4.0;
  fp.max_states = 8;
  fp.max_contexts = 4;
  auto gf = gpu::fsa_best_sequences(ctx, m, batch, g, fp);
  if (gpu::fsa_best_sequences(ctx, m, batch, trivial_graph(cfg.vocab_size), fp) != gf) {  // cached graph
    std::printf("fsa (cached graph) mismatch\n");
    ++bad;
  }
  std::vector<Fsa> graphs(batch.size(), g);
  auto lats = fsa_beam_search(m, batch, graphs, fp);
  for (size_t i = 0; i < batch.size(); ++i)
    if (gf[i] != lattice_to_best_seq(lats[i], MergeOp::kMax)) {
      std::printf("fsa mismatch %zu\n", i);
      ++bad;
    }
  // Whole lattices through the reference-typed fsa_beam_search: equal Fsa
  // objects (nodes, arcs, labels, fp64 scores bit for bit, finals) and
  // byte-identical serialize_lattice text (the CLI's lattice files).
  auto glats = gpu::fsa_beam_search(ctx, m, batch, graphs, fp);
  for (size_t i = 0; i < batch.size(); ++i) {
    const Fsa& a = glats[i];
    const Fsa& b = lats[i];
    const bool same = a == b && serialize_lattice(a, static_cast<int32_t>(i), batch[i].rows) ==
                                    serialize_lattice(b, static_cast<int32_t>(i), batch[i].rows);
    if (!same || lattice_to_best_seq(a, MergeOp::kMax) != lattice_to_best_seq(b, MergeOp::kMax)) {
      std::printf("lattice mismatch %zu\n", i);
      ++bad;
    }
    // Log-add best sequence: the reference's own
    // lattice_to_best_seq(kLogAdd) — n-best sampling, blank-strip dedup,
    // per-sequence totals — on the GPU lattice, as the CLI calls it
    // (rnnt_main.cpp:302: nbest 100, the run seed).
    for (uint64_t seed : {0ull, 7ull})
      if (lattice_to_best_seq(a, MergeOp::kLogAdd, 100, seed) !=
          lattice_to_best_seq(b, MergeOp::kLogAdd, 100, seed)) {
        std::printf("log-add mismatch %zu seed %llu\n", i, static_cast<unsigned long long>(seed));
        ++bad;
      }
  }
  // ... and computed on the GPU (rnntg_fsa_lattice_best)
  for (uint64_t seed : {0ull, 7ull}) {
    auto gl = gpu::fsa_best_sequences(ctx, m, batch, g, fp, MergeOp::kLogAdd, 100, seed);
    for (size_t i = 0; i < batch.size(); ++i)
      if (gl[i] != lattice_to_best_seq(lats[i], MergeOp::kLogAdd, 100, seed)) {
        std::printf("GPU log-add mismatch %zu seed %llu\n", i, static_cast<unsigned long long>(seed));
        ++bad;
      }
  }
  // greedy_search with S = 3 and S unlimited (search.hpp:76-100)
  for (int32_t S : {3, kNoSymbolLimit}) {
    int64_t gcap = 0;
    auto gy = gpu::greedy_search_batched(ctx, m, batch, S, &gcap);
    int64_t rcap = 0;
    for (size_t i = 0; i < batch.size(); ++i) {
      int64_t c = 0;
      if (gy[i] != greedy_search(m, batch[i], S, &c)) {
        std::printf("greedy S=%d mismatch %zu\n", S, i);
        ++bad;
      }
      rcap += c;
    }
    if (S == kNoSymbolLimit && gcap != rcap) {
      std::printf("capped frames %lld vs %lld\n", static_cast<long long>(gcap), static_cast<long long>(rcap));
      ++bad;
    }
  }
  // beam_search with S = 2 and S unlimited (search.hpp:206-277)
  for (int32_t S : {2, kNoSymbolLimit}) {
    SearchParams bp;
    bp.beam_size = 4;
    bp.max_symbols = S;
    auto gb = gpu::beam_search_batch(ctx, m, batch, bp);
    for (size_t i = 0; i < batch.size(); ++i)
      if (gb[i] != beam_search(m, batch[i], bp)) {
        std::printf("beam S=%d mismatch %zu\n", S, i);
        ++bad;
      }
  }
  // The step API with the reference's types, against the reference's own
  // init_streams / get_contexts / expand_arcs / prune_streams on identical
  // caller rows (random_logprob_rows style): equal contexts, equal lattices.
  {
    std::vector<int32_t> nf = {5, 0, 3};
    FsaSearchParams sp2;
    sp2.beam = 3.0;
    sp2.max_states = 6;
    sp2.max_contexts = 3;
    gpu::FsaStreams gs(ctx, g, sp2, nf);
    std::vector<Fsa> rgraphs(nf.size(), g);
    std::vector<DecodeStream> rs = init_streams(rgraphs, sp2, cfg.vocab_size);
    for (size_t i = 0; i < nf.size(); ++i) {
      rs[i].num_frames = nf[i];
      if (nf[i] == 0) detail::finish_stream(rs[i]);
    }
    std::mt19937_64 rng(17);
    std::normal_distribution<double> nd(0.0, 1.0);
    for (int32_t t = 0; t < 5; ++t) {
      auto [gshape, gctx] = gs.get_contexts();
      auto [rshape, rctx] = get_contexts(rs);
      if (gshape.row_splits != rshape.row_splits || !(gctx == rctx)) {
        std::printf("step contexts mismatch t=%d\n", t);
        ++bad;
        break;
      }
      Mat<double> lp(rctx.rows, cfg.vocab_size);
      for (int32_t r = 0; r < lp.rows; ++r) {
        double mx = -1e300, sum = 0.0;
        for (int32_t k = 0; k < lp.cols; ++k) mx = std::max(mx, lp.at(r, k) = nd(rng));
        for (int32_t k = 0; k < lp.cols; ++k) sum += std::exp(lp.at(r, k) - mx);
        for (int32_t k = 0; k < lp.cols; ++k) lp.at(r, k) -= mx + std::log(sum);
      }
      gs.expand_and_prune(lp);
      expand_arcs(rs, rshape, lp);
      prune_streams(rs);
      for (DecodeStream& s : rs)
        if (!s.done && s.t == s.num_frames) detail::finish_stream(s);
    }
    std::vector<Fsa> glat = gs.finish();
    for (size_t i = 0; i < nf.size(); ++i)
      if (!(glat[i] == detail::build_lattice(rs[i]))) {
        std::printf("step lattice mismatch %zu\n", i);
        ++bad;
      }
  }
  try {
    gpu::greedy_search_batch(ctx, m, batch, 2);
    ++bad;
  } catch (const ValidationError&) {
  }
  std::printf(bad ? "FAIL %d\n" : "OK\n", bad);
  return bad ? 1 : 0;
}
