// End-to-end timing of the C++ drop-in (include/rnnt_gpu.hpp): the
// reference's own call shape -- acoustic features in host memory, token
// sequences back -- through rnnt::gpu::beam_search_batch (GPU encoder,
// exact joiner, beam 4).  Inputs are the bench's: init_model(seed 0) with
// blank bias 0.4, features DetRng(7000 + stream).gaussian() [T x 80].
//
//   shim_bench [B=1024] [T=1000] [reps=3]
// prints one JSON line: frames/s over `reps` calls (after one warm-up call)
// and the tokens/frame of the result.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "rnnt/fsa_search.hpp"
#include "rnnt/model.hpp"
#include "rnnt/search.hpp"
#include "rnnt_gpu.hpp"

int main(int argc, char** argv) {
  using namespace rnnt;
  const int B = argc > 1 ? std::atoi(argv[1]) : 1024;
  const int T = argc > 2 ? std::atoi(argv[2]) : 1000;
  const int reps = argc > 3 ? std::atoi(argv[3]) : 3;
  ModelConfig cfg;
  cfg.vocab_size = 500;
  cfg.feat_dim = 80;
  cfg.enc_dim = cfg.emb_dim = cfg.joiner_dim = 512;
  cfg.seed = 0;
  ToyTransducer m = init_model(cfg);
  m.out_b.at(0, 0) += 0.4f;
  std::vector<Mat<float>> batch;
  batch.reserve(B);
  for (int i = 0; i < B; ++i) {
    DetRng rng(7000 + i);
    Mat<float> f(T, cfg.feat_dim);
    for (float& v : f.data) v = static_cast<float>(rng.gaussian());
    batch.push_back(std::move(f));
  }
  gpu::Context ctx(m, 0);
  SearchParams sp;
  sp.beam_size = 4;
  auto ys = gpu::beam_search_batch(ctx, m, batch, sp);  // warm-up
  const auto t0 = std::chrono::steady_clock::now();
  for (int r = 0; r < reps; ++r) ys = gpu::beam_search_batch(ctx, m, batch, sp);
  const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  long long ntok = 0;
  for (const auto& y : ys) ntok += static_cast<long long>(y.size());
  const double frames = static_cast<double>(B) * T * reps;
  std::printf(
      "{\"api\": \"rnnt::gpu::beam_search_batch (C++ drop-in, host features -> tokens)\", \"B\": %d, \"T\": %d, "
      "\"reps\": %d, \"frames_per_s\": %.1f, \"ms_per_call\": %.3f, \"tokens_per_frame\": %.4f, "
      "\"h2d_bytes_per_call\": %lld}\n",
      B, T, reps, frames / s, 1e3 * s / reps, static_cast<double>(ntok) / (static_cast<double>(B) * T),
      static_cast<long long>(B) * T * cfg.feat_dim * 4);
  return 0;
}
