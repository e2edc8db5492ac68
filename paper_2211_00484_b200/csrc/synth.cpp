// Host-side synthetic inputs identical to the reference's: the model weights
// init_model draws (model.hpp:129-169) and the per-stream gaussian features
// of SURVEY.md §8(d) (DetRng(seed).gaussian(), common.hpp:86-127).
//
// The reference derives every random number from raw std::mt19937_64 bits
// (standardised, platform-independent): uniforms as (x >> 11) * 2^-53, and
// gaussians by Box-Muller with a cached spare, in double through glibc
// log/sqrt/sin/cos.  This file restates those rules (no reference code is
// included), so the GPU arm of bench.py and any drop-in user decode the same
// bits the reference arm does.  Built with the library's host flags: no
// -ffast-math, and baseline x86-64 has no FMA to contract into.
#include <cmath>
#include <cstdint>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include "../../include/rnntg.h"

namespace rnntg {
void set_error(const std::string& msg);
}

namespace {

class Rng {  // DetRng's contract
 public:
  explicit Rng(uint64_t seed) : gen_(seed) {}
  double uniform01() { return static_cast<double>(gen_() >> 11) * 0x1.0p-53; }
  double uniform(double lo, double hi) { return lo + (hi - lo) * uniform01(); }
  double gaussian() {
    if (spare_ok_) {
      spare_ok_ = false;
      return spare_;
    }
    double u1 = uniform01();
    const double u2 = uniform01();
    while (u1 <= 1e-300) u1 = uniform01();
    const double r = std::sqrt(-2.0 * std::log(u1));
    const double th = 2.0 * M_PI * u2;
    spare_ = r * std::sin(th);
    spare_ok_ = true;
    return r * std::cos(th);
  }

 private:
  std::mt19937_64 gen_;
  bool spare_ok_ = false;
  double spare_ = 0.0;
};

void fill(float* dst, int64_t n, int32_t fan_in, Rng& rng) {
  const double s = 1.0 / std::sqrt(static_cast<double>(fan_in));
  if (dst) {
    for (int64_t i = 0; i < n; ++i) dst[i] = static_cast<float>(rng.uniform(-s, s));
  } else {
    for (int64_t i = 0; i < n; ++i) rng.uniform(-s, s);  // keep the draw order
  }
}

}  // namespace

extern "C" {

rnntg_status rnntg_init_model_weights(const rnntg_model_config* c, const rnntg_weight_ptrs* w) {
  if (!c || !w) {
    rnntg::set_error("null argument");
    return RNNTG_INVALID_ARGUMENT;
  }
  // check_config (model.hpp:174-182)
  if (c->vocab_size < 2 || c->feat_dim < 1 || c->enc_dim < 1 || c->emb_dim < 1 || c->joiner_dim < 1) {
    rnntg::set_error("model dims must be >= 1 and vocab_size >= 2");
    return RNNTG_INVALID_ARGUMENT;
  }
  const int64_t V = c->vocab_size, F = c->feat_dim, D = c->enc_dim, E = c->emb_dim, J = c->joiner_dim;
  Rng rng(c->seed);
  // Fill order and fan-ins of init_model (model.hpp:151-167); the four
  // auxiliary heads after out_b draw last and are not needed here.
  fill(w->enc_w1, D * F, static_cast<int32_t>(F), rng);
  fill(w->enc_b1, D, static_cast<int32_t>(F), rng);
  fill(w->enc_w2, D * D, static_cast<int32_t>(D), rng);
  fill(w->enc_b2, D, static_cast<int32_t>(D), rng);
  fill(w->emb, V * E, static_cast<int32_t>(E), rng);
  fill(w->ctx_w, E * 2 * E, static_cast<int32_t>(2 * E), rng);
  fill(w->ctx_b, E, static_cast<int32_t>(2 * E), rng);
  fill(w->j_we, J * D, static_cast<int32_t>(D), rng);
  fill(w->j_wd, J * E, static_cast<int32_t>(E), rng);
  fill(w->j_b, J, static_cast<int32_t>(D), rng);
  fill(w->out_w, V * J, static_cast<int32_t>(J), rng);
  fill(w->out_b, V, static_cast<int32_t>(J), rng);
  return RNNTG_OK;
}

rnntg_status rnntg_gaussian_features(uint64_t seed0, int32_t B, int32_t T, int32_t feat_dim, int32_t threads,
                                     float* out) {
  if (B < 0 || T < 0 || feat_dim < 1 || (B > 0 && T > 0 && !out)) {
    rnntg::set_error("bad feature shape");
    return RNNTG_INVALID_ARGUMENT;
  }
  const int64_t per = static_cast<int64_t>(T) * feat_dim;
  auto work = [&](int32_t i0, int32_t i1) {
    for (int32_t i = i0; i < i1; ++i) {
      Rng rng(seed0 + static_cast<uint64_t>(i));
      float* o = out + per * i;
      for (int64_t k = 0; k < per; ++k) o[k] = static_cast<float>(rng.gaussian());
    }
  };
  int32_t nt = threads > 0 ? threads : static_cast<int32_t>(std::thread::hardware_concurrency());
  nt = std::max(1, std::min(nt, B));
  std::vector<std::thread> pool;
  for (int32_t k = 0; k < nt; ++k) {
    const int32_t i0 = static_cast<int32_t>(static_cast<int64_t>(B) * k / nt);
    const int32_t i1 = static_cast<int32_t>(static_cast<int64_t>(B) * (k + 1) / nt);
    pool.emplace_back(work, i0, i1);
  }
  for (auto& t : pool) t.join();
  return RNNTG_OK;
}

}  // extern "C"
