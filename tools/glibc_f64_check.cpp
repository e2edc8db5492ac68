// Host check of paper_2211_00484_b200/csrc/glibc_f64.h against this image's
// libm (glibc 2.39, FMA ifunc variants): random inputs over the ranges the
// decoders evaluate plus edge cases; prints one JSON line of mismatch counts.
//
//   g++ -std=c++17 -O2 -ffp-contract=off -o glibc_f64_check tools/glibc_f64_check.cpp
//   ./glibc_f64_check [samples_per_range] [seed]
#include <cinttypes>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>

#include "../paper_2211_00484_b200/csrc/glibc_f64.h"

static uint64_t bits(double x) {
  uint64_t u;
  std::memcpy(&u, &x, 8);
  return u;
}
static bool same(double a, double b) { return bits(a) == bits(b) || (std::isnan(a) && std::isnan(b)); }

int main(int argc, char** argv) {
  const long n = argc > 1 ? std::atol(argv[1]) : 2000000;
  const uint64_t seed = argc > 2 ? std::strtoull(argv[2], nullptr, 10) : 1;
  std::mt19937_64 g(seed);
  auto uni = [&](double lo, double hi) { return lo + (hi - lo) * (static_cast<double>(g() >> 11) * 0x1.0p-53); };
  long bad_exp = 0, bad_log = 0, bad_log1p = 0, n_exp = 0, n_log = 0, n_log1p = 0;
  double ex_example = 0, lg_example = 0, l1_example = 0;
  auto cexp = [&](double x) {
    ++n_exp;
    if (!same(rnntg_f64::exp(x), std::exp(x))) {
      if (!bad_exp++) ex_example = x;
    }
  };
  auto clog = [&](double x) {
    ++n_log;
    if (!same(rnntg_f64::log(x), std::log(x))) {
      if (!bad_log++) lg_example = x;
    }
  };
  auto clog1p = [&](double x) {
    ++n_log1p;
    if (!same(rnntg_f64::log1p(x), std::log1p(x))) {
      if (!bad_log1p++) l1_example = x;
    }
  };
  // exp: log-softmax arguments double(float l) - float max (<= 0), log_add
  // differences, sampling exponents; whole range incl. the special cases.
  for (long i = 0; i < n; ++i) {
    const float l = static_cast<float>(uni(-30.0, 30.0)), m = static_cast<float>(uni(-30.0, 30.0));
    cexp(static_cast<double>(l) - static_cast<double>(l > m ? l : m));
    cexp(uni(-50.0, 0.0));
    cexp(uni(-1.0, 1.0));
    cexp(uni(-745.2, 709.8));
    cexp(uni(-1e-12, 1e-12));
    uint64_t r = g();
    double x;
    std::memcpy(&x, &r, 8);
    cexp(x);
  }
  const double ex_edges[] = {0.0, -0.0, 1.0, -1.0, 0x1p-54, -0x1p-54, 0x1p-55, 512.0, -512.0, 709.78, 709.79, -708.4,
                             -745.13, -745.14, -1000.0, 1024.0, INFINITY, -INFINITY, NAN};
  for (double x : ex_edges) cexp(x);
  // log: log-softmax sums in [1, V], plus the whole positive range.
  for (long i = 0; i < n; ++i) {
    clog(uni(1.0, 1.1));
    clog(uni(1.0, 600.0));
    clog(uni(0.9, 1.1));
    uint64_t r = g() & 0x7fffffffffffffffull;
    double x;
    std::memcpy(&x, &r, 8);
    clog(x);
    clog(uni(0.0, 0x1p-1022));
  }
  const double lg_edges[] = {1.0, 0.0, -0.0, -1.0, INFINITY, NAN, 0x1p-1074, 0.9395, 1.0449, 2.0, 0.5};
  for (double x : lg_edges) clog(x);
  // log1p: log_add arguments exp(mn - mx) in (0, 1], plus (-1, inf).
  for (long i = 0; i < n; ++i) {
    clog1p(rnntg_f64::exp(uni(-50.0, 0.0)));
    clog1p(uni(0.0, 1.0));
    clog1p(uni(-1.0, 0.0));
    clog1p(uni(0.0, 0x1p-20));
    clog1p(uni(0.0, 0x1p-50));
    uint64_t r = g() & 0x7fffffffffffffffull;
    double x;
    std::memcpy(&x, &r, 8);
    clog1p(x);
  }
  const double l1_edges[] = {0.0, -0.0, 1.0, -1.0, -0.5, 0x1p-29, 0x1p-54, 0x1p-60, 0.41421, 0.41422, -0.2929,
                             -0.29290, 1e300, 0x1p53, INFINITY, NAN, -2.0};
  for (double x : l1_edges) clog1p(x);
  std::printf(
      "{\"exp\": [%ld, %ld], \"log\": [%ld, %ld], \"log1p\": [%ld, %ld], \"first_bad\": [%a, %a, %a]}\n", bad_exp,
      n_exp, bad_log, n_log, bad_log1p, n_log1p, ex_example, lg_example, l1_example);
  return (bad_exp || bad_log || bad_log1p) ? 1 : 0;
}
