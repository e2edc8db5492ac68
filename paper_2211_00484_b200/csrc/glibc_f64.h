// Bit-exact double-precision exp / log / log1p of this image's glibc 2.39,
// for the device kernels and the host test harness.
//
// The reference's fp64 log-probabilities (log_softmax_row, model.hpp:115-125),
// its log_add (common.hpp:48-54) and its lattice sampling / totals
// (fsa.hpp:311-335, 390-448) call libm's exp, log and log1p.  On any x86-64
// with FMA and AVX2 glibc's ifuncs select __exp_fma, __log_fma and
// __log1p_fma: the same C sources (sysdeps/ieee754/dbl-64/e_exp.c, e_log.c,
// s_log1p.c) compiled with -mfma, where gcc contracted some `a * b + c` into
// vfmadd and left others as separate roundings.  The functions below issue
// exactly the operations of the disassembled FMA variants (objdump of
// libm.so.6 at 0x79b60, 0x79d50, 0x7aff0), in the same order, with the
// same constants (read from the same binary, glibc_f64_tables.h), so they
// return the same bits.  Every `fma` is a single correctly rounded fused
// multiply-add (vfmadd / DFMA), every other operation one IEEE rounding.
//
// Verified against the host libm on random and edge inputs over the ranges
// the decoders use (tests/test_glibc_f64.py, tools/glibc_f64_check.cpp) and,
// on the device, through the bit-equal log-probabilities and lattices of the
// parity tests.
//
// On the device every operation is an explicit __d*_rn / __fma_rn intrinsic
// (never contracted); on the host the file must be compiled with
// -ffp-contract=off (std::fma is the correctly rounded fused operation).
//
// log1p is fdlibm's algorithm, whose notice is reproduced as its licence
// requires:
//
//   ====================================================
//   Copyright (C) 1993 by Sun Microsystems, Inc. All rights reserved.
//
//   Developed at SunPro, a Sun Microsystems, Inc. business.
//   Permission to use, copy, modify, and distribute this
//   software is freely granted, provided that this notice
//   is preserved.
//   ====================================================
//
// exp and log are the Arm Optimized Routines implementations contributed to
// glibc (Copyright (c) 2018 Arm Ltd., SPDX-License-Identifier: MIT, as
// distributed in glibc under LGPL-2.1-or-later).
#pragma once

#include <stdint.h>

#include <cmath>
#include <cstring>

// In CUDA translation units the functions are device-only (the tables live
// in constant memory); in host C++ (the checker, the oracle) plain inline.
#if defined(__CUDACC__)
#define RNNTG_F64_HD __device__ __forceinline__
#define RNNTG_F64_TABLE __device__ __constant__ static const
#else
#define RNNTG_F64_HD static inline
#define RNNTG_F64_TABLE static const
#endif

#include "glibc_f64_tables.h"

namespace rnntg_f64 {

#if defined(__CUDA_ARCH__)
RNNTG_F64_HD double xadd(double a, double b) { return __dadd_rn(a, b); }
RNNTG_F64_HD double xsub(double a, double b) { return __dsub_rn(a, b); }
RNNTG_F64_HD double xmul(double a, double b) { return __dmul_rn(a, b); }
RNNTG_F64_HD double xdiv(double a, double b) { return __ddiv_rn(a, b); }
RNNTG_F64_HD double xfma(double a, double b, double c) { return __fma_rn(a, b, c); }
RNNTG_F64_HD uint64_t d2u(double x) { return static_cast<uint64_t>(__double_as_longlong(x)); }
RNNTG_F64_HD double u2d(uint64_t u) { return __longlong_as_double(static_cast<long long>(u)); }
#else
RNNTG_F64_HD double xadd(double a, double b) { return a + b; }
RNNTG_F64_HD double xsub(double a, double b) { return a - b; }
RNNTG_F64_HD double xmul(double a, double b) { return a * b; }
RNNTG_F64_HD double xdiv(double a, double b) { return a / b; }
RNNTG_F64_HD double xfma(double a, double b, double c) { return std::fma(a, b, c); }
RNNTG_F64_HD uint64_t d2u(double x) {
  uint64_t u;
  std::memcpy(&u, &x, 8);
  return u;
}
RNNTG_F64_HD double u2d(uint64_t u) {
  double x;
  std::memcpy(&x, &u, 8);
  return x;
}
#endif

// exp_t takes the table: the device kernels that evaluate exp per logit pass
// their own shared-memory copy of kExpTab (constant memory serialises
// divergent indices); everything else reads the constant/static table.
RNNTG_F64_HD double kInf() { return u2d(0x7ff0000000000000ull); }

// __exp_fma (e_exp.c, EXP_TABLE_BITS 7, specialcase inlined).
RNNTG_F64_HD double exp_t(double x, const uint64_t* T) {
  const double InvLn2N = 0x1.71547652b82fep+7, Shift = 0x1.8p52;
  const double NegLn2hiN = -0x1.62e42fefa0000p-8, NegLn2loN = -0x1.cf79abc9e3b3ap-47;
  const double C2 = 0x1.ffffffffffdbdp-2, C3 = 0x1.555555555543cp-3;
  const double C4 = 0x1.55555cf172b91p-5, C5 = 0x1.1111167a4d017p-7;
  const uint64_t ix = d2u(x);
  uint32_t abstop = static_cast<uint32_t>(ix >> 52) & 0x7ff;
  if (abstop - 0x3c9u > 0x3eu) {
    if (static_cast<int32_t>(abstop - 0x3c9u) < 0) return xadd(x, 1.0);  // |x| < 2^-54
    if (abstop > 0x408u) {                                                // |x| >= 1024
      if (ix == 0xfff0000000000000ull) return 0.0;
      if (abstop == 0x7ffu) return xadd(x, 1.0);
      return (ix >> 63) ? 0.0 : kInf();
    }
    abstop = 0;  // 512 <= |x| < 1024: specialcase below
  }
  double kd = xfma(x, InvLn2N, Shift);
  const uint64_t ki = d2u(kd);
  kd = xsub(kd, Shift);
  double r = xfma(kd, NegLn2hiN, x);
  r = xfma(kd, NegLn2loN, r);
  const uint32_t idx = 2u * static_cast<uint32_t>(ki & 0x7f);
  const uint64_t top = ki << 45;
  const double tail = u2d(T[idx]);
  uint64_t sbits = T[idx + 1] + top;
  const double p23 = xfma(r, C3, C2);
  const double tr = xadd(r, tail);
  const double r2 = xmul(r, r);
  const double p45 = xfma(r, C5, C4);
  const double t1 = xfma(p23, r2, tr);
  const double r4 = xmul(r2, r2);
  const double tmp = xfma(r4, p45, t1);
  if (abstop != 0) {
    const double scale = u2d(sbits);
    return xfma(scale, tmp, scale);
  }
  if ((ki & 0x80000000ull) == 0) {
    sbits -= 1009ull << 52;
    const double scale = u2d(sbits);
    return xmul(xfma(scale, tmp, scale), 0x1p1009);
  }
  sbits += 1022ull << 52;
  const double scale = u2d(sbits);
  const double st = xmul(tmp, scale);
  double y = xadd(scale, st);
  if (1.0 > y) {
    const double hi = xadd(y, 1.0);
    double lo = xsub(scale, y);
    lo = xadd(lo, st);
    double t = xsub(1.0, hi);
    t = xadd(t, y);
    t = xadd(t, lo);
    t = xadd(t, hi);
    y = xsub(t, 1.0);
    if (y == 0.0) y = 0.0;
  }
  return xmul(y, 0x1p-1022);
}

RNNTG_F64_HD double exp(double x) { return exp_t(x, kExpTab); }

// __log_fma (e_log.c, LOG_TABLE_BITS 7, HAVE_FAST_FMA: no tab2).
RNNTG_F64_HD double log(double x) {
  const double Ln2hi = 0x1.62e42fefa3800p-1, Ln2lo = 0x1.ef35793c76730p-45;
  const double A0 = -0x1.0000000000001p-1, A1 = 0x1.555555551305bp-2, A2 = -0x1.fffffffeb4590p-3,
               A3 = 0x1.999b324f10111p-3, A4 = -0x1.55575e506c89fp-3;
  const double B0 = -0x1p-1, B1 = 0x1.5555555555577p-2, B2 = -0x1.ffffffffffdcbp-3,
               B3 = 0x1.999999995dd0cp-3, B4 = -0x1.55555556745a7p-3, B5 = 0x1.24924a344de30p-3,
               B6 = -0x1.fffffa4423d65p-4, B7 = 0x1.c7184282ad6cap-4, B8 = -0x1.999eb43b068ffp-4,
               B9 = 0x1.78182f7afd085p-4, B10 = -0x1.5521375d145cdp-4;
  uint64_t ix = d2u(x);
  const uint32_t top = static_cast<uint32_t>(ix >> 48);
  if (ix - 0x3fee000000000000ull <= 0x308ffffffffffull) {  // x near 1
    if (ix == 0x3ff0000000000000ull) return 0.0;
    const double r = xsub(x, 1.0);
    double p2 = xfma(r, B2, B1);
    double p5 = xfma(r, B5, B4);
    const double r2 = xmul(r, r);
    const double p8 = xfma(r, B8, B7);
    p2 = xfma(r2, B3, p2);
    p5 = xfma(r2, B6, p5);
    const double r3 = xmul(r, r2);
    double q = xfma(r2, B9, p8);
    q = xfma(r3, B10, q);
    q = xfma(q, r3, p5);
    q = xfma(q, r3, p2);
    const double t = xfma(r, 0x1p27, r);
    const double rhi = xfma(-0x1p27, r, t);
    const double rhi2 = xmul(rhi, rhi);
    const double rlo = xsub(r, rhi);
    const double hi = xfma(rhi2, B0, r);
    double lo = xsub(r, hi);
    const double rp = xadd(r, rhi);
    lo = xfma(rhi2, B0, lo);
    const double u = xmul(B0, rlo);
    lo = xfma(u, rp, lo);
    const double y = xfma(q, r3, lo);
    return xadd(hi, y);
  }
  if (top - 0x0010u > 0x7fdfu) {
    if ((ix << 1) == 0) return -kInf();
    if (ix == 0x7ff0000000000000ull) return x;
    if ((top & 0x8000u) || (top & 0x7ff0u) == 0x7ff0u) return u2d(0x7ff8000000000000ull);
    ix = d2u(xmul(x, 0x1p52)) - (52ull << 52);  // subnormal
  }
  const uint64_t tmp = ix - 0x3fe6000000000000ull;
  const uint32_t i = static_cast<uint32_t>(tmp >> 45) & 0x7f;
  const int32_t k = static_cast<int32_t>(static_cast<int64_t>(tmp) >> 52);
  const uint64_t iz = ix - (tmp & 0xfff0000000000000ull);
  const double invc = u2d(kLogTab[2 * i]), logc = u2d(kLogTab[2 * i + 1]);
  const double z = u2d(iz);
  const double kd = static_cast<double>(k);
  const double w = xfma(kd, Ln2hi, logc);
  const double r = xfma(z, invc, -1.0);
  const double p12 = xfma(r, A2, A1);
  const double hi = xadd(r, w);
  const double r2 = xmul(r, r);
  double t = xsub(w, hi);
  t = xadd(t, r);
  const double lo = xfma(kd, Ln2lo, t);
  const double rr2 = xmul(r, r2);
  const double p34 = xfma(r, A4, A3);
  const double lo2 = xfma(r2, A0, lo);
  const double p = xfma(p34, r2, p12);
  const double y = xfma(rr2, p, lo2);
  return xadd(y, hi);
}

// __log1p_fma (fdlibm s_log1p.c).
RNNTG_F64_HD double log1p(double x) {
  const double ln2_hi = 0x1.62e42fee00000p-1, ln2_lo = 0x1.a39ef35793c76p-33;
  const double Lp1 = 0x1.5555555555593p-1, Lp2 = 0x1.999999997fa04p-2, Lp3 = 0x1.2492494229359p-2,
               Lp4 = 0x1.c71c51d8e78afp-3, Lp5 = 0x1.7466496cb03dep-3, Lp6 = 0x1.39a09d078c69fp-3,
               Lp7 = 0x1.2f112df3e5244p-3;
  const int32_t hx = static_cast<int32_t>(d2u(x) >> 32);
  int32_t k;
  double f, hfsq, c = 0.0, u;
  uint32_t hu;
  if (hx <= 0x3fda8279) {
    const uint32_t ax = static_cast<uint32_t>(hx) & 0x7fffffffu;
    if (ax > 0x3fefffffu) {
      if (x == -1.0) return -kInf();
      return u2d(0x7ff8000000000000ull);
    }
    if (ax <= 0x3e1fffffu) {
      if (ax > 0x3c8fffffu) return xfma(-xmul(x, x), 0.5, x);
      return x;
    }
    if (static_cast<uint32_t>(hx + 0x402d413c) > 0x402d413cu) {
      f = x;
      hfsq = xmul(xmul(x, 0.5), x);
      k = 0;
      goto main_path;
    }
    goto k_path;
  }
  if (hx > 0x7fefffff) return xadd(x, x);
  if (hx <= 0x433fffff) goto k_path;
  k = (hx >> 20) - 1023;
  u = x;
  hu = static_cast<uint32_t>(hx);
  c = 0.0;
  goto normalise;
k_path:
  u = xadd(x, 1.0);
  hu = static_cast<uint32_t>(d2u(u) >> 32);
  k = (static_cast<int32_t>(hu) >> 20) - 1023;
  if (k <= 0)
    c = xsub(x, xsub(u, 1.0));
  else
    c = xsub(1.0, xsub(u, x));
  c = xdiv(c, u);
normalise:
  hu &= 0x000fffffu;
  if (hu > 0x6a09du) {
    k += 1;
    u = u2d((static_cast<uint64_t>(hu | 0x3fe00000u) << 32) | (d2u(u) & 0xffffffffull));
    hu = static_cast<uint32_t>(static_cast<int32_t>(0x00100000u - hu) >> 2);
  } else {
    u = u2d((static_cast<uint64_t>(hu | 0x3ff00000u) << 32) | (d2u(u) & 0xffffffffull));
  }
  f = xsub(u, 1.0);
  hfsq = xmul(xmul(f, 0.5), f);
  if (hu == 0) {
    if (f == 0.0) {
      if (k == 0) return 0.0;
      const double kd = static_cast<double>(k);
      return xfma(kd, ln2_hi, xfma(kd, ln2_lo, c));
    }
    const double R = xmul(xfma(-f, 0x1.5555555555555p-1, 1.0), hfsq);
    if (k == 0) return xsub(f, R);
    const double kd = static_cast<double>(k);
    double t = xfma(kd, ln2_lo, c);
    t = xsub(R, t);
    t = xsub(t, f);
    return xfma(kd, ln2_hi, -t);
  }
main_path : {
  const double s = xdiv(f, xadd(f, 2.0));
  const double z = xmul(s, s);
  const double R2 = xfma(z, Lp3, Lp2), R3 = xfma(z, Lp5, Lp4), R4 = xfma(z, Lp7, Lp6);
  const double z2 = xmul(z, z);
  const double z4 = xmul(z2, z2);
  const double z6 = xmul(z2, z4);
  double R = xfma(z, Lp1, xmul(z2, R2));
  R = xfma(z4, R3, R);
  R = xfma(z6, R4, R);
  const double t = xmul(xadd(R, hfsq), s);
  if (k == 0) return xsub(f, xsub(hfsq, t));
  const double kd = static_cast<double>(k);
  double v = xfma(kd, ln2_lo, c);
  v = xadd(v, t);
  v = xsub(hfsq, v);
  v = xsub(v, f);
  return xfma(kd, ln2_hi, -v);
}
}

// common.hpp:48-54.
RNNTG_F64_HD double log_add(double a, double b) {
  if (a == -kInf()) return b;
  if (b == -kInf()) return a;
  const double mx = a > b ? a : b;
  const double mn = a > b ? b : a;
  return xadd(mx, log1p(exp(xsub(mn, mx))));
}

}  // namespace rnntg_f64
