// K0 / K1: bit-exact sequential fp32 projections on CUDA cores.
//
// Reference arithmetic (model.hpp:100-108 affine, 263-281 joiner projections):
// every output is   acc = init; for k in 0..K-1: acc = fl(acc + fl(w[k]*x[k]))
// with scalar SSE mulss/addss — no FMA, no reassociation.  A register-tiled
// SGEMM whose threads walk k in order and issue FMUL then FADD (explicit
// __fmul_rn/__fadd_rn, which nvcc never contracts) reproduces that exactly:
// tiling only changes which thread owns an output, never the order of its sum.
//
// Used for
//   K1  pe[t] = j_we . enc[t]                    (joiner_project_enc, 263-271)
//   K0  dec[c] = tanh(ctx_b + ctx_w . [emb a; emb b])   (decoder_forward 241-259)
//       pd[c]  = j_wd . dec[c]                   (joiner_project_dec, 273-281)
// The decoder-side table pd[c] for every packed context c = a*V+b is a pure
// function of c (model.hpp:240), so it is computed once per model.
#include "exact_math.h"
#include "internal.cuh"

namespace rnntg {
namespace {

using rnntg_exact::fadd;
using rnntg_exact::fmul;

constexpr int BM = 64, BN = 128, BK = 16, TM = 4, TN = 8;
constexpr int kThreads = (BM / TM) * (BN / TN);  // 256

// Row groups: logical row m of a launch is physical row
// (m / grp) * gstride + m % grp of X and Y (grp = 0: m itself).  A time slice
// [t0, t0 + grp) of B streams of uniform length T is grp = slice length,
// gstride = T, X and Y offset by t0 rows.
__device__ __forceinline__ int64_t phys_row(int64_t m, int32_t grp, int64_t gstride) {
  return grp > 0 ? (m / grp) * gstride + m % grp : m;
}

template <bool kGather>
__device__ __forceinline__ float load_x(const float* __restrict__ X, int64_t ldx,
                                        int64_t m, int64_t mp, int32_t k, int64_t M,
                                        int32_t K, const float* __restrict__ emb,
                                        int32_t V, int64_t ctx_base) {
  if (m >= M || k >= K) return 0.0f;
  if constexpr (kGather) {
    const int32_t E = K >> 1;
    const int64_t c = ctx_base + m;
    const int64_t tok = k < E ? c / V : c % V;
    return emb[tok * E + (k < E ? k : k - E)];
  } else {
    return X[mp * ldx + k];
  }
}

template <bool kGather, bool kTanh>
__global__ void __launch_bounds__(kThreads)
    gemm_exact_kernel(const float* __restrict__ X, int64_t ldx,
                      const float* __restrict__ Wt, int32_t ldw,
                      const float* __restrict__ bias, float* __restrict__ Y,
                      int64_t ldy, int64_t M, int32_t N, int32_t K,
                      const float* __restrict__ emb, int32_t V,
                      int64_t ctx_base, int32_t grp, int64_t gstride) {
  __shared__ __align__(16) float Xs[2][BK][BM];
  __shared__ __align__(16) float Ws[2][BK][BN];

  const int tid = threadIdx.x;
  const int tm = tid / (BN / TN);  // 0..15
  const int tn = tid % (BN / TN);  // 0..15
  const int64_t m0 = static_cast<int64_t>(blockIdx.y) * BM;
  const int32_t n0 = blockIdx.x * BN;

  // Global->register staging: X tile is BM x BK (one row, 4 k per thread),
  // W tile is BK x BN (two float4 per thread).
  const int xr = tid / 4, xk = (tid % 4) * 4;
  const int64_t xm = phys_row(m0 + xr, grp, gstride);
  float xreg[4];
  float4 wreg[2];

  auto gload = [&](int32_t k0) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
      xreg[i] = load_x<kGather>(X, ldx, m0 + xr, xm, k0 + xk + i, M, K, emb, V,
                                ctx_base);
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int idx = tid + i * kThreads;  // 0..511 float4 slots
      const int r = idx / (BN / 4), c4 = idx % (BN / 4);
      const int32_t k = k0 + r;
      wreg[i] = k < K ? *reinterpret_cast<const float4*>(
                            Wt + static_cast<int64_t>(k) * ldw + n0 + c4 * 4)
                      : make_float4(0.f, 0.f, 0.f, 0.f);
    }
  };
  auto sstore = [&](int buf) {
#pragma unroll
    for (int i = 0; i < 4; ++i) Xs[buf][xk + i][xr] = xreg[i];
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int idx = tid + i * kThreads;
      const int r = idx / (BN / 4), c4 = idx % (BN / 4);
      *reinterpret_cast<float4*>(&Ws[buf][r][c4 * 4]) = wreg[i];
    }
  };

  float acc[TM][TN];
#pragma unroll
  for (int j = 0; j < TN; ++j) {
    const int32_t n = n0 + (j < 4 ? tn * 4 + j : 64 + tn * 4 + (j - 4));
    const float init = (bias != nullptr && n < N) ? bias[n] : 0.0f;
#pragma unroll
    for (int i = 0; i < TM; ++i) acc[i][j] = init;
  }

  const int32_t nk = (K + BK - 1) / BK;
  gload(0);
  sstore(0);
  __syncthreads();
  for (int32_t c = 0; c < nk; ++c) {
    const int buf = c & 1;
    if (c + 1 < nk) gload((c + 1) * BK);
    const int kk_end = min(BK, K - c * BK);
    auto step = [&](int kk) {
      const float4 x4 = *reinterpret_cast<const float4*>(&Xs[buf][kk][tm * 4]);
      const float4 wa = *reinterpret_cast<const float4*>(&Ws[buf][kk][tn * 4]);
      const float4 wb =
          *reinterpret_cast<const float4*>(&Ws[buf][kk][64 + tn * 4]);
      const float xv[4] = {x4.x, x4.y, x4.z, x4.w};
      const float wv[8] = {wa.x, wa.y, wa.z, wa.w, wb.x, wb.y, wb.z, wb.w};
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = fadd(acc[i][j], fmul(wv[j], xv[i]));
    };
    if (kk_end == BK) {  // full chunk: straight-line code, no loop overhead
#pragma unroll
      for (int kk = 0; kk < BK; ++kk) step(kk);
    } else {
      for (int kk = 0; kk < kk_end; ++kk) step(kk);
    }
    if (c + 1 < nk) {
      sstore(buf ^ 1);
    }
    __syncthreads();
  }

#pragma unroll
  for (int i = 0; i < TM; ++i) {
    const int64_t m = m0 + tm * 4 + i;
    if (m >= M) continue;
    const int64_t mp = phys_row(m, grp, gstride);
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      const int32_t n = n0 + (j < 4 ? tn * 4 + j : 64 + tn * 4 + (j - 4));
      if (n < N) {
        float v = acc[i][j];
        if constexpr (kTanh) v = rnntg_exact::tanhf_glibc(v);
        Y[mp * ldy + n] = v;
      }
    }
  }
}

}  // namespace

cudaError_t launch_gemm_exact_grouped(const float* X, int64_t ldx, const float* Wt, int32_t ldw,
                                      const float* bias, float* Y, int64_t ldy, int64_t M, int32_t N,
                                      int32_t K, bool apply_tanh, const float* ctx_emb,
                                      int32_t ctx_V, int64_t ctx_base, int32_t grp, int64_t gstride,
                                      cudaStream_t stream) {
  if (M <= 0 || N <= 0) return cudaSuccess;
  if (grp > 0 && (ctx_emb || M % grp != 0)) return cudaErrorInvalidValue;
  // The grid's y dimension is limited to 65535 tiles per launch (a multiple
  // of grp rows, so every launch starts on a group boundary).
  int64_t max_rows = static_cast<int64_t>(65535) * BM;
  if (grp > 0) max_rows = max_rows / grp * grp;
  for (int64_t r0 = 0; r0 < M; r0 += max_rows) {
    const int64_t rows = M - r0 < max_rows ? M - r0 : max_rows;
    dim3 grid((N + BN - 1) / BN, static_cast<unsigned>((rows + BM - 1) / BM));
    const int64_t p0 = grp > 0 ? r0 / grp * gstride : r0;
    const float* Xp = ctx_emb ? nullptr : X + p0 * ldx;
    float* Yp = Y + p0 * ldy;
    if (ctx_emb) {
      if (apply_tanh)
        gemm_exact_kernel<true, true><<<grid, kThreads, 0, stream>>>(
            Xp, ldx, Wt, ldw, bias, Yp, ldy, rows, N, K, ctx_emb, ctx_V,
            ctx_base + r0, 0, 0);
      else
        gemm_exact_kernel<true, false><<<grid, kThreads, 0, stream>>>(
            Xp, ldx, Wt, ldw, bias, Yp, ldy, rows, N, K, ctx_emb, ctx_V,
            ctx_base + r0, 0, 0);
    } else {
      if (apply_tanh)
        gemm_exact_kernel<false, true><<<grid, kThreads, 0, stream>>>(
            Xp, ldx, Wt, ldw, bias, Yp, ldy, rows, N, K, nullptr, 0, 0, grp, gstride);
      else
        gemm_exact_kernel<false, false><<<grid, kThreads, 0, stream>>>(
            Xp, ldx, Wt, ldw, bias, Yp, ldy, rows, N, K, nullptr, 0, 0, grp, gstride);
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t launch_gemm_exact(const float* X, int64_t ldx, const float* Wt,
                              int32_t ldw, const float* bias, float* Y,
                              int64_t ldy, int64_t M, int32_t N, int32_t K,
                              bool apply_tanh, const float* ctx_emb,
                              int32_t ctx_V, int64_t ctx_base,
                              cudaStream_t stream) {
  return launch_gemm_exact_grouped(X, ldx, Wt, ldw, bias, Y, ldy, M, N, K, apply_tanh, ctx_emb,
                                   ctx_V, ctx_base, 0, 0, stream);
}

}  // namespace rnntg
