// Device building blocks shared by the persistent decode kernels
// (decode.cu: greedy / modified beam; fsa.cu: FSA beam search).
#pragma once

#include <float.h>
#include <cuda_bf16.h>
#include <math.h>

#include "exact_math.h"
#include "glibc_f64.h"
#include "internal.cuh"
#include "tc_common.cuh"

namespace rnntg {
namespace dec {

using rnntg_exact::fadd;
using rnntg_exact::fmul;

constexpr int kWarps = kDecodeThreads / 32;  // 16
constexpr int kBK = 32;                      // k rows per weight chunk (greedy / beam)
constexpr int kBKSmall = 16;                 // ... where shared memory is tighter (FSA, warp-specialised)
constexpr int kRowCap = 32;                  // joiner rows per CTA per frame
constexpr int kHStride = kRowCap + 4;        // padded k-major h tile stride

struct ModelView {
  int32_t V, J, Vp;
  const float* __restrict__ out_wt;  // [J][Vp]
  const float* __restrict__ out_b;   // [Vp]
  const float* __restrict__ j_b;     // [J]
  const float* __restrict__ pd;      // [V*V][J]
  const uint16_t* __restrict__ out_w_tc;  // bf16 out_w in UMMA chunk layout (tcgen05 variant)
};

// ---------------------------------------------------------------------------
// mbarrier + bulk copy helpers (sm_90+ PTX, SASS UBLKCP / SYNCS).
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
// Explicit shared-space loads: the out_w stage is addressed through a
// runtime stage index, which defeats nvcc's address-space inference (it
// would emit generic LD.E instead of LDS).  Not volatile: the compiler may
// schedule them; the mbarrier wait / __syncthreads asm carry "memory".
__device__ __forceinline__ float4 lds128(uint32_t a) {
  float4 v;
  asm("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ float2 lds64(uint32_t a) {
  float2 v;
  asm("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(a));
  return v;
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile(
      "mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
          smem_u32(bar)),
      "r"(bytes)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src,
                                         uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes "
      "[%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// ---------------------------------------------------------------------------
// Asynchronous copies and cluster (DSMEM) stores.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                   static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
               "l"(src)
               : "memory");
}
// DSMEM address of the same shared variable in CTA `rank` of the cluster.
__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
// Stores into another CTA's shared memory that complete their byte count on
// that CTA's mbarrier (no cluster barrier needed).
__device__ __forceinline__ void st_async_v2(uint32_t dst, uint32_t a, uint32_t b, uint32_t bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.b32 [%0], {%1, %2}, [%3];" ::"r"(dst),
               "r"(a), "r"(b), "r"(bar)
               : "memory");
}
__device__ __forceinline__ void st_async_v4(uint32_t dst, float a, float b, float c, float d, uint32_t bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(
                   dst),
               "r"(__float_as_uint(a)), "r"(__float_as_uint(b)), "r"(__float_as_uint(c)), "r"(__float_as_uint(d)),
               "r"(bar)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
__device__ __forceinline__ void st_async_b32(uint32_t dst, float a, uint32_t bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];" ::"r"(dst),
               "r"(__float_as_uint(a)), "r"(bar)
               : "memory");
}

// acc[j] += w[k] * h_j[k] for k = 0..J-1 in order (FMUL, then FADD: the
// reference's sequential sum) for NR rows h_j = h0 + j * hstep sharing the
// column wc (both k-contiguous, 16-byte aligned).  Operands come 4 k per
// LDS.128; the next U*4 k are loaded while the current ones run, so the
// shared-memory latency hides under the FADD chains.  J % (4U) == 0.
template <int NR, int U>
__device__ __forceinline__ void logit_chain_rows(const float* wc, const float* h0, int hstep, int J, float* acc) {
  float4 w[U], h[NR][U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    w[u] = *reinterpret_cast<const float4*>(wc + 4 * u);
#pragma unroll
    for (int j = 0; j < NR; ++j) h[j][u] = *reinterpret_cast<const float4*>(h0 + j * hstep + 4 * u);
  }
  for (int k = 0; k < J; k += 4 * U) {
    const int kn = min(k + 4 * U, J - 4 * U);  // the last block reloads itself
    float4 wn[U], hn[NR][U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      wn[u] = *reinterpret_cast<const float4*>(wc + kn + 4 * u);
#pragma unroll
      for (int j = 0; j < NR; ++j) hn[j][u] = *reinterpret_cast<const float4*>(h0 + j * hstep + kn + 4 * u);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
#pragma unroll
      for (int j = 0; j < NR; ++j) acc[j] = fadd(acc[j], fmul(w[u].x, h[j][u].x));
#pragma unroll
      for (int j = 0; j < NR; ++j) acc[j] = fadd(acc[j], fmul(w[u].y, h[j][u].y));
#pragma unroll
      for (int j = 0; j < NR; ++j) acc[j] = fadd(acc[j], fmul(w[u].z, h[j][u].z));
#pragma unroll
      for (int j = 0; j < NR; ++j) acc[j] = fadd(acc[j], fmul(w[u].w, h[j][u].w));
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      w[u] = wn[u];
#pragma unroll
      for (int j = 0; j < NR; ++j) h[j][u] = hn[j][u];
    }
  }
}

// ---------------------------------------------------------------------------
// Weight chunk pipeline.  Chunk g (a running sequence number across frames)
// lives in stage g & 1.  The sequence is data independent and periodic:
// optionally a_nc chunks of matrix A (the fused encoder projection j_we^T,
// once per `period` frames), then `period` passes of nc chunks of matrix B
// (out_w^T, once per frame).  Each chunk is kBK k-rows of a k-major [K][N]
// matrix; both matrices share the stage size (N_A == N_B).
// ---------------------------------------------------------------------------
struct WPipe {
  float* stage[2];
  uint64_t* bar;  // [2]
  uint32_t* cur;  // [2] smem issue cursor (thread 0): position in the period, B chunk index
  int32_t bk;     // k rows per chunk
  int32_t nc;     // chunks per B pass
  const float* b_ptr;
  int32_t b_K, b_N;
  const float* a_ptr;  // nullptr: no A passes
  int32_t a_nc, a_K;
  int32_t period;      // B passes per A pass
  int32_t defer;       // 1: the next frame's first two chunks are issued by
                       // wpipe_issue_next after the row reduction (which then
                       // uses both stages as scratch), not by the GEMM
};

__device__ __forceinline__ WPipe make_wpipe(float* W0, float* W1, uint64_t* bar, uint32_t* cur,
                                            const ModelView& m, int bk = kBK) {
  return WPipe{{W0, W1}, bar, cur, bk, (m.J + bk - 1) / bk, m.out_wt, m.J, m.Vp, nullptr, 0, 0, 1, 0};
}

// Issues chunk g (thread 0; chunks are issued strictly in sequence, so the
// schedule position advances by a cursor — no division on the issuing
// warp's path).
__device__ __forceinline__ void wpipe_issue(const WPipe& p, const ModelView& /*m*/, uint32_t g) {
  if (g == 0) {
    p.cur[0] = 0;
    p.cur[1] = 0;
  }
  const int32_t q = static_cast<int32_t>(p.cur[0]);
  const int32_t per = p.a_nc + p.period * p.nc;
  p.cur[0] = q + 1 == per ? 0u : static_cast<uint32_t>(q + 1);
  const float* src;
  int32_t rows;
  if (q < p.a_nc) {
    rows = min(p.bk, p.a_K - q * p.bk);
    src = p.a_ptr + static_cast<int64_t>(q) * p.bk * p.b_N;
  } else {
    const int32_t c = static_cast<int32_t>(p.cur[1]);
    p.cur[1] = c + 1 == p.nc ? 0u : static_cast<uint32_t>(c + 1);
    rows = min(p.bk, p.b_K - c * p.bk);
    src = p.b_ptr + static_cast<int64_t>(c) * p.bk * p.b_N;
  }
  const uint32_t bytes = static_cast<uint32_t>(rows) * p.b_N * 4u;
  uint64_t* bar = p.bar + (g & 1u);
  fence_proxy_async();
  mbar_expect_tx(bar, bytes);
  bulk_g2s(p.stage[g & 1u], src, bytes, bar);
}

// The two refills a deferring GEMM skipped (chunks g, g + 1: the next
// frame's first two), once the stages are free again.  Call after a CTA
// barrier that retired every generic-proxy access of the stages.
__device__ __forceinline__ void wpipe_issue_next(const WPipe& p, const ModelView& m, uint32_t g) {
  if (threadIdx.x == kDecodeThreads - 32) {
    wpipe_issue(p, m, g);
    wpipe_issue(p, m, g + 1);
  }
}

// C. logits[r][n] = out_b[n] + sum_k out_w[n][k] * h[r][k], sequential in k.
// Hs: k-major h tile [J][kHStride]; Ls (aliasing Hs): row-major [R][Vp].
// Work item = (4 rows, a block of 32*TN columns); warp w takes item w.  TN
// is picked per frame so that as many of the 16 warps as possible hold an
// item (TN=8: lane columns {4l..4l+3, 128+4l..}; TN=4: {4l..4l+3};
// TN=2: {2l, 2l+1}).  Every warp walks the k chunks in order, so each
// accumulator still sees k = 0..J-1 sequentially.
template <int TN>
__device__ __forceinline__ void gemm_pass(const ModelView& m, const WPipe& p,
                                          uint32_t& g, float* HL, int R) {
  constexpr int CW = 32 * TN;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int NB = m.Vp / CW;
  const int items = ((R + 3) >> 2) * NB;
  const bool active = warp < items;
  const int rg = warp / NB, blk = warp % NB;
  const int cbase = blk * CW;
  int col[TN];
#pragma unroll
  for (int j = 0; j < TN; ++j) {
    if constexpr (TN == 8) col[j] = cbase + (j < 4 ? lane * 4 + j : 128 + lane * 4 + (j - 4));
    else col[j] = cbase + lane * TN + j;
  }
  float acc[4][TN];
#pragma unroll
  for (int j = 0; j < TN; ++j) {
    const float b = active ? m.out_b[col[j]] : 0.0f;
#pragma unroll
    for (int i = 0; i < 4; ++i) acc[i][j] = b;
  }
  for (int32_t c = 0; c < p.nc; ++c, ++g) {
    const uint32_t st = g & 1u;
    mbar_wait(p.bar + st, (g >> 1) & 1u);
    if (active) {
      const uint32_t ws = smem_u32(p.stage[0]) + st * static_cast<uint32_t>(p.bk * m.Vp * 4);
      const int kk_end = min(p.bk, m.J - c * p.bk);
      const float* hp = HL + static_cast<int64_t>(c * p.bk) * kHStride + rg * 4;
#pragma unroll 4
      for (int kk = 0; kk < kk_end; ++kk) {
        const float4 h4 = *reinterpret_cast<const float4*>(hp + kk * kHStride);
        const float hv[4] = {h4.x, h4.y, h4.z, h4.w};
        float wv[TN];
        const uint32_t wr = ws + static_cast<uint32_t>(kk * m.Vp) * 4u;
        if constexpr (TN == 8) {
          const float4 wa = lds128(wr + col[0] * 4u);
          const float4 wb = lds128(wr + col[4] * 4u);
          wv[0] = wa.x; wv[1] = wa.y; wv[2] = wa.z; wv[3] = wa.w;
          wv[4] = wb.x; wv[5] = wb.y; wv[6] = wb.z; wv[7] = wb.w;
        } else if constexpr (TN == 4) {
          const float4 wa = lds128(wr + col[0] * 4u);
          wv[0] = wa.x; wv[1] = wa.y; wv[2] = wa.z; wv[3] = wa.w;
        } else {
          const float2 wa = lds64(wr + col[0] * 4u);
          wv[0] = wa.x; wv[1] = wa.y;
        }
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < TN; ++j)
            acc[i][j] = fadd(acc[i][j], fmul(wv[j], hv[i]));
      }
    }
    __syncthreads();  // every warp is done with this stage
    if (threadIdx.x == 0 && !(p.defer && c + 2 >= p.nc)) wpipe_issue(p, m, g + 2);
  }
  // The last __syncthreads above also retired every read of Hs, so the logits
  // may overwrite it.
  if (active) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int r = rg * 4 + i;
      if (r < R) {
        float* lr = HL + static_cast<int64_t>(r) * m.Vp;
        if constexpr (TN == 8) {
          *reinterpret_cast<float4*>(lr + col[0]) = make_float4(acc[i][0], acc[i][1], acc[i][2], acc[i][3]);
          *reinterpret_cast<float4*>(lr + col[4]) = make_float4(acc[i][4], acc[i][5], acc[i][6], acc[i][7]);
        } else if constexpr (TN == 4) {
          *reinterpret_cast<float4*>(lr + col[0]) = make_float4(acc[i][0], acc[i][1], acc[i][2], acc[i][3]);
        } else {
          *reinterpret_cast<float2*>(lr + col[0]) = make_float2(acc[i][0], acc[i][1]);
        }
      }
    }
  }
  __syncthreads();
}

// One out_w chunk of a work item: NR <= 4 rows x 32*TN columns (lane
// columns col[0..TN)), accumulated into acc[0..NR)[0..TN).
// k steps unrolled per loop trip (2, 6 and 8 measured slower than 4; a
// source-level software-pipelined variant too: DESIGN.md).
#ifndef RNNTG_GEMM_UNROLL
#define RNNTG_GEMM_UNROLL 4
#endif
constexpr int kGemmUnroll = RNNTG_GEMM_UNROLL;
template <int TN, int NR, int HS = kHStride>
__device__ __forceinline__ void gemm_chunk(const ModelView& m, uint32_t ws, const float* hp, int kk_end,
                                           const int* col, float (&acc)[4][8]) {
#pragma unroll kGemmUnroll
  for (int kk = 0; kk < kk_end; ++kk) {
    const float4 h4 = *reinterpret_cast<const float4*>(hp + kk * HS);
    const float hv[4] = {h4.x, h4.y, h4.z, h4.w};
    float wv[TN];
    const uint32_t wr = ws + static_cast<uint32_t>(kk * m.Vp) * 4u;
    const float4 wa = lds128(wr + col[0] * 4u);
    wv[0] = wa.x; wv[1] = wa.y; wv[2] = wa.z; wv[3] = wa.w;
    if constexpr (TN == 8) {
      const float4 wb = lds128(wr + col[4] * 4u);
      wv[4] = wb.x; wv[5] = wb.y; wv[6] = wb.z; wv[7] = wb.w;
    }
#pragma unroll
    for (int i = 0; i < NR; ++i)
#pragma unroll
      for (int j = 0; j < TN; ++j)
        acc[i][j] = fadd(acc[i][j], fmul(wv[j], hv[i]));
  }
}

// C for Vp = 512, balanced over the four SM sub-partitions (a warp's SMSP is
// warp % 4, and the FMUL/FADD stream is issue-bound per SMSP).  R = 4 full +
// rem rows.  Every pair of full row groups gives 4 "heavy" items (4 rows x
// 256 columns, TN = 8) on 4 consecutive warps; an odd full group gives 4
// "light" items (4 rows x 128 columns); the rem-row partial group gives 4
// light items of rem rows — each on 4 consecutive warps, so every SMSP gets
// the same work for any R and no padding row is computed (up to R = 27;
// beyond, the partial group is padded to 4 rows).  A plain 2-items-per-row-
// group split leaves SMSPs 3:3:2:2 loaded at R = 20 (tools/probes/
// gemm_tiling.cu: 1.23e13 vs 1.47e13 MAC/s).
__device__ __forceinline__ void gemm_pass_bal(const ModelView& m, const WPipe& p, uint32_t& g,
                                              float* HL, int R, long long* g_wait_cycles = nullptr) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int full = R >> 2, rem = R & 3;
  if (rem != 0 && 2 * (full & ~1) + 4 * (full & 1) + 4 > kWarps) {  // pad the partial group
    ++full;
    rem = 0;
  }
  const int heavy = 2 * (full & ~1);
  const int lfull = (full & 1) ? 4 : 0;
  int tn = 0, nr = 4, rg = 0, cbase = 0;
  if (warp < heavy) {
    tn = 8;
    rg = warp >> 1;
    cbase = (warp & 1) * 256;
  } else if (warp < heavy + lfull) {
    tn = 4;
    rg = full - 1;
    cbase = (warp - heavy) * 128;
  } else if (rem != 0 && warp < heavy + lfull + 4) {
    tn = 4;
    nr = rem;
    rg = full;
    cbase = (warp - heavy - lfull) * 128;
  }
  int col[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) col[j] = cbase + (j < 4 ? lane * 4 + j : 128 + lane * 4 + (j - 4));
  float acc[4][8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const float b = (tn == 8 || (tn == 4 && j < 4)) ? m.out_b[col[j]] : 0.0f;
#pragma unroll
    for (int i = 0; i < 4; ++i) acc[i][j] = b;
  }
  for (int32_t c = 0; c < p.nc; ++c, ++g) {
    const uint32_t st = g & 1u;
    // Idle warps go straight to the barrier (bar.sync does not issue) rather
    // than spinning on the mbarrier.  Warp 0 always waits: it refills the
    // stage.
    const long long w0 = clock64();
    if (tn != 0 || warp == 0) mbar_wait(p.bar + st, (g >> 1) & 1u);
    if (threadIdx.x == 0 && g_wait_cycles) *g_wait_cycles += clock64() - w0;
    const uint32_t ws = smem_u32(p.stage[0]) + st * static_cast<uint32_t>(p.bk * m.Vp * 4);
    const int kk_end = min(p.bk, m.J - c * p.bk);
    const float* hp = HL + static_cast<int64_t>(c * p.bk) * kHStride + rg * 4;
    if (tn == 8) gemm_chunk<8, 4>(m, ws, hp, kk_end, col, acc);
    else if (tn == 4 && nr == 4) gemm_chunk<4, 4>(m, ws, hp, kk_end, col, acc);
    else if (tn == 4 && nr == 3) gemm_chunk<4, 3>(m, ws, hp, kk_end, col, acc);
    else if (tn == 4 && nr == 2) gemm_chunk<4, 2>(m, ws, hp, kk_end, col, acc);
    else if (tn == 4) gemm_chunk<4, 1>(m, ws, hp, kk_end, col, acc);
    const long long b0 = clock64();
    __syncthreads();  // every warp is done with this stage
    if (threadIdx.x == 0 && g_wait_cycles) g_wait_cycles[1] += clock64() - b0;
    // The refill is issued by the last warp: idle or light for every R, so
    // the issue latency never delays a heavy warp into the next barrier.
    if (threadIdx.x == kDecodeThreads - 32 && !(p.defer && c + 2 >= p.nc)) wpipe_issue(p, m, g + 2);
  }
  // The last __syncthreads above also retired every read of the h tile.
  if (tn != 0) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int r = rg * 4 + i;
      if (r < R) {
        float* lr = HL + static_cast<int64_t>(r) * m.Vp;
        *reinterpret_cast<float4*>(lr + col[0]) = make_float4(acc[i][0], acc[i][1], acc[i][2], acc[i][3]);
        if (tn == 8)
          *reinterpret_cast<float4*>(lr + col[4]) = make_float4(acc[i][4], acc[i][5], acc[i][6], acc[i][7]);
      }
    }
  }
  __syncthreads();
}

// Rows from which the SMSP-balanced tiling is used; below, the uniform
// tilings of gemm_pass (up to 16 equal items of 4 rows x 32*TN columns).
#ifndef RNNTG_BAL_MIN_R
#define RNNTG_BAL_MIN_R 5
#endif
__device__ __forceinline__ void joiner_gemm(const ModelView& m, const WPipe& p,
                                            uint32_t& g, float* HL, int R, long long* wc = nullptr) {
  if (m.Vp == 512 && R >= RNNTG_BAL_MIN_R) {
    gemm_pass_bal(m, p, g, HL, R, wc);
    return;
  }
  const int rg = (R + 3) >> 2;
  const int nb256 = m.Vp >> 8, nb128 = m.Vp >> 7, nb64 = m.Vp >> 6;
  constexpr int W = kDecodeThreads / 32;
  if (rg * nb256 >= 12 || rg * nb128 > W) {
    gemm_pass<8>(m, p, g, HL, R);
  } else if (rg * nb128 >= 12 || rg * nb64 > W) {
    gemm_pass<4>(m, p, g, HL, R);
  } else {
    gemm_pass<2>(m, p, g, HL, R);
  }
}

// h tile for a thread group of nt threads (tid in [0, nt)), k-major stride.
__device__ __forceinline__ void build_h_g(const ModelView& m, const float* pe, const int64_t* row_pe,
                                          const int32_t* row_ctx, int R, float* HL, int hstride,
                                          int tid, int nt, long long* tsplit = nullptr) {
  const int J = m.J;
  const int total = R * J;
  // Pass 1: gather (pe + pd) + j_b with many independent global loads in
  // flight per thread; pass 2: tanhf in place.  Splitting the passes keeps
  // the glibc-tanhf dependency chains from serialising the HBM/L2 latency.
  if ((J & 3) == 0) {
    // 16-byte loads: unit = 4 consecutive i of one row; units are numbered
    // row-fastest, so a warp's k-major h writes (i * hstride + r) hit
    // consecutive banks (column-fastest units were a 16-way conflict).
    const int J4 = J >> 2, units = R * J4;
    for (int base = tid; base < units; base += 4 * nt) {
      float4 a[4], b[4];
      int rr[4], ii[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int x = base + u * nt;
        const bool ok = x < units;
        ii[u] = ok ? (x / R) * 4 : 0;  // row-fastest units: a warp's lanes take
        rr[u] = ok ? x - (ii[u] >> 2) * R : 0;  // consecutive rows -> conflict-free h writes
        a[u] = ok ? *reinterpret_cast<const float4*>(pe + row_pe[rr[u]] * J + ii[u]) : make_float4(0, 0, 0, 0);
        b[u] = ok ? *reinterpret_cast<const float4*>(m.pd + static_cast<int64_t>(row_ctx[rr[u]]) * J + ii[u])
                  : make_float4(0, 0, 0, 0);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (base + u * nt >= units) continue;
        const float* jb = m.j_b + ii[u];
        float* o = HL + ii[u] * hstride + rr[u];
        o[0] = fadd(fadd(a[u].x, b[u].x), jb[0]);
        o[hstride] = fadd(fadd(a[u].y, b[u].y), jb[1]);
        o[2 * hstride] = fadd(fadd(a[u].z, b[u].z), jb[2]);
        o[3 * hstride] = fadd(fadd(a[u].w, b[u].w), jb[3]);
      }
    }
    if (tsplit && tid == 0) tsplit[0] = clock64();
    // Pass 2 over the same units (each thread reads back what it wrote).
    // Four independent branch-free tanhf chains per unit; the rare special
    // inputs are fixed up afterwards so the main paths interleave.
    for (int x = tid; x < units; x += nt) {
      const int i = (x / R) * 4, r = x - (i >> 2) * R;
      float* o = HL + i * hstride + r;
      float v[4], z[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) v[q] = o[q * hstride];
#pragma unroll
      for (int q = 0; q < 4; ++q) z[q] = rnntg_exact::tanhf_main(v[q]);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if (!rnntg_exact::tanhf_main_path(v[q])) z[q] = rnntg_exact::tanhf_glibc(v[q]);
        o[q * hstride] = z[q];
      }
    }
    return;
  }
  for (int base = tid; base < total; base += 4 * nt) {
    float a[4], b[4];
    int rr[4], ii[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int idx = base + u * nt;
      rr[u] = idx < total ? idx / J : 0;
      ii[u] = idx < total ? idx - rr[u] * J : 0;
      a[u] = idx < total ? pe[row_pe[rr[u]] * J + ii[u]] : 0.0f;
      b[u] = idx < total ? m.pd[static_cast<int64_t>(row_ctx[rr[u]]) * J + ii[u]] : 0.0f;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (base + u * nt < total) HL[ii[u] * hstride + rr[u]] = fadd(fadd(a[u], b[u]), m.j_b[ii[u]]);
  }
  // Each thread reads back only the elements it wrote (idx = tid mod nt).
  for (int idx = tid; idx < total; idx += nt) {
    const int r = idx / J, i = idx - r * J;
    float& x = HL[i * hstride + r];
    x = rnntg_exact::tanhf_glibc(x);
  }
}

// B. h[r][i] = tanhf((pe[r][i] + pd[ctx_r][i]) + j_b[i]) into the k-major tile.
__device__ __forceinline__ void build_h(const ModelView& m, const float* pe,
                                        const int64_t* row_pe,
                                        const int32_t* row_ctx, int R,
                                        float* HL, long long* tsplit = nullptr) {
  build_h_g(m, pe, row_pe, row_ctx, R, HL, kHStride, threadIdx.x, kDecodeThreads, tsplit);
  __syncthreads();
}

// Order-preserving uint32 key of a float (larger float -> larger key; every
// float but -NaN maps above 0, so 0 can mean "none") and its inverse.
__device__ __forceinline__ uint32_t ord_key(float f) {
  const uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float ord_val(uint32_t k) {
  return __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k);
}

__device__ __forceinline__ float warp_max_f(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Exact log-softmax normaliser (model.hpp:115-125): sum = Σ_k exp(double(l_k)
// - max) in index order k = 0..V-1 starting from 0.0, lse = double(max) +
// log(sum), with glibc's own exp / log (glibc_f64.h), so lse -- hence every
// log-probability, score and lattice arc -- has the reference's bits.
//
// The exps are evaluated lane-parallel, 32 consecutive k at a time, and
// staged in a per-warp scratch (kLseScr doubles); the sum is then the
// reference's sequential chain, run by every lane on broadcast reads (two
// doubles per LDS.128), so the result is warp-uniform.  NR rows share each
// chunk so their chains interleave.  `etab` is a shared-memory copy of
// glibc's exp table (a divergent index into constant memory serialises).
constexpr int kLseScr = 64;
#ifndef RNNTG_LSE_GROUP
#define RNNTG_LSE_GROUP 8  // double2 scratch loads in flight per group (lse_exact)
#endif  // doubles of scratch per warp (2 rows x 32)

__host__ __device__ inline int hl_floats_of(int J, int Vp) {
  const int a = J * kHStride, b = kRowCap * Vp + kWarps * kLseScr * 2;
  return a > b ? a : b;
}
// The scratch sits behind the logits tile inside the h/logits buffer (the
// k-major h tile is dead once the joiner GEMM has written the logits).
__device__ __forceinline__ double* lse_scratch(float* HL, int Vp) {
  return reinterpret_cast<double*>(HL + kRowCap * Vp) + (threadIdx.x >> 5) * kLseScr;
}
__device__ __forceinline__ void load_exp_table(uint64_t* etab) {
  for (int i = threadIdx.x; i < 256; i += blockDim.x) etab[i] = rnntg_f64::kExpTab[i];
}

// glibc exp, straight-line: the main path for |x| in [2^-54, 2^9) and
// 1 + x below (the max of every log-softmax row gives x = 0); valid unless
// exp_big(x), where glibc's special-case code (exp_t) must be used.
__device__ __forceinline__ bool exp_big(double x) {
  const uint32_t abstop = static_cast<uint32_t>(__double_as_longlong(x) >> 52) & 0x7ffu;
  return abstop > 0x407u;
}
__device__ __forceinline__ double exp_main(double x, const uint64_t* __restrict__ etab) {
  using namespace rnntg_f64;
  const uint32_t abstop = static_cast<uint32_t>(d2u(x) >> 52) & 0x7ffu;
  const double kd0 = xfma(x, 0x1.71547652b82fep+7, 0x1.8p52);
  const uint64_t ki = d2u(kd0);
  const double kd = xsub(kd0, 0x1.8p52);
  double r = xfma(kd, -0x1.62e42fefa0000p-8, x);
  r = xfma(kd, -0x1.cf79abc9e3b3ap-47, r);
  const uint32_t idx = 2u * static_cast<uint32_t>(ki & 0x7f);
  const double tail = u2d(etab[idx]);
  const double scale = u2d(etab[idx + 1] + (ki << 45));
  const double p23 = xfma(r, 0x1.555555555543cp-3, 0x1.ffffffffffdbdp-2);
  const double tr = xadd(r, tail);
  const double r2 = xmul(r, r);
  const double p45 = xfma(r, 0x1.1111167a4d017p-7, 0x1.55555cf172b91p-5);
  const double t1 = xfma(p23, r2, tr);
  const double tmp = xfma(xmul(r2, r2), p45, t1);
  const double y = xfma(scale, tmp, scale);
  return abstop < 0x3c9u ? xadd(x, 1.0) : y;
}
// Any argument (per-thread branch for the rare |x| >= 512).
__device__ __forceinline__ double exp_g(double x, const uint64_t* __restrict__ etab) {
  return exp_big(x) ? rnntg_f64::exp_t(x, etab) : exp_main(x, etab);
}

template <int NR>
__device__ __forceinline__ void lse_exact(const float* const* L, const float* M, int V,
                                          double* __restrict__ scr, const uint64_t* __restrict__ etab,
                                          double* lse) {
  static_assert(NR == 1 || NR == 2, "one or two rows per warp");
  // Lanes [j*LPR, (j+1)*LPR) own row j; a chunk is LPR consecutive k.
  // Software-pipelined over a double-buffered scratch (buffer b at
  // scr + 32 b): iteration c loads chunk c's exps (broadcast within the
  // row's lanes), evaluates chunk c+1's exps while chunk c's chain runs,
  // then stores them into the other buffer.
  constexpr int LPR = 32 / NR;
  constexpr int NV = LPR / 2;
  constexpr int kLseGroup = NV < RNNTG_LSE_GROUP ? NV : RNNTG_LSE_GROUP;
  const int lane = threadIdx.x & 31;
  const int j = lane / LPR, p = lane % LPR;
  const float* Lj = L[0];
  float Mf = M[0];
#pragma unroll
  for (int q = 1; q < NR; ++q)
    if (j == q) {
      Lj = L[q];
      Mf = M[q];
    }
  const double Mj = static_cast<double>(Mf);
  // exp(double(l) - max) of column k (0.0 past the row end); the whole warp
  // calls it: the rare |x| >= 512 fix-up is a warp-uniform branch, so the
  // straight-line main path interleaves with the chain below.
  auto arg = [&](int k) { return k < V ? rnntg_f64::xsub(static_cast<double>(Lj[k]), Mj) : -1.0; };
  auto fix = [&](double x, double y, int k) {
    if (__any_sync(0xffffffffu, exp_big(x)))
      if (exp_big(x)) y = rnntg_f64::exp_t(x, etab);
    return k < V ? y : 0.0;
  };
  {
    const double x = arg(p);
    scr[j * LPR + p] = fix(x, exp_main(x, etab), p);
  }
  __syncwarp();
  double acc = 0.0;
  const int nc = (V + LPR - 1) / LPR;
  for (int c = 0; c < nc; ++c) {
    const double2* src = reinterpret_cast<const double2*>(scr + (c & 1) * 32 + j * LPR);
    const int kn = (c + 1) * LPR + p;
    const double xn = arg(kn);
    double e = exp_main(xn, etab);
    // + 0.0 past the end of the row is exact (acc >= 1 by then).  Groups of
    // 8 loads (16 values) bound the registers this phase adds.
#pragma unroll
    for (int h = 0; h < NV; h += kLseGroup) {
      double2 v[kLseGroup];
#pragma unroll
      for (int q = 0; q < kLseGroup; ++q) v[q] = src[h + q];
#pragma unroll
      for (int q = 0; q < kLseGroup; ++q) acc = rnntg_f64::xadd(rnntg_f64::xadd(acc, v[q].x), v[q].y);
    }
    e = fix(xn, e, kn);
    scr[((c + 1) & 1) * 32 + j * LPR + p] = e;
    __syncwarp();
  }
  const double lj = rnntg_f64::xadd(Mj, rnntg_f64::log(acc));
#pragma unroll
  for (int q = 0; q < NR; ++q) lse[q] = __shfl_sync(0xffffffffu, lj, q * LPR);
}

// Exact normalisers of R rows for the whole CTA, with `E` (>= ecap doubles;
// the weight stages under WPipe::defer) as scratch:
//  (a) row maxima (model.hpp:117-118), one warp per row -> row_m;
//  (b) every exp(double(l_k) - max) of every row into E (row stride S, odd
//      so the chain lanes below hit distinct banks), one column per thread:
//      all the exp work spread over the CTA;
//  (c) one warp runs the reference's sequential sums (model.hpp:119-121),
//      one lane per row, while the other warps do other work.
// The index-order fp64 chain is ~V dependent DADDs per row; here it costs
// one warp V instructions for all rows.  Requires lse_cta_fits(R, V, ecap).
__host__ __device__ inline int lse_cta_stride(int V, int R, int ecap) {
  const int V8 = (V + 7) / 8 * 8;
  return (V8 + 1) * R <= ecap ? V8 + 1 : V8;
}
__host__ __device__ inline bool lse_cta_fits(int R, int V, int ecap) {
  return V <= kDecodeThreads && lse_cta_stride(V, R, ecap) * R <= ecap;
}
// (a) + (b): row maxima, then every exp into E.  Ends with a CTA barrier.
__device__ __forceinline__ void lse_cta_exps(const float* HL, double* E, int ecap, int Vp, int V, int R,
                                             const uint64_t* etab, float* row_m) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int r = warp; r < R; r += kWarps) {
    const float* L = HL + static_cast<int64_t>(r) * Vp;
    float mx = -FLT_MAX;
    for (int k = lane; k < V; k += 32) mx = fmaxf(mx, L[k]);
    mx = warp_max_f(mx);
    if (lane == 0) row_m[r] = mx;
  }
  __syncthreads();
  // Rows are zero-padded to V8 = V rounded up to 8 (+ 0.0 is exact once the
  // sum holds exp(0) = 1), so the chain runs in whole groups of 8.
  const int V8 = (V + 7) / 8 * 8;
  const int S = lse_cta_stride(V, R, ecap);
  const int k = threadIdx.x;  // V8 <= kDecodeThreads
  auto arg = [&](int r) {
    return k < V ? rnntg_f64::xsub(static_cast<double>(HL[static_cast<int64_t>(r) * Vp + k]),
                                   static_cast<double>(row_m[r]))
                 : -1.0;
  };
  for (int r = 0; r < R; r += 2) {  // two rows per trip: independent exp chains interleave
    const int r1 = r + 1 < R ? r + 1 : r;
    const double x0 = arg(r), x1 = arg(r1);
    double y0 = exp_main(x0, etab), y1 = exp_main(x1, etab);
    if (__any_sync(0xffffffffu, exp_big(x0) || exp_big(x1))) {
      if (exp_big(x0)) y0 = rnntg_f64::exp_t(x0, etab);
      if (exp_big(x1)) y1 = rnntg_f64::exp_t(x1, etab);
    }
    if (k < V8) {
      E[r * S + k] = k < V ? y0 : 0.0;
      E[r1 * S + k] = k < V ? y1 : 0.0;
    }
  }
  __syncthreads();
}

// (c) one warp (lane = row): the reference's sequential sums, software-
// pipelined (group q + 1's loads in flight while group q's 8 dependent
// DADDs run), then lse = max + log(sum).
__device__ __forceinline__ void lse_cta_chain(const float* HL, const double* E, int ecap, int Vp, int V, int R,
                                              const float* row_m, double* lse_out, float* l0_out) {
  constexpr int G8 = 8;
  const int lane = threadIdx.x & 31;
  if (lane >= R) return;
  const int V8 = (V + G8 - 1) / G8 * G8;
  const double* e = E + lane * lse_cta_stride(V, R, ecap);
  double acc = 0.0, cur[G8], nxt[G8];
#pragma unroll
  for (int u = 0; u < G8; ++u) cur[u] = e[u];
  for (int q = G8; q < V8; q += G8) {
#pragma unroll
    for (int u = 0; u < G8; ++u) nxt[u] = e[q + u];
#pragma unroll
    for (int u = 0; u < G8; ++u) acc = rnntg_f64::xadd(acc, cur[u]);
#pragma unroll
    for (int u = 0; u < G8; ++u) cur[u] = nxt[u];
  }
#pragma unroll
  for (int u = 0; u < G8; ++u) acc = rnntg_f64::xadd(acc, cur[u]);
  lse_out[lane] = rnntg_f64::xadd(static_cast<double>(row_m[lane]), rnntg_f64::log(acc));
  if (l0_out) l0_out[lane] = HL[static_cast<int64_t>(lane) * Vp];
}

// One row (one warp): float max, then lse_exact.
__device__ __forceinline__ double row_lse(const float* L, int V, double* scr, const uint64_t* etab) {
  const int lane = threadIdx.x & 31;
  float mx = -FLT_MAX;
  for (int k = lane; k < V; k += 32) mx = fmaxf(mx, L[k]);
  const float Ms[1] = {warp_max_f(mx)};
  const float* const Ls[1] = {L};
  double lse[1];
  lse_exact<1>(Ls, Ms, V, scr, etab, lse);
  return lse[0];
}

// log_add (common.hpp:48-54) with glibc's exp / log1p.
__device__ __forceinline__ double log_add_g(double a, double b, const uint64_t* etab) {
  if (a == -INFINITY) return b;
  if (b == -INFINITY) return a;
  const double mx = a > b ? a : b, mn = a > b ? b : a;
  return rnntg_f64::xadd(mx, rnntg_f64::log1p(rnntg_f64::exp_t(rnntg_f64::xsub(mn, mx), etab)));
}

// (logit desc, token asc): the order of a hypothesis' extensions, whose
// scores s + (double(l) - lse) are monotone in the float logit l.
__device__ __forceinline__ bool tok_before(float la, int ka, float lb, int kb) {
  return la > lb || (la == lb && ka < kb);
}


// ---------------------------------------------------------------------------
// bf16 tcgen05 joiner variant (RNNTG_JOINER_BF16; not token-exact).
//
// logits^T = out_w[Vp x J] . h^T[J x N] with out_w as the UMMA A operand
// (M = 128-row tiles of the vocabulary) and the CTA's h rows as B (N = 16 or
// 32): "swap-AB", so a handful of rows still fills 128-row MMA tiles.  out_w
// is pre-arranged in global memory chunk by chunk (kTcBK k-values, no-swizzle
// K-major core matrices) so one cp.async.bulk moves a chunk; kTcStages
// chunks are in flight.  One thread issues the MMAs and commits each stage
// back to its producer through an mbarrier; fp32 accumulators live in TMEM
// (4 M-tiles x 32 columns) and are read with tcgen05.ld by lane quarter.
// ---------------------------------------------------------------------------
constexpr int kTcBK = 16;      // one UMMA K step per chunk
constexpr int kTcStages = 4;   // 4 x 16 KB = the fp32 path's 64 KB stage area
constexpr uint32_t kTmemCols = 128;

struct TcPipe {
  uint32_t stage0;   // smem address of stage 0
  uint64_t* full;    // [kTcStages] chunk landed
  uint64_t* empty;   // [kTcStages] MMAs finished reading the stage
  uint64_t* done;    // frame's MMAs complete
  uint32_t hb;       // smem address of the bf16 h tile (K-major, 32 x J)
  uint32_t tmem;     // TMEM base address
  int32_t nc;        // chunks per frame (J / kTcBK)
};

__device__ __forceinline__ uint32_t tc_stage_bytes(const ModelView& m) {
  return static_cast<uint32_t>(m.Vp) * kTcBK * 2u;
}

__device__ __forceinline__ void tc_issue(const TcPipe& p, const ModelView& m, uint32_t g) {
  const uint32_t c = g % static_cast<uint32_t>(p.nc), st = g % kTcStages;
  const uint32_t bytes = tc_stage_bytes(m);
  fence_proxy_async();
  mbar_expect_tx(p.full + st, bytes);
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          p.stage0 + st * bytes),
      "l"(m.out_w_tc + static_cast<int64_t>(c) * m.Vp * kTcBK), "r"(bytes),
      "r"(static_cast<uint32_t>(__cvta_generic_to_shared(p.full + st)))
      : "memory");
}

// h[r][i] = tanh((pe + pd[ctx]) + j_b) with the hardware tanh, stored bf16
// into the K-major B tile; rows R..N-1 zero.
__device__ __forceinline__ void build_h_tc(const ModelView& m, const float* pe, const int64_t* row_pe,
                                           const int32_t* row_ctx, int R, int N, unsigned char* hb) {
  const int J = m.J;
  for (int idx = threadIdx.x; idx < N * J; idx += kDecodeThreads) {
    const int r = idx / J, i = idx - r * J;
    float h = 0.0f;
    if (r < R) {
      const float x = pe[row_pe[r] * J + i] + m.pd[static_cast<int64_t>(row_ctx[r]) * J + i] + m.j_b[i];
      asm("tanh.approx.f32 %0, %1;" : "=f"(h) : "f"(x));
    }
    *reinterpret_cast<__nv_bfloat16*>(hb + tc::kmajor_off(r, i, J)) = __float2bfloat16_rn(h);
  }
  fence_proxy_async();  // generic-proxy writes -> visible to the tensor core
  __syncthreads();
}

__device__ __forceinline__ void tc_gemm(const ModelView& m, const TcPipe& p, uint32_t& g, uint32_t frame,
                                        float* Ls, int R) {
  const int N = R <= 16 ? 16 : 32;
  const int MT = m.Vp >> 7;
  if (threadIdx.x == 0) {
    const uint32_t idesc = tc::idesc_bf16_f32(128, N);
    const uint32_t sbo_a = (kTcBK / 8) * 128, sbo_b = static_cast<uint32_t>(m.J / 8) * 128;
    const uint32_t bytes = tc_stage_bytes(m);
    for (int c = 0; c < p.nc; ++c, ++g) {
      const uint32_t st = g % kTcStages;
      mbar_wait(p.full + st, (g / kTcStages) & 1u);
      tc::fence_after_sync();
      const uint32_t sa = p.stage0 + st * bytes;
      const uint64_t b = tc::smem_desc(p.hb + static_cast<uint32_t>(c * kTcBK / 8) * 128u, 128u, sbo_b);
      for (int mt = 0; mt < MT; ++mt) {
        const uint64_t a = tc::smem_desc(sa + static_cast<uint32_t>(mt) * 16u * sbo_a, 128u, sbo_a);
        tc::mma_bf16(p.tmem + static_cast<uint32_t>(mt) * 32u, a, b, idesc, c > 0);
      }
      tc::commit(p.empty + st);
      if (g >= 1) {  // the previous chunk's stage is free once its MMAs finished
        const uint32_t gp = g - 1;
        mbar_wait(p.empty + gp % kTcStages, (gp / kTcStages) & 1u);
        tc_issue(p, m, gp + kTcStages);
      }
    }
    tc::commit(p.done);
  }
  mbar_wait(p.done, frame & 1u);
  tc::fence_after_sync();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q = warp & 3;
  for (int mt = warp >> 2; mt < MT; mt += kWarps / 4) {
    const int v = mt * 128 + q * 32 + lane;
    const float bias = m.out_b[v];
    const uint32_t ta = p.tmem + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(mt) * 32u;
    float acc[16];
    tc::ld_32x32b_x16(ta, acc);
#pragma unroll
    for (int r = 0; r < 16; ++r)
      if (r < R) Ls[static_cast<int64_t>(r) * m.Vp + v] = acc[r] + bias;
    if (N > 16) {
      tc::ld_32x32b_x16(ta + 16u, acc);
#pragma unroll
      for (int r = 0; r < 16; ++r)
        if (16 + r < R) Ls[static_cast<int64_t>(16 + r) * m.Vp + v] = acc[r] + bias;
    }
  }
  tc::fence_before_sync();
  __syncthreads();
}

inline size_t smem_common(const ModelView& m, int bk = kBK) {
  const size_t hl = static_cast<size_t>(hl_floats_of(m.J, m.Vp)) * 4;
  return hl + static_cast<size_t>(2) * bk * m.Vp * 4;
}

inline ModelView view_of(const DeviceModel& d) {
  return ModelView{d.V, d.J, d.Vp, d.out_wt, d.out_b, d.j_b, d.pd_table, d.out_w_bf16};
}

}  // namespace dec
}  // namespace rnntg
