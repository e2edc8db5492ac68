// The SMSP-balanced exact joiner GEMM (decode_common.cuh gemm_pass_bal) as
// ONE out-of-line function in its own translation unit (-rdc): every decode
// kernel calls the same machine code, so the FMUL/FADD loop's schedule no
// longer depends on the register pressure of the kernel around it.  Inlined,
// ptxas scheduled the loop differently in every kernel — in the fused-pe beam
// kernel with each FADD right behind its FMUL (~16% slower GEMM), and small
// unrelated edits to the beam kernel moved it by 2% (tools/fadd_dist.py).
//
// Arithmetic and item layout are gemm_pass_bal's (sequential k per
// accumulator, fl(acc + fl(w*h))); the h tile and the logits are addressed
// as shared-space offsets with explicit ld/st.shared (a generic pointer
// across the call would otherwise turn every h load into a generic LD).
//
// Opt-in experiment, not in the default build (tools/build_rdc_variant.sh):
// the isolated loop is well spaced (FMUL->FADD distance ~20) yet measured
// slower in the single-launch beam kernel (103.0 vs 98.0 ms at B = 1024,
// T = 1000) while lifting the fused-pe kernel (135 -> 126 ms).
#include "decode_common.cuh"

namespace rnntg {
namespace dec {
namespace {

__device__ __forceinline__ void sts128(uint32_t a, float x, float y, float z, float w) {
  asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(a), "f"(x), "f"(y), "f"(z), "f"(w)
               : "memory");
}

template <int TN, int NR>
__device__ __forceinline__ void chunk_s(uint32_t ws, uint32_t hs, int kk_end, uint32_t vp4, uint32_t c0,
                                        uint32_t c4, float (&acc)[4][8]) {
#pragma unroll 4
  for (int kk = 0; kk < kk_end; ++kk) {
    const float4 h4 = lds128(hs + static_cast<uint32_t>(kk) * (kHStride * 4u));
    const float hv[4] = {h4.x, h4.y, h4.z, h4.w};
    float wv[TN];
    const uint32_t wr = ws + static_cast<uint32_t>(kk) * vp4;
    const float4 wa = lds128(wr + c0);
    wv[0] = wa.x; wv[1] = wa.y; wv[2] = wa.z; wv[3] = wa.w;
    if constexpr (TN == 8) {
      const float4 wb = lds128(wr + c4);
      wv[4] = wb.x; wv[5] = wb.y; wv[6] = wb.z; wv[7] = wb.w;
    }
#pragma unroll
    for (int i = 0; i < NR; ++i)
#pragma unroll
      for (int j = 0; j < TN; ++j) acc[i][j] = fadd(acc[i][j], fmul(wv[j], hv[i]));
  }
}

}  // namespace

__device__ __noinline__ uint32_t gemm_bal_x(const WPipe p, uint32_t g, uint32_t hl, int R, int Vp,
                                            const float* __restrict__ bias, int K, int nc,
                                            long long* wc) {
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
  const int col0 = cbase + lane * 4, col4 = cbase + 128 + lane * 4;
  float acc[4][8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const float b = (tn == 8 || (tn == 4 && j < 4)) ? bias[j < 4 ? col0 + j : col4 + j - 4] : 0.0f;
#pragma unroll
    for (int i = 0; i < 4; ++i) acc[i][j] = b;
  }
  const uint32_t vp4 = static_cast<uint32_t>(Vp) * 4u;
  const uint32_t stage0 = smem_u32(p.stage[0]);
  const uint32_t stage_bytes = static_cast<uint32_t>(p.bk) * vp4;
  for (int32_t c = 0; c < nc; ++c, ++g) {
    const uint32_t st = g & 1u;
    const long long w0 = clock64();
    if (tn != 0 || warp == 0) mbar_wait(p.bar + st, (g >> 1) & 1u);
    if (threadIdx.x == 0 && wc) *wc += clock64() - w0;
    const uint32_t ws = stage0 + st * stage_bytes;
    const int kk_end = min(p.bk, K - c * p.bk);
    const uint32_t hs = hl + static_cast<uint32_t>(c * p.bk * kHStride + rg * 4) * 4u;
    if (tn == 8) chunk_s<8, 4>(ws, hs, kk_end, vp4, col0 * 4u, col4 * 4u, acc);
    else if (tn == 4 && nr == 4) chunk_s<4, 4>(ws, hs, kk_end, vp4, col0 * 4u, col4 * 4u, acc);
    else if (tn == 4 && nr == 3) chunk_s<4, 3>(ws, hs, kk_end, vp4, col0 * 4u, col4 * 4u, acc);
    else if (tn == 4 && nr == 2) chunk_s<4, 2>(ws, hs, kk_end, vp4, col0 * 4u, col4 * 4u, acc);
    else if (tn == 4) chunk_s<4, 1>(ws, hs, kk_end, vp4, col0 * 4u, col4 * 4u, acc);
    const long long b0 = clock64();
    __syncthreads();  // every warp is done with this stage
    if (threadIdx.x == 0 && wc) wc[1] += clock64() - b0;
    if (threadIdx.x == kDecodeThreads - 32) wpipe_issue(p, ModelView{}, g + 2);
  }
  // The last __syncthreads above also retired every read of the h tile.
  if (tn != 0) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int r = rg * 4 + i;
      if (r < R) {
        const uint32_t lr = hl + static_cast<uint32_t>(r) * vp4;
        sts128(lr + col0 * 4u, acc[i][0], acc[i][1], acc[i][2], acc[i][3]);
        if (tn == 8) sts128(lr + col4 * 4u, acc[i][4], acc[i][5], acc[i][6], acc[i][7]);
      }
    }
  }
  __syncthreads();
  return g;
}

}  // namespace dec
}  // namespace rnntg
