// Probe: MAC rate of exact (FMUL then FADD, k in order) joiner-GEMM inner
// loops with h and out_w resident in shared memory, for several register
// tilings.  One CTA per SM (or two for the 256-thread variants), R joiner
// rows x 512 columns x K=512 per "frame", repeated.
#include <cstdio>
#include <cuda_runtime.h>
#define FMUL(a, b) __fmul_rn(a, b)
#define FADD(a, b) __fadd_rn(a, b)
constexpr int Vp = 512, J = 512, KC = 16;  // KC k-rows of out_w resident (reused cyclically)

__device__ __forceinline__ float4 lds128(unsigned a) { float4 v; asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a)); return v; }
__device__ __forceinline__ float lds32(unsigned a) { float v; asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a)); return v; }
__device__ __forceinline__ float2 lds64(unsigned a) { float2 v; asm volatile("ld.shared.v2.f32 {%0,%1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(a)); return v; }

// A: warp item = 4 rows x 256 cols (TN=8), items = (R/4)*2, warps = NT/32
template <int NT>
__global__ void __launch_bounds__(NT, 1) tileA(float* out, int R, int frames) {
  extern __shared__ float sm[];
  float* H = sm;                 // [J][36]
  float* W = sm + J * 36;        // [KC][Vp]
  for (int i = threadIdx.x; i < J * 36; i += NT) H[i] = 0.001f * (i % 97);
  for (int i = threadIdx.x; i < KC * Vp; i += NT) W[i] = 0.002f * (i % 89);
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int items = ((R + 3) / 4) * 2;
  float tot = 0;
  const unsigned hb = (unsigned)__cvta_generic_to_shared(H), wb = (unsigned)__cvta_generic_to_shared(W);
  for (int f = 0; f < frames; ++f) {
    for (int it = warp; it < items; it += NT / 32) {
      const int rg = it / 2, blk = it % 2;
      float acc[4][8];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = 0;
      const int c0 = blk * 256 + lane * 4;
#pragma unroll 4
      for (int k = 0; k < J; ++k) {
        const float4 h = lds128(hb + (k * 36 + rg * 4) * 4);
        const unsigned wr = wb + ((k % KC) * Vp) * 4;
        const float4 wa = lds128(wr + c0 * 4), wb2 = lds128(wr + (c0 + 128) * 4);
        const float hv[4] = {h.x, h.y, h.z, h.w};
        const float wv[8] = {wa.x, wa.y, wa.z, wa.w, wb2.x, wb2.y, wb2.z, wb2.w};
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 8; ++j) acc[i][j] = FADD(acc[i][j], FMUL(wv[j], hv[i]));
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) tot += acc[i][j];
    }
  }
  out[blockIdx.x * NT + threadIdx.x] = tot;
}

// B: warp owns 32*TC columns (lane columns c0 + 32*j ... ), all R rows (NG groups of 4)
template <int NT, int NG, int TC>
__global__ void __launch_bounds__(NT, 512 / NT) tileB(float* out, int frames) {
  extern __shared__ float sm[];
  constexpr int HS = NG * 4 + 4;
  float* H = sm;
  float* W = sm + J * HS;
  for (int i = threadIdx.x; i < J * HS; i += NT) H[i] = 0.001f * (i % 97);
  for (int i = threadIdx.x; i < KC * Vp; i += NT) W[i] = 0.002f * (i % 89);
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int NW = NT / 32;
  float tot = 0;
  const unsigned hb = (unsigned)__cvta_generic_to_shared(H), wb = (unsigned)__cvta_generic_to_shared(W);
  // columns: TC per lane, contiguous per lane (TC=2 -> lds64; TC=4 -> lds128)
  const int cpw = Vp / NW;  // columns per warp
  for (int f = 0; f < frames; ++f) {
    for (int cb = warp * cpw; cb < warp * cpw + cpw; cb += 32 * TC) {
      float acc[NG * 4][TC];
#pragma unroll
      for (int i = 0; i < NG * 4; ++i)
#pragma unroll
        for (int j = 0; j < TC; ++j) acc[i][j] = 0;
      const int c0 = cb + lane * TC;
#pragma unroll 2
      for (int k = 0; k < J; ++k) {
        const unsigned wr = wb + ((k % KC) * Vp + c0) * 4;
        float wv[TC];
        if (TC == 1) wv[0] = lds32(wr);
        if (TC == 2) { float2 t = lds64(wr); wv[0] = t.x; wv[TC - 1] = t.y; }
        if (TC == 4) { float4 t = lds128(wr); wv[0] = t.x; wv[1 % TC] = t.y; wv[2 % TC] = t.z; wv[3 % TC] = t.w; }
#pragma unroll
        for (int q = 0; q < NG; ++q) {
          const float4 h = lds128(hb + (k * HS + q * 4) * 4);
          const float hv[4] = {h.x, h.y, h.z, h.w};
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < TC; ++j) acc[q * 4 + i][j] = FADD(acc[q * 4 + i][j], FMUL(wv[j], hv[i]));
        }
      }
#pragma unroll
      for (int i = 0; i < NG * 4; ++i)
#pragma unroll
        for (int j = 0; j < TC; ++j) tot += acc[i][j];
    }
  }
  out[blockIdx.x * NT + threadIdx.x] = tot;
}


// P: tiling A + the real out_w pipeline (cp.async.bulk from global, KS stages
// of 16 k-rows, mbarrier full; release by __syncthreads (SYNC=1) or by a
// last-arriver counter (SYNC=0)).
__device__ __forceinline__ void mbar_init(unsigned b, unsigned c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(b), "r"(c)); }
__device__ __forceinline__ void mbar_wait(unsigned b, unsigned ph) {
  asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(b), "r"(ph) : "memory"); }
__device__ __forceinline__ void issue(unsigned dst, const float* src, unsigned bytes, unsigned bar) {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst), "l"(src), "r"(bytes), "r"(bar) : "memory");
}
template <int KS, int SYNC>
__global__ void __launch_bounds__(512, 1) tileP(float* out, const float* __restrict__ wg, int R, int frames) {
  extern __shared__ __align__(128) float sm[];
  float* H = sm;                       // [J][36]
  float* W = sm + J * 36;              // [KS][16][Vp]
  __shared__ __align__(8) unsigned long long bar[KS];
  __shared__ unsigned cnt[KS];
  for (int i = threadIdx.x; i < J * 36; i += 512) H[i] = 0.001f * (i % 97);
  const unsigned wb = (unsigned)__cvta_generic_to_shared(W), hb = (unsigned)__cvta_generic_to_shared(H);
  const unsigned sb = 16 * Vp * 4;
  if (threadIdx.x == 0) {
    for (int s = 0; s < KS; ++s) { mbar_init((unsigned)__cvta_generic_to_shared(&bar[s]), 1); cnt[s] = 0; }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0)
    for (int s = 0; s < KS; ++s) issue(wb + s * sb, wg + (s % 32) * 16 * Vp, sb, (unsigned)__cvta_generic_to_shared(&bar[s]));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int items = ((R + 3) / 4) * 2;
  const bool active = warp < items;
  const int rg = warp / 2, blk = warp % 2;
  const int c0 = blk * 256 + lane * 4;
  float tot = 0;
  unsigned g = 0;
  for (int f = 0; f < frames; ++f) {
    float acc[4][8];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[i][j] = 0;
    for (int c = 0; c < 32; ++c, ++g) {
      const unsigned st = g % KS;
      mbar_wait((unsigned)__cvta_generic_to_shared(&bar[st]), (g / KS) & 1);
      if (active) {
        const unsigned ws = wb + st * sb;
#pragma unroll 4
        for (int kk = 0; kk < 16; ++kk) {
          const float4 h = lds128(hb + ((c * 16 + kk) * 36 + rg * 4) * 4);
          const unsigned wr = ws + kk * Vp * 4;
          const float4 wa = lds128(wr + c0 * 4), wb2 = lds128(wr + (c0 + 128) * 4);
          const float hv[4] = {h.x, h.y, h.z, h.w};
          const float wv[8] = {wa.x, wa.y, wa.z, wa.w, wb2.x, wb2.y, wb2.z, wb2.w};
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 8; ++j) acc[i][j] = FADD(acc[i][j], FMUL(wv[j], hv[i]));
        }
      }
      if (SYNC) {
        __syncthreads();
        if (threadIdx.x == 0) issue(wb + st * sb, wg + ((g + KS) % 32) * 16 * Vp, sb, (unsigned)__cvta_generic_to_shared(&bar[st]));
      } else {
        __syncwarp();
        if (lane == 0) {
          __threadfence_block();
          if (atomicAdd(&cnt[st], 1u) % 16 == 15) {
            __threadfence_block();
            issue(wb + st * sb, wg + ((g + KS) % 32) * 16 * Vp, sb, (unsigned)__cvta_generic_to_shared(&bar[st]));
          }
        }
      }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j) tot += acc[i][j];
  }
  if (threadIdx.x == 0)
    for (unsigned x = g; x < g + KS; ++x) mbar_wait((unsigned)__cvta_generic_to_shared(&bar[x % KS]), (x / KS) & 1);
  out[blockIdx.x * 512 + threadIdx.x] = tot;
}

template <typename K>
double timeit(K kern, int grid, int nt, size_t smem, double macs, float* out, int frames) {
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  double best = 0;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(a);
    kern<<<grid, nt, smem>>>(out, frames);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    best = fmax(best, macs / (ms * 1e-3));
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("err %s\n", cudaGetErrorString(e));
  return best;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* out; cudaMalloc(&out, 148 * 2 * 512 * 4 * 4);
  const int frames = 40;
  setvbuf(stdout, NULL, _IONBF, 0);
  printf("{");
  for (int R : {8, 12, 16, 20, 24, 28, 32}) {
    const double macs = double(sms) * frames * R * Vp * J;
    auto k = [](float* o, int f) {};
    (void)k;
    cudaFuncSetAttribute(tileA<512>, cudaFuncAttributeMaxDynamicSharedMemorySize, (J * 36 + KC * Vp) * 4);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    double best = 0;
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(a);
      tileA<512><<<sms, 512, (J * 36 + KC * Vp) * 4>>>(out, R, frames);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      best = fmax(best, macs / (ms * 1e-3));
    }
    printf("\"A512_R%d\": %.3e, ", R, best); fflush(stdout); { cudaError_t e = cudaGetLastError(); if (e) { printf("err %s\n", cudaGetErrorString(e)); return 1; } }
  }
  // B variants: per SM rows = NG*4 per CTA x CTAs/SM
  {
    double m;
    m = timeit(tileB<512, 6, 1>, sms, 512, (J * 28 + KC * Vp) * 4, double(sms) * frames * 24 * Vp * J, out, frames);
    printf("\"B512_NG6_TC1(R24)\": %.3e, ", m);
    m = timeit(tileB<512, 8, 1>, sms, 512, (J * 36 + KC * Vp) * 4, double(sms) * frames * 32 * Vp * J, out, frames);
    printf("\"B512_NG8_TC1(R32)\": %.3e, ", m);
    m = timeit(tileB<256, 3, 2>, 2 * sms, 256, (J * 16 + KC * Vp) * 4, double(2 * sms) * frames * 12 * Vp * J, out, frames);
    printf("\"B256x2_NG3_TC2(R12/CTA)\": %.3e, ", m);
    m = timeit(tileB<256, 4, 2>, 2 * sms, 256, (J * 20 + KC * Vp) * 4, double(2 * sms) * frames * 16 * Vp * J, out, frames);
    printf("\"B256x2_NG4_TC2(R16/CTA)\": %.3e", m);
  }
  {
    float* wg; cudaMalloc(&wg, J * Vp * 4);
    { float* hw = (float*)malloc(J * Vp * 4); unsigned st = 7; for (int i = 0; i < J * Vp; ++i) { st = st * 1664525u + 1013904223u; hw[i] = ((st >> 8) * (1.0f / 16777216.0f) - 0.5f) * 0.088f; }
      cudaMemcpy(wg, hw, J * Vp * 4, cudaMemcpyHostToDevice); free(hw); }
    for (int v = 0; v < 4; ++v) {
      for (int R : {16, 24}) {
        const int KS = v < 2 ? 2 : 3;
        const size_t smem = (J * 36 + KS * 16 * Vp) * 4;
        auto kern = v == 0 ? tileP<2, 1> : v == 1 ? tileP<2, 0> : v == 2 ? tileP<3, 1> : tileP<3, 0>;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        double best = 0;
        for (int rep = 0; rep < 3; ++rep) {
          cudaEventRecord(a);
          kern<<<sms, 512, smem>>>(out, wg, R, frames);
          cudaEventRecord(b); cudaEventSynchronize(b);
          float ms; cudaEventElapsedTime(&ms, a, b);
          best = fmax(best, double(sms) * frames * R * Vp * J / (ms * 1e-3));
        }
        cudaError_t e = cudaGetLastError();
        printf(", \"P_KS%d_SYNC%d_R%d\": %.3e%s", KS, v % 2 == 0, R, best, e ? cudaGetErrorString(e) : "");
      }
    }
  }
  printf("}\n");
  return 0;
}
