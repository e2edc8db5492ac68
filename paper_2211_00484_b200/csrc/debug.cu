// Kernel-level parity entry points: an independent straight-line joiner row
// kernel and the exhaustive tanhf sweep.  Not on the decode hot path.
#include "decode_common.cuh"
#include "exact_math.h"
#include "glibc_f64.h"
#include "internal.cuh"

namespace rnntg {
namespace {

using rnntg_exact::fadd;
using rnntg_exact::fmul;

// One CTA per row: h = tanhf((pe + pd[ctx]) + j_b) in smem, then each thread
// walks one logit's k sum in order (joiner_logits_from_proj,
// model.hpp:284-292).
__global__ void joiner_rows_kernel(int32_t V, int32_t J,
                                   const float* __restrict__ out_wt, int32_t Vp,
                                   const float* __restrict__ out_b,
                                   const float* __restrict__ j_b,
                                   const float* __restrict__ pd_table,
                                   const float* __restrict__ pe,
                                   const int32_t* __restrict__ ctxs,
                                   float* __restrict__ logits) {
  __shared__ float h[kMaxJoiner];
  const int r = blockIdx.x;
  const float* per = pe + static_cast<int64_t>(r) * J;
  const float* pdr = pd_table + static_cast<int64_t>(ctxs[r]) * J;
  for (int i = threadIdx.x; i < J; i += blockDim.x)
    h[i] = rnntg_exact::tanhf_glibc(fadd(fadd(per[i], pdr[i]), j_b[i]));
  __syncthreads();
  for (int n = threadIdx.x; n < V; n += blockDim.x) {
    float acc = out_b[n];
    for (int k = 0; k < J; ++k) acc = fadd(acc, fmul(out_wt[static_cast<int64_t>(k) * Vp + n], h[k]));
    logits[static_cast<int64_t>(r) * V + n] = acc;
  }
}

__device__ __forceinline__ unsigned long long mix(unsigned long long x) {
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdull;
  x ^= x >> 33;
  x *= 0xc4ceb9fe1a85ec53ull;
  x ^= x >> 33;
  return x;
}

// Order-independent chunk hash: sum over i of mix((i << 32) | bits(tanhf(i))).
// NaN outputs are canonicalised to 0x7fc00000 (glibc and the port may
// propagate different NaN payloads; tanhf(NaN) is NaN either way).
__global__ void tanhf_hash_kernel(uint32_t first_chunk,
                                  unsigned long long* __restrict__ hashes) {
  const uint32_t chunk = first_chunk + blockIdx.y;
  const uint32_t base = chunk << 24;
  unsigned long long acc = 0;
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < (1u << 24);
       j += gridDim.x * blockDim.x) {
    const uint32_t u = base + j;
    const float y = rnntg_exact::tanhf_glibc(__uint_as_float(u));
    uint32_t bits = __float_as_uint(y);
    if ((bits & 0x7fffffffu) > 0x7f800000u) bits = 0x7fc00000u;
    acc += mix((static_cast<unsigned long long>(u) << 32) | bits);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(&hashes[blockIdx.y], acc);
}

// One warp per row: the decoders' exact log-softmax normaliser (row_lse:
// index-order sum with glibc exp / log).
__global__ void log_softmax_rows_kernel(const float* __restrict__ logits, int32_t n, int32_t V,
                                        double* __restrict__ lse) {
  __shared__ uint64_t etab[256];
  __shared__ __align__(16) double scr[4 * dec::kLseScr];
  dec::load_exp_table(etab);
  __syncthreads();
  const int warp = threadIdx.x >> 5;
  for (int r = blockIdx.x * 4 + warp; r < n; r += gridDim.x * 4) {
    const double v = dec::row_lse(logits + static_cast<int64_t>(r) * V, V, scr + warp * dec::kLseScr, etab);
    if ((threadIdx.x & 31) == 0) lse[r] = v;
  }
}

// glibc exp / log / log1p ports over x[i] (op 0 / 1 / 2; op 3: exp_g, the
// decoders' branch-light exp).
__global__ void f64_math_kernel(int32_t op, const double* __restrict__ x, int64_t n, double* __restrict__ y) {
  __shared__ uint64_t etab[256];
  dec::load_exp_table(etab);
  __syncthreads();
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const double v = x[i];
    y[i] = op == 0 ? rnntg_f64::exp(v) : op == 1 ? rnntg_f64::log(v) : op == 2 ? rnntg_f64::log1p(v)
                                                                                 : dec::exp_g(v, etab);
  }
}

}  // namespace

cudaError_t launch_log_softmax_rows(const float* logits, int32_t n, int32_t V, double* lse, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  log_softmax_rows_kernel<<<(n + 3) / 4, 128, 0, s>>>(logits, n, V, lse);
  return cudaGetLastError();
}

cudaError_t launch_f64_math(int32_t op, const double* x, int64_t n, double* y, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  f64_math_kernel<<<296, 256, 0, s>>>(op, x, n, y);
  return cudaGetLastError();
}

cudaError_t launch_joiner_rows_exact(const DeviceModel& m, const float* pe,
                                     const int32_t* ctxs, int32_t n,
                                     float* logits, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  joiner_rows_kernel<<<n, 256, 0, s>>>(m.V, m.J, m.out_wt, m.Vp, m.out_b, m.j_b,
                                       m.pd_table, pe, ctxs, logits);
  return cudaGetLastError();
}

cudaError_t launch_tanhf_hash(int32_t first_chunk, int32_t num_chunks,
                              unsigned long long* d_hashes, cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(d_hashes, 0, sizeof(unsigned long long) * num_chunks, s);
  if (e != cudaSuccess) return e;
  dim3 grid(256, num_chunks);
  tanhf_hash_kernel<<<grid, 256, 0, s>>>(static_cast<uint32_t>(first_chunk), d_hashes);
  return cudaGetLastError();
}

}  // namespace rnntg
