// Kernel-level parity entry points: an independent straight-line joiner row
// kernel and the exhaustive tanhf sweep.  Not on the decode hot path.
#include "exact_math.h"
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

}  // namespace

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
