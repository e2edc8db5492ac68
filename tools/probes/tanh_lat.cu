// Latency of the exact tanhf (exact_math.h) per thread, 1..4 in flight:
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -std=c++17 \
//   -Ipaper_2211_00484_b200/csrc tools/probes/tanh_lat.cu -o tools/probes/bin/tanh_lat
#include <cstdio>
#include <cuda_runtime.h>
#include "exact_math.h"
template <int U, bool FIX>
__global__ void k(const float* in, float* out, long long* cyc) {
  __shared__ float buf[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) buf[i] = in[i];
  __syncthreads();
  float v[U], z[U];
  long long t0 = clock64();
#pragma unroll
  for (int u = 0; u < U; ++u) v[u] = buf[threadIdx.x + u * 256];
#pragma unroll
  for (int u = 0; u < U; ++u) z[u] = rnntg_exact::tanhf_main(v[u]);
  if (FIX) {
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (!rnntg_exact::tanhf_main_path(v[u])) z[u] = rnntg_exact::tanhf_glibc(v[u]);
  }
#pragma unroll
  for (int u = 0; u < U; ++u) buf[threadIdx.x + u * 256] = z[u];
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  out[threadIdx.x] = buf[threadIdx.x];
}
template <int U, bool FIX>
void run(const float* d_in, float* d_out, long long* d_c) {
  k<U, FIX><<<1, 256>>>(d_in, d_out, d_c);
  k<U, FIX><<<1, 256>>>(d_in, d_out, d_c);
  long long h;
  cudaMemcpy(&h, d_c, 8, cudaMemcpyDeviceToHost);
  printf("U=%d fix=%d: %lld cycles\n", U, (int)FIX, h);
}
int main() {
  float h_in[1024];
  for (int i = 0; i < 1024; ++i) h_in[i] = (i % 97) * 0.05f - 2.4f;
  float *d_in, *d_out; long long* d_c;
  cudaMalloc(&d_in, 4096); cudaMalloc(&d_out, 4096); cudaMalloc(&d_c, 8);
  cudaMemcpy(d_in, h_in, 4096, cudaMemcpyHostToDevice);
  run<1, false>(d_in, d_out, d_c); run<1, true>(d_in, d_out, d_c);
  run<2, false>(d_in, d_out, d_c); run<2, true>(d_in, d_out, d_c);
  run<4, false>(d_in, d_out, d_c); run<4, true>(d_in, d_out, d_c);
}
