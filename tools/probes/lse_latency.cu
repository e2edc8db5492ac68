// Probe: dependent DADD latency, LDS->DADD chain, and lse_exact<NR> cycles per
// row on this GPU (one CTA of 16 warps, every warp reducing NR rows, as in
// the beam kernel's row-reduction phase).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -fmad=false \
//        -I paper_2211_00484_b200/csrc -o tools/probes/lse_latency tools/probes/lse_latency.cu
#include <cstdio>
#include <cuda_runtime.h>

#include "decode_common.cuh"

using namespace rnntg::dec;

__global__ void dadd_chain(double* out, double s, int n, long long* cyc) {
  double a = s + threadIdx.x;
  const long long t0 = clock64();
  for (int i = 0; i < n; ++i) a = __dadd_rn(a, 1e-3);
  const long long t1 = clock64();
  out[threadIdx.x] = a;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

template <int NR>
__global__ void __launch_bounds__(512, 1) lse_rows(const float* logits, int V, int reps, double* out, long long* cyc) {
  extern __shared__ __align__(128) unsigned char smem[];
  float* HL = reinterpret_cast<float*>(smem);
  uint64_t* etab = reinterpret_cast<uint64_t*>(HL + hl_floats_of(512, 512));
  for (int i = threadIdx.x; i < kRowCap * 512; i += blockDim.x) HL[i] = logits[i % (kRowCap * 512)];
  load_exp_table(etab);
  __syncthreads();
  const int warp = threadIdx.x >> 5;
  const float* L[NR];
  float M[NR];
  for (int j = 0; j < NR; ++j) {
    L[j] = HL + (warp + 16 * j) * 512;
    float mx = -1e30f;
    for (int k = 0; k < V; ++k) mx = fmaxf(mx, L[j][k]);
    M[j] = mx;
  }
  double acc = 0;
  __syncthreads();
  const long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    double lse[NR];
    lse_exact<NR>(L, M, V, lse_scratch(HL, 512), etab, lse);
    acc += lse[0];
    __syncwarp();
  }
  const long long t1 = clock64();
  out[threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

int main() {
  double* d_out;
  long long* d_cyc;
  float* d_log;
  cudaMalloc(&d_out, 4096 * 8);
  cudaMalloc(&d_cyc, 8);
  const int n = kRowCap * 512;
  float* h = new float[n];
  unsigned s = 1;
  for (int i = 0; i < n; ++i) {
    s = s * 1664525u + 1013904223u;
    h[i] = ((s >> 8) & 0xffff) / 4096.0f - 8.0f;
  }
  cudaMalloc(&d_log, n * 4);
  cudaMemcpy(d_log, h, n * 4, cudaMemcpyHostToDevice);
  long long c;
  dadd_chain<<<1, 32>>>(d_out, 1.0, 4096, d_cyc);
  cudaMemcpy(&c, d_cyc, 8, cudaMemcpyDeviceToHost);
  printf("{\"dadd_latency_cycles\": %.2f", c / 4096.0);
  const size_t smem = hl_floats_of(512, 512) * 4 + 2048;
  cudaFuncSetAttribute(lse_rows<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(lse_rows<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int reps = 64;
  lse_rows<1><<<1, 512, smem>>>(d_log, 500, reps, d_out, d_cyc);
  cudaMemcpy(&c, d_cyc, 8, cudaMemcpyDeviceToHost);
  printf(", \"lse1_cycles_per_row\": %.1f", c / double(reps));
  lse_rows<2><<<1, 512, smem>>>(d_log, 500, reps, d_out, d_cyc);
  cudaMemcpy(&c, d_cyc, 8, cudaMemcpyDeviceToHost);
  printf(", \"lse2_cycles_per_2rows\": %.1f", c / double(reps));
  printf(", \"err\": \"%s\"}\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
