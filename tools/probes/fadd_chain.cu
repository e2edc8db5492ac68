// FADD chain latency probe (dependent FADD; with an independent FMUL; with LDS.128 operands).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false tools/probes/fadd_chain.cu -o tools/probes/bin/fadd_mb
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k1(float* out, long long* cyc, float a, int n, int mode) {
  __shared__ float4 buf[16 * 130];
  for (int i = threadIdx.x; i < 16 * 130; i += blockDim.x) buf[i] = make_float4(i * 1e-3f, 1, 2, 3);
  __syncthreads();
  float acc = a, x = a * 0.5f;
  long long t0 = clock64();
  if (mode == 0) {
#pragma unroll 16
    for (int i = 0; i < n; ++i) acc = __fadd_rn(acc, x);
  } else if (mode == 1) {
#pragma unroll 16
    for (int i = 0; i < n; ++i) acc = __fadd_rn(acc, __fmul_rn(x, (float)i));
  } else if (mode == 2) {
    const float4* w = buf + (threadIdx.x % 16) * 129;
#pragma unroll 4
    for (int i = 0; i < n / 4; ++i) {
      float4 v = w[i & 127];
      acc = __fadd_rn(acc, v.x); acc = __fadd_rn(acc, v.y); acc = __fadd_rn(acc, v.z); acc = __fadd_rn(acc, v.w);
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  out[threadIdx.x] = acc;
}
int main() {
  float* o; long long* c; cudaMalloc(&o, 4096); cudaMalloc(&c, 8);
  for (int mode = 0; mode < 3; ++mode) for (int nt : {32, 64, 256}) {
    k1<<<1, nt>>>(o, c, 1.0f, 4096, mode); k1<<<1, nt>>>(o, c, 1.0f, 4096, mode);
    long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("mode %d threads %d: %.2f cycles/op\n", mode, nt, h / 4096.0);
  }
}
