// Issue rate of independent fp32 FADD / FMUL / FADD+FMUL streams per SM
// sub-partition (16 warps, 8 independent chains per thread, -fmad=false).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false tools/probes/fp32_rate.cu -o tools/probes/bin/fp32_rate
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void k(float* out, long long* cyc, float s, int n) {
  float a[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) a[j] = threadIdx.x * 0.001f + j;
  const float b = s * 0.5f;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (MODE == 0) a[j] = __fadd_rn(a[j], b);
      if (MODE == 1) a[j] = __fmul_rn(a[j], b);
      if (MODE == 2) a[j] = __fadd_rn(__fmul_rn(a[j], b), s);
      if (MODE == 3) a[j] = __fmaf_rn(a[j], b, s);
    }
  }
  __syncthreads();
  long long t1 = clock64();
  float r = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) r += a[j];
  out[threadIdx.x] = r;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
template <int MODE>
void run(const char* name, int per) {
  float* o; long long* c; cudaMalloc(&o, 4096 * 4); cudaMalloc(&c, 8);
  const int n = 4096;
  k<MODE><<<1, 512>>>(o, c, 1.0001f, n);
  k<MODE><<<1, 512>>>(o, c, 1.0001f, n);
  long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  const double warp_instr_per_smsp = 16.0 / 4 * n * 8 * per;
  printf("%-10s cycles %lld  -> %.2f cycles per warp-instruction per SMSP\n", name, h, h / warp_instr_per_smsp);
}
int main() {
  run<0>("FADD", 1);
  run<1>("FMUL", 1);
  run<2>("FMUL+FADD", 2);
  run<3>("FFMA", 1);
}
