// Measures the non-fused fp32 multiply+add rate the exact joiner is bound by
// (FMUL then FADD per MAC, as the reference's sequential affine requires),
// beside the FFMA rate, on this GPU.  Prints one JSON line.
//
// Every fp32 pipe instruction of the timed loop is counted: per iteration 32
// MACs (64 FMUL/FADD, or 32 FFMA) plus the 4 FADDs that keep the
// multipliers loop-variant (so ptxas cannot hoist the products).  The
// instruction rate is what the nominal peak (SMs x 128 lanes x clock) bounds.
#include <cstdio>
#include <cuda_runtime.h>

template <bool kFused>
__global__ void __launch_bounds__(512) mac_kernel(float* out, float seed, int iters) {
  float acc[32], w[4], x[8];
#pragma unroll
  for (int i = 0; i < 32; ++i) acc[i] = seed * (threadIdx.x + i);
#pragma unroll
  for (int i = 0; i < 4; ++i) w[i] = seed + i;
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = seed - i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (kFused) acc[i * 8 + j] = __fmaf_rn(w[i], x[j], acc[i * 8 + j]);
        else acc[i * 8 + j] = __fadd_rn(acc[i * 8 + j], __fmul_rn(w[i], x[j]));
      }
#pragma unroll
    for (int i = 0; i < 4; ++i) w[i] = __fadd_rn(w[i], 1e-7f);
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < 32; ++i) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float* out;
  cudaMalloc(&out, sizeof(float) * sms * 4 * 512);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int iters = 20000;
  double res[2];
  for (int f = 0; f < 2; ++f) {
    for (int rep = 0; rep < 4; ++rep) {
      cudaEventRecord(a);
      if (f) mac_kernel<true><<<sms * 2, 512>>>(out, 1.0f, iters);
      else mac_kernel<false><<<sms * 2, 512>>>(out, 1.0f, iters);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms = 0;
      cudaEventElapsedTime(&ms, a, b);
      // fp32 pipe instructions: 64 FMUL/FADD (or 32 FFMA) + 4 FADD per iteration
      const double inst = double(sms) * 2 * 512 * iters * (f ? 36.0 : 68.0);
      res[f] = inst / (ms * 1e-3);
    }
  }
  const double nominal = double(sms) * 128 * clk * 1e3;  // fp32 lane-instructions / s at the attribute clock
  printf("{\"sms\": %d, \"clock_khz_attr\": %d, \"nonfused_fp32_inst_per_s\": %.4e, \"ffma_fp32_inst_per_s\": %.4e, "
         "\"nominal_fp32_inst_per_s\": %.4e, \"nonfused_tflops\": %.3f, \"nonfused_frac_of_nominal\": %.3f, "
         "\"ffma_frac_of_nominal\": %.3f}\n",
         sms, clk, res[0], res[1], nominal, res[0] / 1e12, res[0] / nominal, res[1] / nominal);
  return 0;
}
