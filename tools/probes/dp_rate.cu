// Probe: fp64 DFMA rate and exp(double) throughput on this GPU.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void __launch_bounds__(512, 1) dfma(double* out, double s, int it) {
  double a[8];
  for (int i = 0; i < 8; ++i) a[i] = s * (threadIdx.x + i);
  for (int k = 0; k < it; ++k)
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fma(a[i], 0.999999, 1e-9);
  double t = 0;
  for (int i = 0; i < 8; ++i) t += a[i];
  out[blockIdx.x * 512 + threadIdx.x] = t;
}
__global__ void __launch_bounds__(512, 1) dexp(double* out, float s, int it) {
  double acc = 0;
  float x = -s * (threadIdx.x & 63);
  for (int k = 0; k < it; ++k) {
#pragma unroll
    for (int i = 0; i < 8; ++i) acc += exp((double)(x - 0.01f * i) - 1.0);
    x = x * 0.9999f;
  }
  out[blockIdx.x * 512 + threadIdx.x] = acc;
}
__global__ void __launch_bounds__(512, 1) fexp(double* out, float s, int it) {
  float acc = 0;
  float x = -s * (threadIdx.x & 63);
  for (int k = 0; k < it; ++k) {
#pragma unroll
    for (int i = 0; i < 8; ++i) acc += __expf(x - 0.01f * i);
    x = x * 0.9999f;
  }
  out[blockIdx.x * 512 + threadIdx.x] = acc;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* o; cudaMalloc(&o, sms * 512 * 8);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  float ms;
  const int it = 4000;
  dfma<<<sms, 512>>>(o, 1.0, it);
  cudaEventRecord(a); dfma<<<sms, 512>>>(o, 1.0, it); cudaEventRecord(b); cudaEventSynchronize(b);
  cudaEventElapsedTime(&ms, a, b);
  const double n = double(sms) * 512 * it * 8;
  printf("{\"dfma_per_s\": %.3e, ", n / (ms * 1e-3));
  dexp<<<sms, 512>>>(o, 0.01f, it);
  cudaEventRecord(a); dexp<<<sms, 512>>>(o, 0.01f, it); cudaEventRecord(b); cudaEventSynchronize(b);
  cudaEventElapsedTime(&ms, a, b);
  printf("\"exp_f64_per_s\": %.3e, ", n / (ms * 1e-3));
  fexp<<<sms, 512>>>(o, 0.01f, it);
  cudaEventRecord(a); fexp<<<sms, 512>>>(o, 0.01f, it); cudaEventRecord(b); cudaEventSynchronize(b);
  cudaEventElapsedTime(&ms, a, b);
  printf("\"expf_fast_per_s\": %.3e}\n", n / (ms * 1e-3));
}
