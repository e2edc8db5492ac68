// Probe: device throughput of the glibc-exact tanhf port on joiner-like
// inputs (|x| mostly < 3), 22 values per thread per "frame" as in build_h.
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2211_00484_b200/csrc/exact_math.h"
__global__ void __launch_bounds__(512, 1) k(const float* __restrict__ x, float* out, int frames) {
  __shared__ float s[512 * 24];
  float acc = 0;
  for (int f = 0; f < frames; ++f) {
    for (int i = 0; i < 22; ++i) s[threadIdx.x + 512 * i] = x[(threadIdx.x * 7 + i * 131 + f * 17) & 65535];
    __syncthreads();
    for (int i = 0; i < 22; i += 2) {
      float a = rnntg_exact::tanhf_main(s[threadIdx.x + 512 * i]);
      float b = rnntg_exact::tanhf_main(s[threadIdx.x + 512 * (i + 1)]);
      s[threadIdx.x + 512 * i] = a;
      s[threadIdx.x + 512 * (i + 1)] = b;
    }
    __syncthreads();
    acc += s[(threadIdx.x * 3) % (512 * 22)];
  }
  out[blockIdx.x * 512 + threadIdx.x] = acc;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float h[65536];
  unsigned st = 1;
  for (int i = 0; i < 65536; ++i) {  // ~N(0, 0.8) by sum of uniforms
    float s = 0;
    for (int j = 0; j < 4; ++j) { st = st * 1664525u + 1013904223u; s += (st >> 8) * (1.0f / 16777216.0f) - 0.5f; }
    h[i] = s * 1.4f;
  }
  float *x, *out; cudaMalloc(&x, sizeof(h)); cudaMalloc(&out, sms * 512 * 4);
  cudaMemcpy(x, h, sizeof(h), cudaMemcpyHostToDevice);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int frames = 1000;
  float best = 1e9;
  for (int r = 0; r < 3; ++r) {
    cudaEventRecord(a); k<<<sms, 512>>>(x, out, frames); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); best = fminf(best, ms);
  }
  printf("{\"tanhf_per_s\": %.3e, \"us_per_frame_22x512\": %.3f}\n", double(sms) * frames * 512 * 22 / (best * 1e-3), best * 1e3 / frames);
}
