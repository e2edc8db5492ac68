// Probe: issue rates of the non-fused fp32 MAC forms on this GPU (scalar
// FMUL+FADD vs packed FMUL2 / FADD2 mixes that ptxas does not contract).
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__device__ __forceinline__ u64 pk(float a, float b){u64 r; asm("mov.b64 %0, {%1,%2};":"=l"(r):"f"(a),"f"(b)); return r;}
__device__ __forceinline__ void upk(u64 r, float&a, float&b){asm("mov.b64 {%0,%1}, %2;":"=f"(a),"=f"(b):"l"(r));}
__device__ __forceinline__ u64 mul2(u64 a, u64 b){u64 r; asm("mul.rn.f32x2 %0, %1, %2;":"=l"(r):"l"(a),"l"(b)); return r;}
__device__ __forceinline__ u64 add2(u64 a, u64 b){u64 r; asm("add.rn.f32x2 %0, %1, %2;":"=l"(r):"l"(a),"l"(b)); return r;}
__device__ __forceinline__ u64 fma2(u64 a, u64 b, u64 c){u64 r; asm("fma.rn.f32x2 %0, %1, %2, %3;":"=l"(r):"l"(a),"l"(b),"l"(c)); return r;}

// MODE 0: scalar FMUL+FADD; 1: FMUL2 + 2xFADD; 2: 2xFMUL + FADD2; 3: FMUL2 only; 4: FADD2 only; 5: FFMA2; 6: FMUL only; 7: FFMA scalar
template <int MODE>
__global__ void __launch_bounds__(512) k(float* out, float seed, int iters) {
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
      for (int j = 0; j < 8; j += 2) {
        float& a0 = acc[i * 8 + j]; float& a1 = acc[i * 8 + j + 1];
        if (MODE == 0) { a0 = __fadd_rn(a0, __fmul_rn(w[i], x[j])); a1 = __fadd_rn(a1, __fmul_rn(w[i], x[j + 1])); }
        else if (MODE == 1) { float p0, p1; upk(mul2(pk(w[i], w[i]), pk(x[j], x[j + 1])), p0, p1); a0 = __fadd_rn(a0, p0); a1 = __fadd_rn(a1, p1); }
        else if (MODE == 2) { u64 r = add2(pk(a0, a1), pk(__fmul_rn(w[i], x[j]), __fmul_rn(w[i], x[j + 1]))); upk(r, a0, a1); }
        else if (MODE == 3) { u64 r = mul2(pk(a0, a1), pk(x[j], x[j + 1])); upk(r, a0, a1); }
        else if (MODE == 4) { u64 r = add2(pk(a0, a1), pk(x[j], x[j + 1])); upk(r, a0, a1); }
        else if (MODE == 5) { u64 r = fma2(pk(w[i], w[i]), pk(x[j], x[j + 1]), pk(a0, a1)); upk(r, a0, a1); }
        else if (MODE == 6) { a0 = __fmul_rn(a0, x[j]); a1 = __fmul_rn(a1, x[j + 1]); }
        else { a0 = __fmaf_rn(w[i], x[j], a0); a1 = __fmaf_rn(w[i], x[j + 1], a1); }
      }
#pragma unroll
    for (int i = 0; i < 4; ++i) w[i] = __fadd_rn(w[i], 1e-7f);
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = __fmul_rn(x[i], 0.9999999f);
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < 32; ++i) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int MODE>
double run(float* out, int sms, int blocks_per_sm) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int iters = 20000; double best = 0;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(a);
    k<MODE><<<sms * blocks_per_sm, 512>>>(out, 1.0f, iters);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms = 0; cudaEventElapsedTime(&ms, a, b);
    const double ops = double(sms) * blocks_per_sm * 512 * iters * 32.0;  // lane element-ops (MAC or single op)
    if (ops / (ms * 1e-3) > best) best = ops / (ms * 1e-3);
  }
  return best;
}
int main() {
  int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* out; cudaMalloc(&out, sizeof(float) * sms * 4 * 512);
  const char* names[] = {"fmul+fadd", "fmul2+2fadd", "2fmul+fadd2", "fmul2_only", "fadd2_only", "ffma2", "fmul_only", "ffma"};
  double r[8];
  r[0] = run<0>(out, sms, 2); r[1] = run<1>(out, sms, 2); r[2] = run<2>(out, sms, 2); r[3] = run<3>(out, sms, 2);
  r[4] = run<4>(out, sms, 2); r[5] = run<5>(out, sms, 2); r[6] = run<6>(out, sms, 2); r[7] = run<7>(out, sms, 2);
  printf("{");
  for (int i = 0; i < 8; ++i) printf("\"%s_elem_per_s\": %.4e%s", names[i], r[i], i < 7 ? ", " : "}\n");
  return 0;
}
