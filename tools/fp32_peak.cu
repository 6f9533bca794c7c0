// FP32 pipe microbenchmark for B200 (sm_100a): FFMA register / immediate / c-bank forms and FFMA2.
#include <cstdio>
#include <cuda_runtime.h>
struct W { float w[4]; };
template <int MODE>
__global__ void __launch_bounds__(256) k_ffma(float* out, int iters, float a0, W cw) {
  float acc[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) acc[i] = threadIdx.x * 1e-6f + i;
  float b = a0 + threadIdx.x * 1e-7f;
  float c = a0 * 0.5f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 8; ++r) {
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        if (MODE == 0) acc[i] = fmaf(acc[i], b, c);          // 3-register form
        else if (MODE == 1) acc[i] = fmaf(acc[i], 0.9999f, 1e-5f);  // immediate
        else acc[i] = fmaf(acc[i], cw.w[i & 3], cw.w[(i + 1) & 3]); // constant-bank
      }
    }
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += acc[i];
  if (s == 1234.5f) out[0] = s;
}
__global__ void __launch_bounds__(256) k_ffma2(float* out, int iters, float a0) {
  unsigned long long acc[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) { float2 v = make_float2(threadIdx.x * 1e-6f + i, i * 0.5f); acc[i] = *reinterpret_cast<unsigned long long*>(&v); }
  float2 bb = make_float2(a0, a0 * 0.99f), cc = make_float2(a0 * 0.5f, a0 * 0.25f);
  unsigned long long b = *reinterpret_cast<unsigned long long*>(&bb), c = *reinterpret_cast<unsigned long long*>(&cc);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 8; ++r) {
#pragma unroll
      for (int i = 0; i < 8; ++i) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(acc[i]) : "l"(b), "l"(c));
    }
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) { float2 v = *reinterpret_cast<float2*>(&acc[i]); s += v.x + v.y; }
  if (s == 1234.5f) out[0] = s;
}
int main() {
  float* d; cudaMalloc(&d, 4);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  W cw = {{0.999f, 1e-5f, 0.998f, 2e-5f}};
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 20000; const int blocks = sms * 8, threads = 256;
  for (int mode = 0; mode < 4; ++mode) {
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(e0);
      if (mode == 0) k_ffma<0><<<blocks, threads>>>(d, iters, 1.0001f, cw);
      if (mode == 1) k_ffma<1><<<blocks, threads>>>(d, iters, 1.0001f, cw);
      if (mode == 2) k_ffma<2><<<blocks, threads>>>(d, iters, 1.0001f, cw);
      if (mode == 3) k_ffma2<<<blocks, threads>>>(d, iters, 1.0001f);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double fmas = (double)blocks * threads * iters * 8 * 16;  // FFMA2 does 8 x 2 lanes
      const char* nm[] = {"ffma_reg", "ffma_imm", "ffma_cbank", "ffma2_reg"};
      if (rep == 2) printf("%s: %.2f TFLOP/s (%.3f ms)\n", nm[mode], 2 * fmas / ms / 1e9, ms);
    }
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
