// FFMA2 issue-rate microbenchmark (sm_100a): operand forms and co-issue with ALU / LDS work,
// at the persistent K1's occupancy (one 512-thread CTA per SM = 4 warps per scheduler).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ffma2_forms ffma2_forms.cu
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__device__ __forceinline__ u64 pk(float lo, float hi) { u64 r; asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi)); return r; }
__device__ __forceinline__ u64 fma2(u64 a, u64 b, u64 c) { u64 d; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c)); return d; }

// MODE 0: w uniform (UR.F32 broadcast form expected)   1: w per-thread vector registers
// MODE 2: mode 0 + one LOP3 per FFMA2                   3: mode 0 + one LDS.64 per 4 FFMA2
// MODE 4: mode 1 + one LDS.64 per 4 FFMA2               5: mode 0 + LOP3 per FFMA2 + LDS.64 per 4
template <int MODE, int NACC>
__global__ void __launch_bounds__(512, 1) k(float* out, int iters, float w0, float w1, float w2, float w3) {
  __shared__ u64 sh[1024];
  for (int i = threadIdx.x; i < 1024; i += 512) sh[i] = pk(i * 1e-3f, i * 2e-3f);
  __syncthreads();
  u64 acc[NACC];
#pragma unroll
  for (int i = 0; i < NACC; ++i) acc[i] = pk(threadIdx.x * 1e-6f + i, i * 0.5f);
  const float t = (MODE == 1 || MODE == 4) ? threadIdx.x * 1e-9f : 0.f;
  __shared__ float sw[4];
  if (threadIdx.x == 0) { sw[0] = w0; sw[1] = w1; sw[2] = w2; sw[3] = w3; }
  __syncthreads();
  u64 w[4];
  if (MODE == 6) {  // scalar broadcast from a per-thread vector register (R.F32 form)
    w[0] = pk(w0 + threadIdx.x * 1e-9f, w0 + threadIdx.x * 1e-9f); w[1] = pk(w1 + threadIdx.x * 1e-9f, w1 + threadIdx.x * 1e-9f);
    w[2] = pk(w2 + threadIdx.x * 1e-9f, w2 + threadIdx.x * 1e-9f); w[3] = pk(w3 + threadIdx.x * 1e-9f, w3 + threadIdx.x * 1e-9f);
  } else if (MODE == 1 || MODE == 4) {  // full 64-bit vector operand
    w[0] = pk(w0 + t, w0 + 2 * t); w[1] = pk(w1 + t, w1 + 2 * t); w[2] = pk(w2 + t, w2 + 2 * t); w[3] = pk(w3 + t, w3 + 2 * t);
  } else {  // uniform (as K1: taps read from shared memory at uniform addresses)
    w[0] = pk(w0, w0); w[1] = pk(w1, w1); w[2] = pk(w2, w2); w[3] = pk(w3, w3);
  }
  u64 v[4] = {pk(0.5f + threadIdx.x, 1.f), pk(0.25f, threadIdx.x), pk(1.5f, 2.f + threadIdx.x), pk(threadIdx.x, 3.f)};
  unsigned x = threadIdx.x * 2654435761u, y = 0x9e3779b9u;
  const u64* sp = sh + (threadIdx.x & 511);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
#pragma unroll
      for (int i = 0; i < NACC; ++i) {
        acc[i] = fma2(w[(i + r) & 3], v[i & 3], acc[i]);
        if (MODE == 2 || MODE == 5) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x) : "r"(y), "r"(it));
        if ((MODE == 3 || MODE == 4 || MODE == 5) && (i & 3) == 3) {
          u64 l; asm volatile("ld.shared.b64 %0, [%1];" : "=l"(l) : "l"(sp + ((i + r * 16) & 255)));
          v[(i >> 2) & 3] = l;
        }
      }
    }
  }
  float s = (float)x;
#pragma unroll
  for (int i = 0; i < NACC; ++i) { float lo, hi; asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(acc[i])); s += lo + hi; }
  if (s == 1234.5f) out[0] = s;
}
template <int MODE, int NACC>
void run(const char* name, float* d, int sms) {
  const int iters = 4000;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float best = 1e9f;
  for (int rep = 0; rep < 4; ++rep) {
    cudaEventRecord(e0);
    k<MODE, NACC><<<sms, 512>>>(d, iters, 0.9991f, 0.9992f, 0.9993f, 0.9994f);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    if (rep && ms < best) best = ms;
  }
  const double ffma2 = (double)sms * 16 * iters * 4 * NACC;  // warp instructions
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const double cyc = best * 1e-3 * clk * 1e3;
  printf("%-34s nacc %2d: %.3f ms, %.2f TFLOP/s, %.2f cycles per FFMA2 per scheduler\n", name, NACC, best,
         ffma2 * 32 * 4 / best / 1e9, cyc / (ffma2 / sms / 4));
}
int main() {
  float* d; cudaMalloc(&d, 4);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<0, 16>("uniform w", d, sms);
  run<0, 8>("uniform w", d, sms);
  run<0, 4>("uniform w", d, sms);
  run<1, 16>("vector w", d, sms);
  run<1, 8>("vector w", d, sms);
  run<2, 16>("uniform w + LOP3/FFMA2", d, sms);
  run<3, 16>("uniform w + LDS.64/4", d, sms);
  run<4, 16>("vector w + LDS.64/4", d, sms);
  run<5, 16>("uniform w + LOP3 + LDS.64/4", d, sms);
  run<6, 16>("R.F32 broadcast w", d, sms);
  run<6, 8>("R.F32 broadcast w", d, sms);
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
