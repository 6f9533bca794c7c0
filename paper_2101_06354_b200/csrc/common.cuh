// Shared device helpers for the SSIM engine kernels (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/ssimk.h"

namespace ssk {

// ---------------------------------------------------------------------------
// cp.async (LDGSTS) 16-byte staging with zero fill of the bytes past `valid`.
// ---------------------------------------------------------------------------
// Synchronisation stress build (-DSSK_SYNC_STRESS, tools/sync_stress.py): at every hand-off
// point of the barrier / mbarrier rings, one warp in four sleeps a pseudo-random 0-1 us,
// reshuffling the producer/consumer interleavings; a race shows up as results that are no
// longer bit-identical to the production build's.  Compiled out otherwise.
#ifdef SSK_SYNC_STRESS
__device__ __forceinline__ void ssk_jitter(unsigned site) {
  unsigned h = (unsigned)clock() ^ (blockIdx.x * 0x9E3779B1u) ^ (blockIdx.y * 0x7FEB352Du) ^
               ((threadIdx.x >> 5) * 0x85EBCA77u) ^ (site * 0xC2B2AE3Du);
  h ^= h >> 15;
  h *= 0x2C1B3C6Du;
  h ^= h >> 12;
  if ((h & 3u) == 0u) __nanosleep((h >> 4) & 1023u);
}
#define SSK_JITTER(site) ::ssk::ssk_jitter(site)
#else
#define SSK_JITTER(site) ((void)0)
#endif

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int valid_bytes) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem),
               "r"(valid_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// ---------------------------------------------------------------------------
// Exact integer -> float for values < 2^23: splice the bits into the mantissa
// of 2^23 (one PRMT/LOP on the ALU pipe); the caller folds the -2^23 bias into
// the FFMA that applies scale and shift.
// ---------------------------------------------------------------------------
__device__ __forceinline__ float u8_as_biased(uint32_t word, int byte) {
  // result bytes: [b, 0, 0, 0x4B] -> 0x4B0000bb == 8388608 + b
  return __int_as_float(__byte_perm(word, 0x4Bu, 0x4550u | byte));
}
__device__ __forceinline__ float u16_as_biased(uint32_t word, int half) {
  return __int_as_float(
      __byte_perm(word, 0x4Bu, half ? 0x4532u : 0x4510u));  // [lo, hi, 0, 0x4B]
}

// ---------------------------------------------------------------------------
// FP64 warp reduction and block reduction of NV values (deterministic order).
// ---------------------------------------------------------------------------
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <int NV, int NWARPS>
__device__ __forceinline__ void block_sum_store(double (&v)[NV], double* scratch /*NWARPS*NV*/,
                                                double* out /*NV*/) {
  const int tid = threadIdx.x + threadIdx.y * blockDim.x;  // 1-D or 2-D blocks
  const int lane = tid & 31, warp = tid >> 5;
#pragma unroll
  for (int i = 0; i < NV; ++i) v[i] = warp_sum(v[i]);
  if (lane == 0) {
#pragma unroll
    for (int i = 0; i < NV; ++i) scratch[warp * NV + i] = v[i];
  }
  __syncthreads();
  if (tid < NV) {
    double s = 0.0;
#pragma unroll
    for (int wi = 0; wi < NWARPS; ++wi) s += scratch[wi * NV + tid];
    out[tid] = s;
  }
}

// Reciprocal from the MUFU seed refined by two Newton steps (~1 ulp).
__device__ __forceinline__ double rcp_nr(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}

// Score-only epilogue of the rect-window kernels (no maps and no integer sums
// requested).  The window moments stay exact integers -- k^2 var = k^2 Q - S^2
// (>= 0) and k^2 cov = k^2 P - S1 S2 in 64-bit, exactly representable in
// float64 below 2^53 (BoxArgs::fast_ok) -- so no cancellation is left, and
//   l  = (2 S1 S2 + C1')           / (S1^2 + S2^2 + C1')
//   cs = (2 (k^2 P - S1 S2) + C2') / ((k^2 Q1 - S1^2) + (k^2 Q2 - S2^2) + C2'),
// C' = C k^4 4^scale, each with one rounded add and a Newton reciprocal:
// scores agree with the reference's float64 expression to ~1e-15.  Maps keep
// the reference's own operation order (bit-identical) and never come here.
template <typename Args, bool Q2>
__device__ __forceinline__ void box_fast_terms(const Args& a, unsigned long long s1, unsigned long long s2,
                                               unsigned long long q1, unsigned long long q2, unsigned long long p,
                                               double& sq, double& sl, double& scs, double& sq2) {
  const unsigned long long A = (unsigned long long)a.area_i;
  const unsigned long long p11 = s1 * s1, p22 = s2 * s2, p12 = s1 * s2;
  const unsigned long long v12 = (A * q1 - p11) + (A * q2 - p22);
  const long long cv2 = 2 * ((long long)(A * p) - (long long)p12);
  const double l = __dmul_rn(__dadd_rn((double)(2 * p12), a.c1d), rcp_nr(__dadd_rn((double)(p11 + p22), a.c1d)));
  const double cs = __dmul_rn(__dadd_rn((double)cv2, a.c2d), rcp_nr(__dadd_rn((double)v12, a.c2d)));
  const double q = __dmul_rn(l, cs);
  sq += q;
  sl += l;
  scs += cs;
  if constexpr (Q2) sq2 += __dmul_rn(q, q);
}

// Per-CTA sum of q^2 for SSK_WANT_Q2 (CoV / MD(2) pooling fused into the rect kernels);
// uniform branch, so the block barrier inside is safe.
template <typename Args, int NWARPS>
__device__ __forceinline__ void store_q2(const Args& a, double sq2, double* scratch /*NWARPS*/, long long part) {
  if (!a.partials2) return;
  double v[1] = {sq2};
  block_sum_store<1, NWARPS>(v, scratch, a.partials2 + part * 3);
}

// Number of kernels launched by this library (bench.py's gpu_launches claim).
void note_launch(int count = 1);

inline int esize_of(int dtype) {
  switch (dtype) {
    case SSK_U8: return 1;
    case SSK_U16: return 2;
    case SSK_U32: return 4;
    case SSK_F32: return 4;
    case SSK_F64: return 8;
    default: return 0;
  }
}

inline int grid_extent(int n, int k, int s) { return (n - k) / s + 1; }

}  // namespace ssk
