// K1s: strided Gaussian SSIM scores (stride S = 2..8 at compile time, k <= 31, 8/16-bit).
//
// The paper's cheapest Gaussian variant evaluates the window only at anchors (i s, j s):
// O(MNk^2/s^2) for the 2-D kernel, "25x" at s = 5; the reference
// samples anchors the same way (_sliding_weighted_sums on strided slices, src/stats.py:
// 160-163).  K1 computes every output row and column and discards non-anchors, so its
// cost does not fall with s.  K1s runs the separable filter at anchors only:
//   stage  : cp.async 16-byte copies of the next chunk's new input rows (4 images: ref /
//            dist x 2 frames) into a ring of RR rows while the current chunk computes.
//   V pass : thread = input column of the strip; walks the chunk's (G-1) S + k input rows
//            once, forms x, y, x^2 + y^2, xy once per row and adds them into the G anchor
//            rows whose windows contain the row -- k/S FMAs per sample and moment instead
//            of K1's k (the row -> anchor scatter is resolved at compile time from S).
//   H pass : item = one anchor; k-tap horizontal filter of its V values (shared memory),
//            then K1's epilogue (the same sum / difference algebra, 2 C2 carried by the filter).
// Two frames per CTA as packed fp32 pairs (FFMA2), K1's per-tile symmetric sample shift,
// fp64 partial sums per (frame, CTA) in K1's [n][nseg][nstrips][3] layout.  Score-only:
// map launches stay on K1, whose strided maps equal its dense maps at [::s, ::s] exactly.
#pragma once
#include "gauss_ssim.cuh"

namespace ssk {
namespace gk {

constexpr int SG_THREADS = 256;  // input columns per strip (one per V-pass thread)

template <int S>
__host__ __device__ constexpr int sg_g() { return S <= 3 ? 8 : 4; }  // anchor rows per chunk
template <int K, int S>
__host__ __device__ constexpr int sg_nin() { return (sg_g<S>() - 1) * S + K; }  // input rows per chunk
template <int K, int S>
__host__ __device__ constexpr int sg_rr() { return sg_nin<K, S>() + sg_g<S>() * S; }  // ring rows
__host__ __device__ constexpr int sg_gcd(int x, int y) { return y == 0 ? x : sg_gcd(y, x % y); }
// anchor columns per strip: as many as fit 256 input columns, rounded so that every strip
// starts on a 16-byte boundary (cx0 = strip * TWA * S samples) for the cp.async copies
template <int K, int S, int ES>
__host__ __device__ constexpr int sg_twa() {
  return ((SG_THREADS - K) / S + 1) / (16 / sg_gcd(16, S * ES)) * (16 / sg_gcd(16, S * ES));
}

template <int K, typename TIN, int S>
__host__ __device__ constexpr size_t sg_smem() {
  return (size_t)sg_rr<K, S>() * 4 * SG_THREADS * sizeof(TIN) + (size_t)4 * sg_g<S>() * SG_THREADS * 8;
}

template <int K, typename TIN, int S>
__global__ void __launch_bounds__(SG_THREADS, 2) gauss_stride_kernel(const __grid_constant__ GaussArgs a) {
  constexpr int ES = (int)sizeof(TIN);
  static_assert(ES <= 2, "8/16-bit samples only");
  constexpr int G = sg_g<S>();
  constexpr int NIN = sg_nin<K, S>();
  constexpr int RR = sg_rr<K, S>();
  constexpr int TWA = sg_twa<K, S, ES>();
  constexpr int TWI = (TWA - 1) * S + K;      // input columns a full strip reads
  constexpr int RB = SG_THREADS * ES;          // raw row bytes per image (16-byte multiple)
  constexpr int NCH = RB / 16;
  constexpr int NH = (K + 1) / 2;
  extern __shared__ __align__(16) unsigned char smem[];
  unsigned char* raw = smem;                                    // [RR][4][RB]
  u64* vt = reinterpret_cast<u64*>(smem + (size_t)RR * 4 * RB);  // [4][G][SG_THREADS]
  __shared__ double s_red[(SG_THREADS / 32) * 6];
  __shared__ unsigned s_tsum[SG_THREADS / 32][2];

  const int tid = threadIdx.x;
  const int strip = blockIdx.x, seg = blockIdx.y;
  const int f0 = 2 * blockIdx.z;
  const bool has1 = f0 + 1 < a.n;
  const int f1 = has1 ? f0 + 1 : f0;
  const int ac0 = strip * TWA;
  const int cx0 = ac0 * S;
  const int nac = min(TWA, a.gw - ac0);
  const int ar0 = seg * a.seg_rows;
  const int ar1 = min(ar0 + a.seg_rows, a.gh);
  const int nchunks = (ar1 - ar0 + G - 1) / G;
  const int y0 = ar0 * S;                    // first input row of the segment
  const int in_end = (ar1 - 1) * S + K;      // one past its last input row
  const long long fo0 = (long long)f0 * a.frame_pitch_b, fo1 = (long long)f1 * a.frame_pitch_b;
  const int row_bytes_left = (a.w - cx0) * ES;

  // staging: a thread always copies the same 16-byte chunk q of the same image im, of every
  // RPP-th row -- source base, chunk validity and ring offset are fixed per thread, so the
  // copy loop is a pointer increment and a ring-slot wrap (no divisions per item)
  constexpr int IPR = 4 * NCH;              // 16-byte items per input row (4 images)
  static_assert(SG_THREADS % IPR == 0, "whole rows per pass");
  constexpr int RPP = SG_THREADS / IPR;     // rows per pass
  const int st_im = (tid % IPR) / NCH, st_q = tid % NCH, st_r0 = tid / IPR;
  const long long pitch = a.row_pitch_b;
  int st_valid = row_bytes_left - st_q * 16;
  st_valid = st_valid < 0 ? 0 : (st_valid > 16 ? 16 : st_valid);
  const unsigned char* st_base = ((st_im & 2) ? a.dist : a.ref) + ((st_im & 1) ? fo1 : fo0) +
                                 (st_valid ? (long long)cx0 * ES + st_q * 16 : 0);
  unsigned char* st_dst = raw + st_im * RB + st_q * 16;
  auto stage_rows = [&](int r_lo, int r_hi) {  // input rows [r_lo, r_hi) -> ring slots
    r_hi = min(r_hi, in_end);
    int row = r_lo + st_r0;
    int slot = (row - y0) % RR;
    const unsigned char* src = st_base + (long long)row * pitch;
    for (; row < r_hi; row += RPP) {
      cp_async16(st_dst + slot * 4 * RB, src, st_valid);
      src += RPP * pitch;
      slot += RPP;
      if (slot >= RR) slot -= RR;
    }
    cp_async_commit();
  };
  stage_rows(y0, y0 + NIN);

  // per-tile symmetric shifts (as K1): rounded means of (x + y) / 2 and of x - y over the
  // tile's middle row
  __shared__ int s_dsum[SG_THREADS / 32][2];
  {
    const int r = min(((ar0 + ar1) / 2) * S + K / 2, a.h - 1);
    unsigned v0 = 0u, v1 = 0u;
    int w0 = 0, w1 = 0;
    if (tid < TWI && cx0 + tid < a.w) {
      const long long off = (long long)r * a.row_pitch_b + (long long)(cx0 + tid) * ES;
      const unsigned xr0 = raw_uint<TIN>(a.ref + fo0 + off), yd0 = raw_uint<TIN>(a.dist + fo0 + off);
      const unsigned xr1 = raw_uint<TIN>(a.ref + fo1 + off), yd1 = raw_uint<TIN>(a.dist + fo1 + off);
      v0 = xr0 + yd0;
      v1 = xr1 + yd1;
      w0 = (int)xr0 - (int)yd0;
      w1 = (int)xr1 - (int)yd1;
    }
    v0 = __reduce_add_sync(0xffffffffu, v0);
    v1 = __reduce_add_sync(0xffffffffu, v1);
    w0 = __reduce_add_sync(0xffffffffu, w0);
    w1 = __reduce_add_sync(0xffffffffu, w1);
    if ((tid & 31) == 0) {
      s_tsum[tid >> 5][0] = v0;
      s_tsum[tid >> 5][1] = v1;
      s_dsum[tid >> 5][0] = w0;
      s_dsum[tid >> 5][1] = w1;
    }
  }
  __syncthreads();
  unsigned t0 = 0u, t1 = 0u;
  int u0 = 0, u1 = 0;
#pragma unroll
  for (int wi = 0; wi < SG_THREADS / 32; ++wi) {
    t0 += s_tsum[wi][0];
    t1 += s_tsum[wi][1];
    u0 += s_dsum[wi][0];
    u1 += s_dsum[wi][1];
  }
  const unsigned nsh = (unsigned)max(1, min(TWI, a.w - cx0));
  const float sc = a.conv_scale;
  const float cv0 = (float)((t0 + nsh) / (2u * nsh)) * sc, cv1 = (float)((t1 + nsh) / (2u * nsh)) * sc;
  const int d0 = (int)(((unsigned)abs(u0) + nsh / 2u) / nsh), d1 = (int)(((unsigned)abs(u1) + nsh / 2u) / nsh);
  const float dv0 = (float)(u0 < 0 ? -d0 : d0) * sc, dv1 = (float)(u1 < 0 ? -d1 : d1) * sc;
  const float base = -8388608.f * sc;
  const float baseb = -(8388608.f + (float)SD_OFF) * sc;
  const u64 vbias = pk(base - cv0, base - cv1);
  const u64 abias = pk(base - 2.f * cv0, base - 2.f * cv1);  // sum / difference form (gauss_ssim.cuh)
  const u64 bbias = pk(baseb - dv0, baseb - dv1);
  const u64 dshift = pk(dv0, dv1);
  const u64 twoc1_2 = pk(2.f * a.c1, 2.f * a.c1), twoc2_2 = pk(2.f * a.c2, 2.f * a.c2);
  const u64 h2shift = pk(2.f * cv0, 2.f * cv1);
  const u64 scale2 = pk(sc, sc);
  const u64 c1_2 = pk(a.c1, a.c1), c2_2 = pk(a.c2, a.c2);
  const u64 two2 = pk(2.f, 2.f), one2 = pk(a.one, a.one), half2 = pk(0.5f, 0.5f), mhalf2 = pk(-0.5f, -0.5f);
  const bool exact_sq = a.exact_sq != 0;
  const bool full_terms = (a.want & (SSK_WANT_Q | SSK_WANT_L)) != 0;
  u64 w2[NH];
#pragma unroll
  for (int i = 0; i < NH; ++i) w2[i] = pk(a.taps[i], a.taps[i]);

  u64 fq = 0ull, fl = 0ull, fc = 0ull;
  for (int c = 0; c < nchunks; ++c) {
    // the next chunk's new rows go into slots the current chunk does not read (RR >= NIN + G S)
    if (c + 1 < nchunks) {
      stage_rows(y0 + c * G * S + NIN, y0 + (c + 1) * G * S + NIN);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();  // chunk c's rows landed; the previous H pass is done with the V tile
    const int ga = min(G, ar1 - (ar0 + c * G));
    // ---- V pass: thread = input column ----
    if (tid < TWI) {
      u64 acc[4][G];
#pragma unroll
      for (int m = 0; m < 4; ++m)
#pragma unroll
        for (int r = 0; r < G; ++r) acc[m][r] = 0ull;
      const int s0 = (c * G * S) % RR;
      const int wrap = RR - s0;
      const unsigned char* pa = raw + s0 * 4 * RB + tid * ES;
      const unsigned char* pb = pa - RR * 4 * RB;
#pragma unroll
      for (int u = 0; u < NIN; ++u) {
        const unsigned char* rp = (u < wrap ? pa : pb) + u * 4 * RB;
        u64 P[4];
#if SSK_SD
        {
          const unsigned x0 = raw_uint<TIN>(rp), x1 = raw_uint<TIN>(rp + RB);
          const unsigned y0 = raw_uint<TIN>(rp + 2 * RB), y1 = raw_uint<TIN>(rp + 3 * RB);
          P[0] = fma2(pk(__uint_as_float(0x4B000000u + x0 + y0), __uint_as_float(0x4B000000u + x1 + y1)),
                      scale2, abias);
          P[1] = fma2(pk(__uint_as_float((0x4B000000u + SD_OFF) + x0 - y0),
                         __uint_as_float((0x4B000000u + SD_OFF) + x1 - y1)),
                      scale2, bbias);
          P[2] = mul2(P[0], P[0]);
          P[3] = mul2(P[1], P[1]);
        }
#else
        const u64 X = fma2(pk(raw_to_float<TIN>(rp), raw_to_float<TIN>(rp + RB)), scale2, vbias);
        const u64 Y = fma2(pk(raw_to_float<TIN>(rp + 2 * RB), raw_to_float<TIN>(rp + 3 * RB)), scale2, vbias);
        P[0] = X;
        P[1] = Y;
        if constexpr (ES == 1) P[2] = fma2(X, X, mul2(Y, Y));
        else if (exact_sq) P[2] = fma2(X, X, mul2(Y, Y));
        else P[2] = sumsq2(X, Y);
        P[3] = mul2(X, Y);
#endif
#pragma unroll
        for (int r = 0; r < G; ++r) {
          const int i = u - r * S;
          if (i >= 0 && i < K) {
            const u64 wi = w2[i < K - 1 - i ? i : K - 1 - i];
#pragma unroll
            for (int m = 0; m < 4; ++m) acc[m][r] = fma2(wi, P[m], acc[m][r]);
          }
        }
      }
#pragma unroll
      for (int m = 0; m < 4; ++m)
#pragma unroll
        for (int r = 0; r < G; ++r) vt[(m * G + r) * SG_THREADS + tid] = acc[m][r];
    }
    __syncthreads();  // V tile complete
    // ---- H pass + epilogue: item = one anchor ----
    for (int it = tid; it < ga * nac; it += SG_THREADS) {
      const int r = it / nac, j = it - r * nac;
      u64 h[4];
#pragma unroll
      for (int m = 0; m < 4; ++m) {
        const u64* vr = vt + (m * G + r) * SG_THREADS + j * S;
        u64 t = (m == 2) ? (SSK_SD ? twoc2_2 : c2_2) : 0ull;  // the squared-sum moment carries C2 (as K1)
#pragma unroll
        for (int i = 0; i < K; ++i) t = fma2(w2[i < K - 1 - i ? i : K - 1 - i], vr[i], t);
        h[m] = t;
      }
#if SSK_SD
      u64 cs, l, q;
      if (full_terms) {
        sd_terms<true>(h[0], h[1], h[2], h[3], 2.f * a.c2, h2shift, dshift, twoc1_2, cs, l, q);
        fq = fma2(q, one2, fq);
        fl = fma2(l, one2, fl);
      } else {
        sd_terms<false>(h[0], h[1], h[2], h[3], 2.f * a.c2, h2shift, dshift, twoc1_2, cs, l, q);
      }
      fc = fma2(cs, one2, fc);
#else
      const u64 m1 = h[0], m2 = h[1];
      const u64 nm2 = m2 ^ 0x8000000080000000ull;
      const u64 Sm = add2(m1, m2);
      const u64 Dm = add2(m1, nm2);
      const u64 Dq = mul2(Dm, Dm);
      const u64 den2 = maxc_2(fma2(fma2(Sm, Sm, Dq), mhalf2, h[2]), a.c2);
      const u64 cv = fma2(m1, nm2, h[3]);
      const u64 cs = mul2(fma2(two2, cv, c2_2), rcp2(den2));
      fc = fma2(cs, one2, fc);
      if (full_terms) {
        const u64 Su = add2(Sm, h2shift);
        const u64 H = fma2(mul2(Su, Su), half2, c1_2);
        const u64 l = mul2(fma2(Dq, mhalf2, H), rcp2(fma2(Dq, half2, H)));
        fq = fma2(mul2(l, cs), one2, fq);
        fl = fma2(l, one2, fl);
      }
#endif
    }
  }

  double v[6];
  float lo, hi;
  upk(fq, lo, hi);
  v[0] = lo;
  v[3] = hi;
  upk(fl, lo, hi);
  v[1] = lo;
  v[4] = hi;
  upk(fc, lo, hi);
  v[2] = lo;
  v[5] = hi;
#pragma unroll
  for (int i = 0; i < 6; ++i) v[i] = warp_sum(v[i]);
  if ((tid & 31) == 0) {
#pragma unroll
    for (int i = 0; i < 6; ++i) s_red[(tid >> 5) * 6 + i] = v[i];
  }
  __syncthreads();
  if (tid < 6 && (tid < 3 || has1)) {
    double t = 0.0;
#pragma unroll
    for (int wi = 0; wi < SG_THREADS / 32; ++wi) t += s_red[wi * 6 + tid];
    const int fr = tid < 3 ? f0 : f1;
    const long long part = ((long long)fr * gridDim.y + seg) * gridDim.x + strip;
    a.partials[part * 3 + (tid % 3)] = t;
  }
}

template <int K, typename TIN, int S>
int launch_stride_k(const GaussArgs& a, dim3 grid, cudaStream_t st) {
  auto fn = gauss_stride_kernel<K, TIN, S>;
  constexpr size_t smem = sg_smem<K, TIN, S>();
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return SSK_E_CUDA;
  fn<<<grid, SG_THREADS, smem, st>>>(a);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? SSK_OK : SSK_E_CUDA;
}

template <typename TIN, int S>
int launch_stride_t(const GaussArgs& a, dim3 grid, int k, cudaStream_t st) {
  switch (k) {
    case 11: return launch_stride_k<11, TIN, S>(a, grid, st);
#ifndef SSK_K11_ONLY  // (A/B builds: only the 11-tap kernels, a quarter of the compile time)
    case 3: return launch_stride_k<3, TIN, S>(a, grid, st);
    case 5: return launch_stride_k<5, TIN, S>(a, grid, st);
    case 7: return launch_stride_k<7, TIN, S>(a, grid, st);
    case 9: return launch_stride_k<9, TIN, S>(a, grid, st);
    case 13: return launch_stride_k<13, TIN, S>(a, grid, st);
    case 15: return launch_stride_k<15, TIN, S>(a, grid, st);
    case 17: return launch_stride_k<17, TIN, S>(a, grid, st);
    case 19: return launch_stride_k<19, TIN, S>(a, grid, st);
    case 21: return launch_stride_k<21, TIN, S>(a, grid, st);
    case 23: return launch_stride_k<23, TIN, S>(a, grid, st);
    case 25: return launch_stride_k<25, TIN, S>(a, grid, st);
    case 27: return launch_stride_k<27, TIN, S>(a, grid, st);
    case 29: return launch_stride_k<29, TIN, S>(a, grid, st);
    case 31: return launch_stride_k<31, TIN, S>(a, grid, st);
#endif
    default: return SSK_E_SHAPE;
  }
}

template <int S>
int launch_stride_s(const GaussArgs& a, dim3 grid, int k, cudaStream_t st) {
  return a.dtype == SSK_U8 ? launch_stride_t<uint8_t, S>(a, grid, k, st)
                           : launch_stride_t<uint16_t, S>(a, grid, k, st);
}

}  // namespace gk
}  // namespace ssk
