// K1g: Gaussian windows wider than 31 taps (sigma > 5 at the default size 2*ceil(3 sigma)+1).
//
// Replaces, for those windows, the same reference chain as K1 (gauss_ssim.cuh):
//   gaussian_kernel(sigma, k)   (src/stats.py:30-44; any odd k >= 3, src/config.py:55-56)
//   _sliding_weighted_sums x5   (src/stats.py:155-164)
//   stats_from_sums(area = 1)   (src/stats.py:185-202)
//   term_maps_from_stats        (src/ssim.py:31-46) and the mean pooling (src/ssim.py:55-65)
//
// Also the map API's kernel for every Gaussian window (SSK_MAP_F64: ssim_map and
// local_statistics return the reference's float64 maps, so they are computed in fp64).
// Wide windows are rare (the paper's and the reference's default is sigma 1.5 -> 11 taps),
// so this kernel is generic in K instead of templated: taps live in shared memory and the
// whole computation runs in fp64 -- the reference's own precision, so no shift or
// cancellation handling is needed however dark, flat or wide the window is (fp32 error
// grows with K; B200's fp64 pipe runs at half the fp32 rate, which is ample for this path).
//
// CTA = 256 threads = a strip of TW = 64 output columns x a segment of output rows, one
// frame.  Per chunk of TH = 8 output rows:
//   V pass : thread = input column (TW + K - 1 of them); walks the TH + K - 1 input rows
//            once (coalesced global loads, L1/L2 resident across neighbouring strips) and
//            scatters each row into the TH x 5 vertical accumulators it contributes to;
//            the five moments x, y, x^2, y^2, xy go to shared memory.
//   H pass : thread = (row, column) pair of outputs; K-tap horizontal filter from shared
//            memory, the reference's epilogue in its own operation order (IEEE products
//            and sums, never contracted), optional map stores, fp64 sums.
//   reduce : warp shuffles + shared memory -> one fp64 partial per (frame, CTA), the same
//            [n][nseg][nstrips][3] layout K1 writes, folded by the same fixed-order kernel.
// Strided grids evaluate anchors only in the H pass; V rows are computed for the whole
// chunk (bit-identical values at anchors, so stride s equals dense[::s, ::s] exactly).
#include "common.cuh"
#include "kernels.h"

namespace ssk {
namespace {

constexpr int GG_THREADS = 256;
constexpr int GG_TW = 64;  // output columns per strip
constexpr int GG_TH = 8;   // output rows per chunk

__device__ __forceinline__ double load_sample(const unsigned char* base, long long off, int dtype, double scale) {
  switch (dtype) {
    case SSK_U8: return (double)base[off] * scale;
    case SSK_U16: return (double)reinterpret_cast<const unsigned short*>(base)[off] * scale;
    case SSK_U32: return (double)reinterpret_cast<const unsigned*>(base)[off] * scale;
    default: return (double)reinterpret_cast<const float*>(base)[off];
  }
}

__global__ void __launch_bounds__(GG_THREADS) gauss_generic_kernel(const __grid_constant__ GaussGenericArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int K = a.k;
  const int twc = GG_TW + K - 1;
  double* s_taps = reinterpret_cast<double*>(smem);
  double* s_v = s_taps + ((K + 1) & ~1);      // [5][GG_TH][twc]
  __shared__ double s_red[GG_THREADS / 32][3];

  const int tid = threadIdx.x;
  const int strip = blockIdx.x, seg = blockIdx.y, frame = blockIdx.z;
  const int x0 = strip * GG_TW;                // first output (= first input) column
  const int y_begin = seg * a.seg_rows;
  const int y_end = min(a.ho, y_begin + a.seg_rows);
  for (int i = tid; i < K; i += GG_THREADS) s_taps[i] = a.taps[i];

  const unsigned char* ref = a.ref + (long long)frame * a.frame_pitch_b;
  const unsigned char* dst = a.dist + (long long)frame * a.frame_pitch_b;
  const long long rp = a.row_pitch_b / a.esize;  // elements
  const bool terms = (a.want & SSK_MAP_TERMS) != 0;
  const bool stats = (a.want & SSK_MAP_STATS) != 0;
  double sq = 0.0, sl = 0.0, scs = 0.0;
  __syncthreads();

  for (int r0 = y_begin; r0 < y_end; r0 += GG_TH) {
    // ---- V pass ----
    SSK_JITTER(400);
    for (int c = tid; c < twc; c += GG_THREADS) {
      const int gc = x0 + c;
      double acc[5][GG_TH];
#pragma unroll
      for (int m = 0; m < 5; ++m)
#pragma unroll
        for (int r = 0; r < GG_TH; ++r) acc[m][r] = 0.0;
      if (gc < a.w) {
        const int nin = GG_TH + K - 1;
        for (int i = 0; i < nin; ++i) {
          const int gr = r0 + i;
          if (gr >= a.h) break;
          const long long off = (long long)gr * rp + gc;
          const double x = load_sample(ref, off, a.dtype, a.scale);
          const double y = load_sample(dst, off, a.dtype, a.scale);
          const double xx = __dmul_rn(x, x), yy = __dmul_rn(y, y), xy = __dmul_rn(x, y);
#pragma unroll
          for (int r = 0; r < GG_TH; ++r) {
            const int t = i - r;
            if (t >= 0 && t < K) {
              const double w = s_taps[t];
              acc[0][r] = fma(w, x, acc[0][r]);
              acc[1][r] = fma(w, y, acc[1][r]);
              acc[2][r] = fma(w, xx, acc[2][r]);
              acc[3][r] = fma(w, yy, acc[3][r]);
              acc[4][r] = fma(w, xy, acc[4][r]);
            }
          }
        }
      }
#pragma unroll
      for (int m = 0; m < 5; ++m)
#pragma unroll
        for (int r = 0; r < GG_TH; ++r) s_v[(m * GG_TH + r) * twc + c] = acc[m][r];
    }
    __syncthreads();
    SSK_JITTER(401);
    // ---- H pass + epilogue ----
    for (int o = tid; o < GG_TH * GG_TW; o += GG_THREADS) {
      const int r = o / GG_TW, j = o % GG_TW;
      const int orow = r0 + r, ocol = x0 + j;
      if (orow >= y_end || ocol >= a.wo || orow % a.stride || ocol % a.stride) continue;
      double m5[5];
#pragma unroll
      for (int m = 0; m < 5; ++m) {
        const double* row = s_v + (m * GG_TH + r) * twc + j;
        double h = 0.0;
        for (int t = 0; t < K; ++t) h = fma(s_taps[t], row[t], h);
        m5[m] = h;
      }
      // stats_from_sums (area = 1) and term_maps_from_stats, in the reference's order
      const double mu1 = m5[0], mu2 = m5[1];
      const double mu12 = __dmul_rn(mu1, mu2);
      const double var1 = fmax(__dsub_rn(m5[2], __dmul_rn(mu1, mu1)), 0.0);
      const double var2 = fmax(__dsub_rn(m5[3], __dmul_rn(mu2, mu2)), 0.0);
      const double cov = __dsub_rn(m5[4], mu12);
      const double l = __ddiv_rn(__dadd_rn(__dmul_rn(2.0, mu12), a.c1),
                                 __dadd_rn(__dadd_rn(__dmul_rn(mu1, mu1), __dmul_rn(mu2, mu2)), a.c1));
      const double cs = __ddiv_rn(__dadd_rn(__dmul_rn(2.0, cov), a.c2),
                                  __dadd_rn(__dadd_rn(var1, var2), a.c2));
      const double q = __dmul_rn(l, cs);
      sq += q;
      sl += l;
      scs += cs;
      if (terms || stats) {
        const long long idx = (long long)frame * a.map_frame + (long long)(orow / a.stride) * a.gw + ocol / a.stride;
        const double vals[5] = {terms ? l : mu1, terms ? cs : mu2, terms ? q : var1, var2, cov};
        const int np = terms ? 3 : 5;
        for (int pl = 0; pl < np; ++pl) {
          if (a.map_f64) reinterpret_cast<double*>(a.maps)[idx + pl * a.map_plane] = vals[pl];
          else reinterpret_cast<float*>(a.maps)[idx + pl * a.map_plane] = (float)vals[pl];
        }
      }
    }
    __syncthreads();  // s_v is rewritten by the next chunk
  }

  double v[3] = {sq, sl, scs};
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v[i] += __shfl_down_sync(0xffffffffu, v[i], o);
  if ((tid & 31) == 0)
#pragma unroll
    for (int i = 0; i < 3; ++i) s_red[tid >> 5][i] = v[i];
  __syncthreads();
  if (tid < 3) {
    double t = 0.0;
#pragma unroll
    for (int wi = 0; wi < GG_THREADS / 32; ++wi) t += s_red[wi][tid];
    const long long part = ((long long)frame * gridDim.y + seg) * gridDim.x + strip;
    a.partials[part * 3 + tid] = t;
  }
}

}  // namespace

size_t gauss_generic_smem(int k) {
  return (size_t)((k + 1) & ~1) * sizeof(double) + (size_t)5 * GG_TH * (GG_TW + k - 1) * sizeof(double);
}

int gauss_generic_grid(int ho, int wo, int n, int seg_rows, dim3* grid) {
  const long long nstrips = (wo + GG_TW - 1) / GG_TW;
  const long long nseg = (ho + seg_rows - 1) / seg_rows;
  if (nseg > 65535 || n > 65535) return SSK_E_ARG;
  *grid = dim3((unsigned)nstrips, (unsigned)nseg, (unsigned)n);
  return SSK_OK;
}

int launch_gauss_generic(const GaussGenericArgs& a, dim3 grid, cudaStream_t st) {
  if (a.k < 3 || a.k > SSK_GAUSS_MAX_K) return SSK_E_SHAPE;
  const size_t smem = gauss_generic_smem(a.k);
  if (cudaFuncSetAttribute(gauss_generic_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
      cudaSuccess)
    return SSK_E_CUDA;
  gauss_generic_kernel<<<grid, GG_THREADS, smem, st>>>(a);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? SSK_OK : SSK_E_CUDA;
}

}  // namespace ssk
