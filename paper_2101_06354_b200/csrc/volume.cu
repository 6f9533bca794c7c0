// SSIM-3D rolling volumes (src/spatiotemporal.py:28-207) on the device.
//
// A RollingVolume keeps the five per-pixel temporal sums (x, y, x^2, y^2, xy
// over the last depth <= Kt frame pairs) as planes in HBM and updates them per
// pushed frame with T += I(new) - I(old) (src/spatiotemporal.py:84-90), so the
// per-frame cost does not depend on Kt.  Integer samples keep the planes in
// int64: the recursion is exact, so the reference's periodic refresh
// (REFRESH_INTERVAL, :28-30, :95-101) is a no-op and results match the
// reference's float64 sums (exact integers there too) bit for bit.  Float
// samples keep float64 planes updated in the reference's order (s -= old;
// s += new) and are refreshed from the buffered frames like the reference.
// The spatial k x k window over the planes (the reference's SATs + 4-corner
// rule, :122-138) reuses the exact running-sum box kernel (box_int_kernel<MOM>)
// with area = k*k*depth.
#include <type_traits>

#include "common.cuh"
#include "kernels.h"

namespace ssk {

template <typename TS, typename TA>
__global__ void volume_update_kernel(TA* __restrict__ planes, long long pp, long long prp,
                                     const TS* __restrict__ nr, const TS* __restrict__ nd,
                                     const TS* __restrict__ orf, const TS* __restrict__ od, long long srp,
                                     int h, int w, int mode) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y;
  if (x >= w) return;
  const long long si = (long long)y * srp + x;
  const TA a = (TA)nr[si], b = (TA)nd[si];
  const TA nt[5] = {a, b, a * a, b * b, a * b};
  TA* p = planes + (long long)y * prp + x;
  if (mode == 0) {
#pragma unroll
    for (int m = 0; m < 5; ++m) p[m * pp] = nt[m];
  } else if (mode == 1) {
#pragma unroll
    for (int m = 0; m < 5; ++m) p[m * pp] = p[m * pp] + nt[m];
  } else {
    const TA oa = (TA)orf[si], ob = (TA)od[si];
    const TA ot[5] = {oa, ob, oa * oa, ob * ob, oa * ob};
#pragma unroll
    for (int m = 0; m < 5; ++m) {
      TA v = p[m * pp];
      v = v - ot[m];  // T(k) = T(k-1) - I(k-Kt) + I(k), in the reference's order
      v = v + nt[m];
      p[m * pp] = v;
    }
  }
}

int launch_volume_update(void* planes, int is_float, long long pp, long long prp, const void* nr, const void* nd,
                         const void* orf, const void* od, int dtype, long long srp, int h, int w, int mode,
                         cudaStream_t st) {
  dim3 block(128), grid((w + 127) / 128, h);
#define VU(TS, TA)                                                                                     \
  volume_update_kernel<TS, TA><<<grid, block, 0, st>>>((TA*)planes, pp, prp, (const TS*)nr, (const TS*)nd, \
                                                       (const TS*)orf, (const TS*)od, srp, h, w, mode)
  if (!is_float && dtype == SSK_U8) VU(uint8_t, long long);
  else if (!is_float && dtype == SSK_U16) VU(uint16_t, long long);
  else if (is_float && dtype == SSK_F64) VU(double, double);
  else return SSK_E_ARG;
#undef VU
  note_launch();
  return cudaGetLastError() == cudaSuccess ? SSK_OK : SSK_E_CUDA;
}

// Recompute float64 sums from the buffered frames, oldest first (direct_sums, :103-115).
struct RefreshArgs {
  const double* refs[64];
  const double* dists[64];
};

__global__ void volume_refresh_kernel(double* __restrict__ planes, long long pp, long long prp,
                                      const __grid_constant__ RefreshArgs r, int count, long long srp, int h, int w) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y;
  if (x >= w) return;
  double s[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
  const long long si = (long long)y * srp + x;
  for (int i = 0; i < count; ++i) {
    const double a = r.refs[i][si], b = r.dists[i][si];
    s[0] += a;
    s[1] += b;
    s[2] += a * a;
    s[3] += b * b;
    s[4] += a * b;
  }
  double* p = planes + (long long)y * prp + x;
#pragma unroll
  for (int m = 0; m < 5; ++m) p[m * pp] = s[m];
}

int launch_volume_refresh(void* planes, long long pp, long long prp, const void* const* refs,
                          const void* const* dists, int count, int dtype, long long srp, int h, int w,
                          cudaStream_t st) {
  if (dtype != SSK_F64 || count < 1 || count > 64) return SSK_E_ARG;
  RefreshArgs r{};
  for (int i = 0; i < count; ++i) {
    r.refs[i] = static_cast<const double*>(refs[i]);
    r.dists[i] = static_cast<const double*>(dists[i]);
  }
  dim3 block(128), grid((w + 127) / 128, h);
  volume_refresh_kernel<<<grid, block, 0, st>>>(static_cast<double*>(planes), pp, prp, r, count, srp, h, w);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? SSK_OK : SSK_E_CUDA;
}

// float64 planes: direct k x k window sums (row order) + the reference's epilogue.
__global__ void __launch_bounds__(128) volume_direct_kernel(const __grid_constant__ BoxArgs a, const double* planes) {
  __shared__ double s_red[4 * 3];
  const int ac = blockIdx.x * blockDim.x + threadIdx.x;
  const int ar = blockIdx.y * blockDim.y + threadIdx.y;
  double sq = 0.0, sl = 0.0, scs = 0.0;
  if (ac < a.gw && ar < a.gh) {
    double t[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
    for (int i = 0; i < a.k; ++i) {
      const double* row = planes + (long long)(ar * a.s + i) * a.mom_rp + ac * a.s;
      for (int j = 0; j < a.k; ++j)
#pragma unroll
        for (int m = 0; m < 5; ++m) t[m] += row[m * a.mom_plane + j];
    }
    const double mu1 = __ddiv_rn(t[0], a.area), mu2 = __ddiv_rn(t[1], a.area);
    const double var1 = fmax(__dsub_rn(__ddiv_rn(t[2], a.area), __dmul_rn(mu1, mu1)), 0.0);
    const double var2 = fmax(__dsub_rn(__ddiv_rn(t[3], a.area), __dmul_rn(mu2, mu2)), 0.0);
    const double cov = __dsub_rn(__ddiv_rn(t[4], a.area), __dmul_rn(mu1, mu2));
    const double l = __ddiv_rn(__dadd_rn(__dmul_rn(__dmul_rn(2.0, mu1), mu2), a.c1),
                               __dadd_rn(__dadd_rn(__dmul_rn(mu1, mu1), __dmul_rn(mu2, mu2)), a.c1));
    const double cs = __ddiv_rn(__dadd_rn(__dmul_rn(2.0, cov), a.c2), __dadd_rn(__dadd_rn(var1, var2), a.c2));
    const double q = __dmul_rn(l, cs);
    sq = q;
    sl = l;
    scs = cs;
    if (a.want & (SSK_MAP_TERMS | SSK_MAP_STATS)) {
      double* mp = a.maps + (long long)ar * a.gw + ac;
      const bool terms = (a.want & SSK_MAP_TERMS) != 0;
      mp[0] = terms ? l : mu1;
      mp[a.map_plane] = terms ? cs : mu2;
      mp[2 * a.map_plane] = terms ? q : var1;
      if (!terms) {
        mp[3 * a.map_plane] = var2;
        mp[4 * a.map_plane] = cov;
      }
    }
  }
  double v[3] = {sq, sl, scs};
  block_sum_store<3, 4>(v, s_red, a.partials + ((long long)blockIdx.y * gridDim.x + blockIdx.x) * 3);
}

int launch_volume_direct(const BoxArgs& a, const double* planes, dim3 grid, dim3 block, cudaStream_t st) {
  volume_direct_kernel<<<grid, block, 0, st>>>(a, planes);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? SSK_OK : SSK_E_CUDA;
}

}  // namespace ssk
