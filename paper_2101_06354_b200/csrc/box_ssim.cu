// K2: rect-window SSIM with exact integer window sums.
//
// Replaces the reference's integral engine for rect windows
//   build_integral_set / _sat   (src/stats.py:66-71, :96-116)  int64 SATs
//   _grid_window_sums           (src/stats.py:130-141)         4-corner rule
//   stats_from_sums(area=k*k)   (src/stats.py:185-202)
//   term_maps_from_stats        (src/ssim.py:31-46)
// and its naive rect route (_sliding_raw_sums, src/stats.py:144-152), which
// yields the same grids.  Instead of materialising five (H+1)x(W+1) int64
// tables in HBM (the reference's 88% hot spot), each CTA keeps per-column
// running sums in registers: one input column per thread slides down the
// rows accumulating x, y, x^2, y^2, xy in u32 (modular: window sums below
// 2^32 are exact even when the running sum wraps) or u64; at the rows that
// close a window the vertical window sum is the difference with the prefix
// recorded k rows earlier.  The horizontal window sums are taken from a
// shared-memory row of vertical sums.  The float64 epilogue replays the
// reference's operation order (mu = S/area, var = max(Q/area - mu*mu, 0),
// cov = P/area - mu1*mu2, l, cs, q) with IEEE-rounded intrinsics, so maps are
// bit-identical to the reference's for integer samples and for the scaled
// integer pyramid levels (whose float64 sums the reference also forms
// exactly).
#include "common.cuh"
#include "kernels.h"

namespace ssk {

namespace {

__device__ __forceinline__ double div_area(double x, const BoxArgs& a) {
  return a.area_pow2 ? __dmul_rn(x, a.inv_area) : __ddiv_rn(x, a.area);
}

// The reference's float64 expression order (src/stats.py:197-201, src/ssim.py:39-40).
struct BoxTerms {
  double mu1, mu2, var1, var2, cov, l, cs, q;
};

__device__ __forceinline__ BoxTerms box_terms(double s1, double s2, double q1, double q2, double p12,
                                              const BoxArgs& a) {
  BoxTerms t;
  t.mu1 = div_area(s1, a);
  t.mu2 = div_area(s2, a);
  t.var1 = fmax(__dsub_rn(div_area(q1, a), __dmul_rn(t.mu1, t.mu1)), 0.0);
  t.var2 = fmax(__dsub_rn(div_area(q2, a), __dmul_rn(t.mu2, t.mu2)), 0.0);
  t.cov = __dsub_rn(div_area(p12, a), __dmul_rn(t.mu1, t.mu2));
  const double num1 = __dadd_rn(__dmul_rn(__dmul_rn(2.0, t.mu1), t.mu2), a.c1);
  const double den1 = __dadd_rn(__dadd_rn(__dmul_rn(t.mu1, t.mu1), __dmul_rn(t.mu2, t.mu2)), a.c1);
  const double num2 = __dadd_rn(__dmul_rn(2.0, t.cov), a.c2);
  const double den2 = __dadd_rn(__dadd_rn(t.var1, t.var2), a.c2);
  t.l = __ddiv_rn(num1, den1);
  t.cs = __ddiv_rn(num2, den2);
  t.q = __dmul_rn(t.l, t.cs);
  return t;
}

template <bool Q2>
__device__ __forceinline__ void box_emit(const BoxTerms& t, const BoxArgs& a, int frame, int ar,
                                         int ac, double& sq, double& sl, double& scs, double& sq2) {
  sq += t.q;
  if constexpr (Q2) sq2 += __dmul_rn(t.q, t.q);
  sl += t.l;
  scs += t.cs;
  if (a.want & (SSK_MAP_TERMS | SSK_MAP_STATS)) {
    double* mp = a.maps + (long long)frame * a.map_frame + (long long)ar * a.gw + ac;
    if (a.want & SSK_MAP_TERMS) {
      mp[0] = t.l;
      mp[a.map_plane] = t.cs;
      mp[2 * a.map_plane] = t.q;
    } else {
      mp[0] = t.mu1;
      mp[a.map_plane] = t.mu2;
      mp[2 * a.map_plane] = t.var1;
      mp[3 * a.map_plane] = t.var2;
      mp[4 * a.map_plane] = t.cov;
    }
  }
}

template <typename T>
__device__ __forceinline__ T load_sample(const unsigned char* p) {
  return *reinterpret_cast<const T*>(p);
}

}  // namespace

// ---------------------------------------------------------------------------
// Integer kernel: TIN in {u8, u16, u32}, ACC in {u32, u64}.
// Grid: (strips, segments, frames); block = 128 threads = 128 input columns.
// ---------------------------------------------------------------------------
// MOM = true: the five per-pixel moments come precomputed from int64 planes
// (the rolling temporal sums of a RollingVolume, src/spatiotemporal.py:60-138)
// instead of being formed from staged x / y samples; everything else is shared.
template <typename TIN, typename ACC, bool MOM = false, bool FAST = false, bool Q2 = false>
__global__ void __launch_bounds__(BX_THREADS) box_int_kernel(const __grid_constant__ BoxArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ double s_red[(BX_THREADS / 32) * 3];
  const int CH = a.ch, s = a.s, k = a.k, P = a.in_pitch, NSL = a.nslot;
  constexpr int VP = BX_THREADS + 4;
  unsigned char* stage = smem;                                            // [2][2][CH][P]
  ACC* hist = reinterpret_cast<ACC*>(smem + (size_t)4 * CH * P);          // [NSL][5][128]
  ACC* vrow = hist + (size_t)NSL * 5 * BX_THREADS;                        // [VR][5][VP]

  const int tid = threadIdx.x;
  const int strip = blockIdx.x, seg = blockIdx.y, frame = blockIdx.z;
  const int A0 = strip * a.na;
  // stage from a 16-byte aligned column; anchors sit `delta` columns into the stage
  const int c0 = (A0 * s) & ~((16 / (int)sizeof(TIN)) - 1);
  const int delta = A0 * s - c0;
  const int b0 = seg * a.seg_anchors;
  const int b1 = min(b0 + a.seg_anchors, a.gh);
  const int r0 = b0 * s;
  const int rend = (b1 - 1) * s + k;
  const int nrows = rend - r0;
  const int nchunks = (nrows + CH - 1) / CH;
  const int esz = (int)sizeof(TIN);
  const int nch = (BX_THREADS * esz) >> 4;
  const int row_bytes_left = (a.w - c0) * esz;
  const unsigned char* base_x = a.ref + (long long)frame * a.frame_pitch_b;
  const unsigned char* base_y = a.dist + (long long)frame * a.frame_pitch_b;

  auto issue_stage = [&](int chunk, int buf) {
    if constexpr (MOM) return;  // moment planes are read straight from HBM
    const int rbase = r0 + chunk * CH;
    const int total = 2 * CH * nch;
    for (int i = tid; i < total; i += BX_THREADS) {
      const int img = i / (CH * nch);
      const int rem = i - img * (CH * nch);
      const int g = rem / nch;
      const int q = rem - g * nch;
      const int row = rbase + g;
      if (row >= rend) continue;
      const int off = q * 16;
      int valid = row_bytes_left - off;
      valid = valid < 0 ? 0 : (valid > 16 ? 16 : valid);
      const unsigned char* rowp = (img ? base_y : base_x) + (long long)row * a.row_pitch_b;
      const unsigned char* src = valid ? rowp + (long long)c0 * esz + off : rowp;
      cp_async16(stage + ((buf * 2 + img) * CH + g) * P + off, src, valid);
    }
    cp_async_commit();
  };

  // prefix state: P(rows < r0) == 0 is anchor 0's record
  ACC pre[5] = {0, 0, 0, 0, 0};
#pragma unroll
  for (int m = 0; m < 5; ++m) hist[m * BX_THREADS + tid] = 0;
  int rec_at = s, rec_slot = 1 % NSL;   // next prefix record: after row u where u+1 == rec_at
  int emit_at = k, emit_slot = 0;       // next window close: after row u where u+1 == emit_at
  int bnext = 0;                        // next anchor row (relative) to close

  double sq = 0.0, sl = 0.0, scs = 0.0, sq2 = 0.0;
  issue_stage(0, 0);

  // MOM with chunks of <= MCH rows: the chunk's 5 x CH moment values of this column are
  // loaded into registers one chunk ahead (issued before the previous chunk's horizontal
  // pass), so HBM latency overlaps compute instead of stalling every row
  constexpr int MCH = 8;
  const bool mom_pre = MOM && CH <= MCH;
  long long mv[MOM ? MCH : 1][5];
  auto load_moments = [&](int chunk) {
    if constexpr (MOM) {
      const int colx = c0 + tid;
      const int rb = r0 + chunk * CH;
#pragma unroll
      for (int g = 0; g < MCH; ++g) {
        const int row = rb + g;
        const bool ok = g < CH && row < rend && colx < a.w;
        const long long* mp = a.mom + (long long)(ok ? row : r0) * a.mom_rp + (ok ? colx : 0);
#pragma unroll
        for (int m = 0; m < 5; ++m) mv[g][m] = ok ? mp[m * a.mom_plane] : 0ll;
      }
    }
  };
  if (mom_pre) load_moments(0);

  for (int c = 0; c < nchunks; ++c) {
    if (c + 1 < nchunks) {
      issue_stage(c + 1, (c + 1) & 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();

    // ---- vertical: running sums down this thread's column ----
    const int ubase = c * CH;
    const int urows = min(CH, nrows - ubase);
    const unsigned char* sx = stage + ((c & 1) * 2 + 0) * CH * P + tid * esz;
    const unsigned char* sy = stage + ((c & 1) * 2 + 1) * CH * P + tid * esz;
    const int bfirst = bnext;
    int nemit = 0;
    auto row_step = [&](const int g) {
      const int u1 = ubase + g + 1;
      if (u1 == emit_at) {
        ACC* vr = vrow + (size_t)nemit * 5 * VP + tid;
        const ACC* hs = hist + (size_t)emit_slot * 5 * BX_THREADS + tid;
#pragma unroll
        for (int m = 0; m < 5; ++m) vr[m * VP] = pre[m] - hs[m * BX_THREADS];
        ++nemit;
        ++bnext;
        emit_at += s;
        emit_slot = emit_slot + 1 == NSL ? 0 : emit_slot + 1;
      }
      if (u1 == rec_at) {
        ACC* hs = hist + (size_t)rec_slot * 5 * BX_THREADS + tid;
#pragma unroll
        for (int m = 0; m < 5; ++m) hs[m * BX_THREADS] = pre[m];
        rec_at += s;
        rec_slot = rec_slot + 1 == NSL ? 0 : rec_slot + 1;
      }
    };
    if (mom_pre) {
#pragma unroll
      for (int g = 0; g < MCH; ++g) {
        if (g < urows) {
#pragma unroll
          for (int m = 0; m < 5; ++m) pre[m] += (ACC)mv[g][m];
          row_step(g);
        }
      }
      if (c + 1 < nchunks) load_moments(c + 1);
    }
    for (int g = 0; g < (mom_pre ? 0 : urows); ++g) {
      if constexpr (MOM) {
        const int row = r0 + ubase + g, colx = c0 + tid;
        if (colx < a.w) {
          const long long* mp = a.mom + (long long)row * a.mom_rp + colx;
#pragma unroll
          for (int m = 0; m < 5; ++m) pre[m] += (ACC)mp[m * a.mom_plane];
        }
      } else {
        const ACC x = (ACC)load_sample<TIN>(sx + g * P);
        const ACC y = (ACC)load_sample<TIN>(sy + g * P);
        pre[0] += x;
        pre[1] += y;
        pre[2] += x * x;
        pre[3] += y * y;
        pre[4] += x * y;
      }
      row_step(g);
    }
    __syncthreads();

    // ---- horizontal window sums + float64 epilogue for the closed anchor rows ----
    const int items = nemit * a.na;
    for (int i = tid; i < items; i += BX_THREADS) {
      const int g = i / a.na;
      const int jj = i - g * a.na;
      const int ac = A0 + jj;
      const int ar = b0 + bfirst + g;
      if (ac >= a.gw || ar >= b1) continue;
      const ACC* vr = vrow + (size_t)g * 5 * VP + jj * s + delta;
      ACC sums[5];
#pragma unroll
      for (int m = 0; m < 5; ++m) {
        ACC t = 0;
        for (int q = 0; q < k; ++q) t += vr[m * VP + q];
        sums[m] = t;
      }
      if (a.wsums) {
        long long* ws = a.wsums + ((long long)frame * 5) * a.map_plane + (long long)ar * a.gw + ac;
#pragma unroll
        for (int m = 0; m < 5; ++m) ws[m * a.map_plane] = (long long)sums[m];
      }
      if constexpr (FAST) {
        box_fast_terms<BoxArgs, Q2>(a, (unsigned long long)sums[0], (unsigned long long)sums[1],
                                    (unsigned long long)sums[2],
                       (unsigned long long)sums[3], (unsigned long long)sums[4], sq, sl, scs, sq2);
        continue;
      }
      const BoxTerms t = box_terms(__dmul_rn((double)sums[0], a.sscale1),
                                   __dmul_rn((double)sums[1], a.sscale1),
                                   __dmul_rn((double)sums[2], a.sscale2),
                                   __dmul_rn((double)sums[3], a.sscale2),
                                   __dmul_rn((double)sums[4], a.sscale2), a);
      box_emit<Q2>(t, a, frame, ar, ac, sq, sl, scs, sq2);
    }
    // the barrier at the top of the next chunk protects vrow
  }

  double v[3] = {sq, sl, scs};
  const long long part = ((long long)frame * gridDim.y + seg) * gridDim.x + strip;
  block_sum_store<3, BX_THREADS / 32>(v, s_red, a.partials + part * 3);
  if constexpr (Q2) {
    __shared__ double s_red2[BX_THREADS / 32];
    store_q2<BoxArgs, BX_THREADS / 32>(a, sq2, s_red2, part);
  }
}

// ---------------------------------------------------------------------------
// Direct kernel (any dtype, any k): one thread per anchor, k x k loop in row
// order.  Integer samples accumulate in int64 (exact, any window size);
// float samples in float64.  Used for float planes and windows wider than a
// strip.
// ---------------------------------------------------------------------------
template <typename TIN, bool INT>
__global__ void __launch_bounds__(128) box_direct_kernel(const __grid_constant__ BoxArgs a) {
  __shared__ double s_red[4 * 3];
  const int ac = blockIdx.x * blockDim.x + threadIdx.x;
  const int ar = blockIdx.y * blockDim.y + threadIdx.y;
  const int frame = blockIdx.z;
  double sq = 0.0, sl = 0.0, scs = 0.0, sq2 = 0.0;
  if (ac < a.gw && ar < a.gh) {
    const unsigned char* bx = a.ref + (long long)frame * a.frame_pitch_b;
    const unsigned char* by = a.dist + (long long)frame * a.frame_pitch_b;
    using T = typename std::conditional<INT, long long, double>::type;
    T s1 = 0, s2 = 0, q1 = 0, q2 = 0, p = 0;
    for (int i = 0; i < a.k; ++i) {
      const long long roff = (long long)(ar * a.s + i) * a.row_pitch_b;
      for (int j = 0; j < a.k; ++j) {
        const long long off = roff + (long long)(ac * a.s + j) * (long long)sizeof(TIN);
        const T x = (T)load_sample<TIN>(bx + off);
        const T y = (T)load_sample<TIN>(by + off);
        s1 += x;
        s2 += y;
        q1 += x * x;
        q2 += y * y;
        p += x * y;
      }
    }
    if (INT && a.wsums) {
      long long* ws = a.wsums + ((long long)frame * 5) * a.map_plane + (long long)ar * a.gw + ac;
      ws[0] = (long long)s1;
      ws[a.map_plane] = (long long)s2;
      ws[2 * a.map_plane] = (long long)q1;
      ws[3 * a.map_plane] = (long long)q2;
      ws[4 * a.map_plane] = (long long)p;
    }
    const BoxTerms t = box_terms(__dmul_rn((double)s1, a.sscale1), __dmul_rn((double)s2, a.sscale1),
                                 __dmul_rn((double)q1, a.sscale2), __dmul_rn((double)q2, a.sscale2),
                                 __dmul_rn((double)p, a.sscale2), a);
    box_emit<true>(t, a, frame, ar, ac, sq, sl, scs, sq2);
  }
  double v[3] = {sq, sl, scs};
  const long long part = ((long long)frame * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
  block_sum_store<3, 4>(v, s_red, a.partials + part * 3);
  __shared__ double s_red2[4];
  store_q2<BoxArgs, 4>(a, sq2, s_red2, part);
}

// ---------------------------------------------------------------------------

size_t box_smem_bytes(const BoxArgs& a, bool wide) {
  const size_t acc = wide ? 8 : 4;
  const int VR = a.ch / a.s;
  return (size_t)4 * a.ch * a.in_pitch + (size_t)a.nslot * 5 * BX_THREADS * acc +
         (size_t)VR * 5 * (BX_THREADS + 4) * acc;
}

template <typename TIN, typename ACC>
static int launch_int_t(const BoxArgs& a, dim3 grid, size_t smem, cudaStream_t st) {
  const bool fast = !(a.want & (SSK_MAP_TERMS | SSK_MAP_STATS)) && !a.wsums && a.fast_ok;
  const bool q2 = a.partials2 != nullptr;
  auto fn = fast ? (q2 ? box_int_kernel<TIN, ACC, false, true, true> : box_int_kernel<TIN, ACC, false, true, false>)
                 : (q2 ? box_int_kernel<TIN, ACC, false, false, true> : box_int_kernel<TIN, ACC, false, false, false>);
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return SSK_E_CUDA;
  fn<<<grid, BX_THREADS, smem, st>>>(a);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? SSK_OK : SSK_E_CUDA;
}

int launch_box_moments(const BoxArgs& a, dim3 grid, cudaStream_t st) {
  const bool fast = !(a.want & (SSK_MAP_TERMS | SSK_MAP_STATS)) && !a.wsums && a.fast_ok;
  auto fn = fast ? box_int_kernel<uint8_t, unsigned long long, true, true> : box_int_kernel<uint8_t, unsigned long long, true>;
  const size_t smem = box_smem_bytes(a, true);
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return SSK_E_CUDA;
  fn<<<grid, BX_THREADS, smem, st>>>(a);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? SSK_OK : SSK_E_CUDA;
}

int launch_box_int(const BoxArgs& a, dim3 grid, bool wide, cudaStream_t st) {
  const size_t smem = box_smem_bytes(a, wide);
  switch (a.dtype) {
    case SSK_U8:
      return wide ? launch_int_t<uint8_t, unsigned long long>(a, grid, smem, st)
                  : launch_int_t<uint8_t, uint32_t>(a, grid, smem, st);
    case SSK_U16:
      return wide ? launch_int_t<uint16_t, unsigned long long>(a, grid, smem, st)
                  : launch_int_t<uint16_t, uint32_t>(a, grid, smem, st);
    case SSK_U32:
      return wide ? launch_int_t<uint32_t, unsigned long long>(a, grid, smem, st)
                  : launch_int_t<uint32_t, uint32_t>(a, grid, smem, st);
    default:
      return SSK_E_ARG;
  }
}

int launch_box_float(const BoxArgs& a, dim3 grid, dim3 block, cudaStream_t st) {
  switch (a.dtype) {
    case SSK_U8: box_direct_kernel<uint8_t, true><<<grid, block, 0, st>>>(a); break;
    case SSK_U16: box_direct_kernel<uint16_t, true><<<grid, block, 0, st>>>(a); break;
    case SSK_U32: box_direct_kernel<uint32_t, true><<<grid, block, 0, st>>>(a); break;
    case SSK_F32: box_direct_kernel<float, false><<<grid, block, 0, st>>>(a); break;
    case SSK_F64: box_direct_kernel<double, false><<<grid, block, 0, st>>>(a); break;
    default: return SSK_E_ARG;
  }
  note_launch();
  return cudaGetLastError() == cudaSuccess ? SSK_OK : SSK_E_CUDA;
}

}  // namespace ssk
