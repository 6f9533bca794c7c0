// K2b: rect windows whose stride divides the window (k = S*R, S in {2, 4, 8}):
// every window is the sum of R x R disjoint S x S blocks, so each input sample is
// touched once (block sums) and each window costs R*R block additions.
//
// Same semantics and exactness as box_int_kernel (src/stats.py:96-141 int64
// window sums, float64 epilogue in the reference's operation order), built for
// the HBM-bound configuration 4 (3840x2160 10-bit, k = 8, s = 4):
//   * lane = 8 adjacent columns (one 16-byte u16 vector / 8-byte u8 vector per row
//     and frame), a warp = 256 columns advancing by 248 so that lane 31 only
//     feeds its neighbours' windows (no shared memory, no block barrier);
//   * sums of x and y accumulate on packed u16 pairs (SIMD-in-register), the
//     squares and the cross term on IMAD; a ring of the last R block rows stays
//     in registers while the lane slides down its segment;
//   * the horizontal R-block window takes the right-hand blocks from lane+1 by
//     warp shuffle.
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace ssk {
namespace {

__device__ __forceinline__ double div_area_b(double x, const BoxArgs& a) {
  return a.area_pow2 ? __dmul_rn(x, a.inv_area) : __ddiv_rn(x, a.area);
}

// reference float64 expression order (src/stats.py:197-201, src/ssim.py:39-40)
__device__ __forceinline__ void emit_window(const BoxArgs& a, int frame, int ar, int ac, const uint32_t (&s)[5],
                                            double& sq, double& sl, double& scs) {
  if (a.wsums) {
    long long* ws = a.wsums + ((long long)frame * 5) * a.map_plane + (long long)ar * a.gw + ac;
#pragma unroll
    for (int m = 0; m < 5; ++m) ws[m * a.map_plane] = (long long)s[m];
  }
  const double s1 = __dmul_rn((double)s[0], a.sscale1), s2 = __dmul_rn((double)s[1], a.sscale1);
  const double q1 = __dmul_rn((double)s[2], a.sscale2), q2 = __dmul_rn((double)s[3], a.sscale2);
  const double p12 = __dmul_rn((double)s[4], a.sscale2);
  const double mu1 = div_area_b(s1, a), mu2 = div_area_b(s2, a);
  const double var1 = fmax(__dsub_rn(div_area_b(q1, a), __dmul_rn(mu1, mu1)), 0.0);
  const double var2 = fmax(__dsub_rn(div_area_b(q2, a), __dmul_rn(mu2, mu2)), 0.0);
  const double cov = __dsub_rn(div_area_b(p12, a), __dmul_rn(mu1, mu2));
  const double num1 = __dadd_rn(__dmul_rn(__dmul_rn(2.0, mu1), mu2), a.c1);
  const double den1 = __dadd_rn(__dadd_rn(__dmul_rn(mu1, mu1), __dmul_rn(mu2, mu2)), a.c1);
  const double num2 = __dadd_rn(__dmul_rn(2.0, cov), a.c2);
  const double den2 = __dadd_rn(__dadd_rn(var1, var2), a.c2);
  const double l = __ddiv_rn(num1, den1);
  const double cs = __ddiv_rn(num2, den2);
  const double q = __dmul_rn(l, cs);
  sq += q;
  sl += l;
  scs += cs;
  if (a.want & (SSK_MAP_TERMS | SSK_MAP_STATS)) {
    double* mp = a.maps + (long long)frame * a.map_frame + (long long)ar * a.gw + ac;
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

__device__ __forceinline__ void emit_fast(const BoxArgs& a, const uint32_t (&s)[5], double& sq, double& sl,
                                          double& scs) {
  double unused = 0.0;  // q^2 sums are a running-sum-kernel feature (plan_ssim routes SSK_WANT_Q2 there)
  box_fast_terms<BoxArgs, false>(a, (unsigned long long)s[0], (unsigned long long)s[1], (unsigned long long)s[2],
                                 (unsigned long long)s[3], (unsigned long long)s[4], sq, sl, scs, unused);
}

// 8 samples of one row as 4 packed u16 pairs (a0|a1<<16, ...), zero past the row end
template <typename TIN>
__device__ __forceinline__ void load8(const unsigned char* rowp, int col, int w, uint32_t (&v)[4]) {
  const TIN* p = reinterpret_cast<const TIN*>(rowp) + col;
  if (col + 8 <= w) {
    if constexpr (sizeof(TIN) == 2) {
      const uint4 t = *reinterpret_cast<const uint4*>(p);
      v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
    } else {
      const uint2 t = *reinterpret_cast<const uint2*>(p);
      v[0] = __byte_perm(t.x, 0, 0x5150);  // (b0, b1)
      v[1] = __byte_perm(t.x, 0, 0x5352);  // (b2, b3)
      v[2] = __byte_perm(t.y, 0, 0x5150);
      v[3] = __byte_perm(t.y, 0, 0x5352);
    }
  } else {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint32_t lo = col + 2 * i < w ? (uint32_t)p[2 * i] : 0u;
      const uint32_t hi = col + 2 * i + 1 < w ? (uint32_t)p[2 * i + 1] : 0u;
      v[i] = lo | (hi << 16);
    }
  }
}

}  // namespace

template <typename TIN, int S, int R>
__global__ void __launch_bounds__(128) box_block_kernel(const __grid_constant__ BoxArgs a) {
  constexpr int NB = 8 / S;               // blocks per lane
  constexpr int WPL = S / 2;              // packed u16 words per block row segment
  static_assert(R - 1 <= NB, "window reaches past the right neighbour lane");
  __shared__ double s_red[4 * 3];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int frame = blockIdx.z;
  const int wcol = (blockIdx.x * 4 + warp) * 248;  // first column of this warp
  const int col = wcol + lane * 8;
  const int b0 = blockIdx.y * a.seg_anchors;      // first anchor row of the segment
  const int b1 = min(b0 + a.seg_anchors, a.gh);
  const unsigned char* bx = a.ref + (long long)frame * a.frame_pitch_b;
  const unsigned char* by = a.dist + (long long)frame * a.frame_pitch_b;
  const int jfirst = col / S;                      // this lane's first block column

  const bool fast = !(a.want & (SSK_MAP_TERMS | SSK_MAP_STATS)) && !a.wsums && a.fast_ok;
  // ring of the last R block rows: [slot][block][moment]
  uint32_t ring[R][NB][5];
  double sq = 0.0, sl = 0.0, scs = 0.0;
  const bool active = b0 < b1 && wcol < a.w;
  const int nrows = active ? (b1 - b0) + R - 1 : 0;  // block rows to read

  for (int base = 0; base < nrows; base += R) {
#pragma unroll
    for (int rr = 0; rr < R; ++rr) {
      const int br = base + rr;  // block row relative to the segment
      if (br < nrows) {
        uint32_t sx[NB] = {}, sy[NB] = {}, xx[NB] = {}, yy[NB] = {}, xy[NB] = {};
        uint32_t vx[S][4], vy[S][4];
#pragma unroll
        for (int r = 0; r < S; ++r) {
          const long long roff = (long long)((b0 + br) * S + r) * a.row_pitch_b;
          load8<TIN>(bx + roff, col, a.w, vx[r]);
          load8<TIN>(by + roff, col, a.w, vy[r]);
        }
#pragma unroll
        for (int r = 0; r < S; ++r) {
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int blk = (2 * q) / S;
            const uint32_t x0 = vx[r][q] & 0xFFFFu, x1 = vx[r][q] >> 16;
            const uint32_t y0 = vy[r][q] & 0xFFFFu, y1 = vy[r][q] >> 16;
            sx[blk] += vx[r][q];   // packed: both halves stay below 2^16 (S*S/2 samples)
            sy[blk] += vy[r][q];
            xx[blk] += x0 * x0 + x1 * x1;
            yy[blk] += y0 * y0 + y1 * y1;
            xy[blk] += x0 * y0 + x1 * y1;
          }
        }
        (void)WPL;
#pragma unroll
        for (int b = 0; b < NB; ++b) {
          ring[rr][b][0] = (sx[b] & 0xFFFFu) + (sx[b] >> 16);
          ring[rr][b][1] = (sy[b] & 0xFFFFu) + (sy[b] >> 16);
          ring[rr][b][2] = xx[b];
          ring[rr][b][3] = yy[b];
          ring[rr][b][4] = xy[b];
        }
        // window rows closed by this block row: anchor row = br - (R - 1)
        if (br >= R - 1) {
          const int ar = b0 + br - (R - 1);
          uint32_t vert[NB][5];
#pragma unroll
          for (int b = 0; b < NB; ++b)
#pragma unroll
            for (int m = 0; m < 5; ++m) {
              uint32_t t = 0;
#pragma unroll
              for (int k = 0; k < R; ++k) t += ring[k][b][m];  // ring holds exactly the last R rows
              vert[b][m] = t;
            }
          // right-hand neighbours (first R-1 blocks of lane+1)
          uint32_t nb[R > 1 ? R - 1 : 1][5];
#pragma unroll
          for (int k = 0; k < R - 1; ++k)
#pragma unroll
            for (int m = 0; m < 5; ++m) nb[k][m] = __shfl_down_sync(0xffffffffu, vert[k][m], 1);
          if (lane < 31) {
#pragma unroll
            for (int b = 0; b < NB; ++b) {
              const int ac = jfirst + b;
              if (ac < a.gw) {
                uint32_t s[5];
#pragma unroll
                for (int m = 0; m < 5; ++m) {
                  uint32_t t = 0;
#pragma unroll
                  for (int k = 0; k < R; ++k) t += (b + k < NB) ? vert[b + k][m] : nb[b + k - NB][m];
                  s[m] = t;
                }
                if (fast)
                  emit_fast(a, s, sq, sl, scs);
                else
                  emit_window(a, frame, ar, ac, s, sq, sl, scs);
              }
            }
          }
        }
      }
    }
  }
  double v[3] = {sq, sl, scs};
  const long long part = ((long long)frame * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
  block_sum_store<3, 4>(v, s_red, a.partials + part * 3);
}

// ---------------------------------------------------------------------------
// Bulk-copy variant (default): the same lane mapping and arithmetic, but each
// warp streams its 256-column strip through a ring of shared-memory stages
// filled by 1-D bulk async copies (cp.async.bulk, completion on an mbarrier),
// ST block rows ahead of the compute.  The loads no longer occupy registers
// or wait in the scoreboard: HBM latency hides behind ST-1 block rows of work.
// ---------------------------------------------------------------------------
namespace {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

template <int S>
__host__ __device__ constexpr int bulk_stages() { return S == 2 ? 4 : 2; }

}  // namespace

template <typename TIN, int S>
__host__ __device__ constexpr size_t bulk_smem_bytes() {
  return (size_t)4 * bulk_stages<S>() * 2 * S * (256 * sizeof(TIN) + (sizeof(TIN) == 1 ? 16 : 0));
}

template <typename TIN, int S, int R, bool FAST>
__global__ void __launch_bounds__(128) box_bulk_kernel(const __grid_constant__ BoxArgs a) {
  constexpr int NB = 8 / S;
  constexpr int ST = bulk_stages<S>();
  constexpr int ES = (int)sizeof(TIN);
  constexpr int ROWB = 256 * ES + (ES == 1 ? 16 : 0);  // u16 strips start 16-byte aligned
  constexpr int STAGEB = 2 * S * ROWB;
  static_assert(R - 1 <= NB, "window reaches past the right neighbour lane");
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ __align__(8) uint64_t bars[4][ST];
  __shared__ double s_red[4 * 3];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int frame = blockIdx.z;
  const int wcol = (blockIdx.x * 4 + warp) * 248;
  const int col = wcol + lane * 8;
  const int b0 = blockIdx.y * a.seg_anchors;
  const int b1 = min(b0 + a.seg_anchors, a.gh);
  const unsigned char* bx = a.ref + (long long)frame * a.frame_pitch_b;
  const unsigned char* by = a.dist + (long long)frame * a.frame_pitch_b;
  const int jfirst = col / S;
  const bool active = b0 < b1 && wcol < a.w;
  const int nrows = active ? (b1 - b0) + R - 1 : 0;
  // source strip: from a 16-byte aligned column, clipped to the (16-byte multiple) row pitch
  const int c_al = wcol & ~(16 / ES - 1);
  const int delta = (wcol - c_al) * ES;
  const int bytes = (int)min((long long)((256 * ES + delta + 15) & ~15), a.row_pitch_b - (long long)c_al * ES);
  // (u16: delta = 0, so bytes <= 512 = ROWB)
  unsigned char* wbuf = smem + (size_t)warp * ST * STAGEB;
  uint64_t* bar = bars[warp];

  if (lane == 0) {
#pragma unroll
    for (int i = 0; i < ST; ++i) mbar_init(&bar[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  auto issue = [&](int br, int stage) {
    const long long row0 = (long long)(b0 + br) * S;
    uint64_t* bb = &bar[stage];
    mbar_expect_tx(bb, (uint32_t)(2 * S * bytes));
#pragma unroll
    for (int img = 0; img < 2; ++img) {
      const unsigned char* base = (img ? by : bx) + (long long)c_al * ES;
#pragma unroll
      for (int r = 0; r < S; ++r)
        bulk_g2s(wbuf + stage * STAGEB + (img * S + r) * ROWB, base + (row0 + r) * a.row_pitch_b, (uint32_t)bytes, bb);
    }
  };
  if (lane == 0) {
    for (int i = 0; i < ST && i < nrows; ++i) issue(i, i);
  }

  constexpr bool fast = FAST;
  uint32_t ring[R][NB][5];
  double sq = 0.0, sl = 0.0, scs = 0.0;
  for (int base = 0; base < nrows; base += R) {
#pragma unroll
    for (int rr = 0; rr < R; ++rr) {
      const int br = base + rr;
      if (br < nrows) {
        const int stage = br % ST;
        SSK_JITTER(200);
        mbar_wait(&bar[stage], (uint32_t)((br / ST) & 1));
        SSK_JITTER(201);
        uint32_t vx[S][4], vy[S][4];
        const unsigned char* sb = wbuf + stage * STAGEB + delta + lane * 8 * ES;
#pragma unroll
        for (int r = 0; r < S; ++r) {
          if constexpr (ES == 2) {
            const uint4 tx = *reinterpret_cast<const uint4*>(sb + r * ROWB);
            const uint4 ty = *reinterpret_cast<const uint4*>(sb + (S + r) * ROWB);
            vx[r][0] = tx.x; vx[r][1] = tx.y; vx[r][2] = tx.z; vx[r][3] = tx.w;
            vy[r][0] = ty.x; vy[r][1] = ty.y; vy[r][2] = ty.z; vy[r][3] = ty.w;
          } else {
            const uint2 tx = *reinterpret_cast<const uint2*>(sb + r * ROWB);
            const uint2 ty = *reinterpret_cast<const uint2*>(sb + (S + r) * ROWB);
            vx[r][0] = __byte_perm(tx.x, 0, 0x5150); vx[r][1] = __byte_perm(tx.x, 0, 0x5352);
            vx[r][2] = __byte_perm(tx.y, 0, 0x5150); vx[r][3] = __byte_perm(tx.y, 0, 0x5352);
            vy[r][0] = __byte_perm(ty.x, 0, 0x5150); vy[r][1] = __byte_perm(ty.x, 0, 0x5352);
            vy[r][2] = __byte_perm(ty.y, 0, 0x5150); vy[r][3] = __byte_perm(ty.y, 0, 0x5352);
          }
        }
        __syncwarp();  // every lane has its samples: the stage can be refilled
        if (lane == 0 && br + ST < nrows) {
          SSK_JITTER(202);
          // order the warp's generic-proxy reads of this stage before the async-proxy refill
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          issue(br + ST, stage);
        }
        uint32_t sx[NB] = {}, sy[NB] = {}, xx[NB] = {}, yy[NB] = {}, xy[NB] = {};
#pragma unroll
        for (int r = 0; r < S; ++r) {
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int blk = (2 * q) / S;
            const uint32_t x0 = vx[r][q] & 0xFFFFu, x1 = vx[r][q] >> 16;
            const uint32_t y0 = vy[r][q] & 0xFFFFu, y1 = vy[r][q] >> 16;
            sx[blk] += vx[r][q];
            sy[blk] += vy[r][q];
            xx[blk] += x0 * x0 + x1 * x1;
            yy[blk] += y0 * y0 + y1 * y1;
            xy[blk] += x0 * y0 + x1 * y1;
          }
        }
#pragma unroll
        for (int b = 0; b < NB; ++b) {
          ring[rr][b][0] = (sx[b] & 0xFFFFu) + (sx[b] >> 16);
          ring[rr][b][1] = (sy[b] & 0xFFFFu) + (sy[b] >> 16);
          ring[rr][b][2] = xx[b];
          ring[rr][b][3] = yy[b];
          ring[rr][b][4] = xy[b];
        }
        if (br >= R - 1) {
          const int ar = b0 + br - (R - 1);
          uint32_t vert[NB][5];
#pragma unroll
          for (int b = 0; b < NB; ++b)
#pragma unroll
            for (int m = 0; m < 5; ++m) {
              uint32_t t = 0;
#pragma unroll
              for (int k = 0; k < R; ++k) t += ring[k][b][m];
              vert[b][m] = t;
            }
          uint32_t nb[R > 1 ? R - 1 : 1][5];
#pragma unroll
          for (int k = 0; k < R - 1; ++k)
#pragma unroll
            for (int m = 0; m < 5; ++m) nb[k][m] = __shfl_down_sync(0xffffffffu, vert[k][m], 1);
          if (lane < 31) {
#pragma unroll
            for (int b = 0; b < NB; ++b) {
              const int ac = jfirst + b;
              if (ac < a.gw) {
                uint32_t s5[5];
#pragma unroll
                for (int m = 0; m < 5; ++m) {
                  uint32_t t = 0;
#pragma unroll
                  for (int k = 0; k < R; ++k) t += (b + k < NB) ? vert[b + k][m] : nb[b + k - NB][m];
                  s5[m] = t;
                }
                if (fast)
                  emit_fast(a, s5, sq, sl, scs);
                else
                  emit_window(a, frame, ar, ac, s5, sq, sl, scs);
              }
            }
          }
        }
      }
    }
  }
  double v[3] = {sq, sl, scs};
  const long long part = ((long long)frame * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
  block_sum_store<3, 4>(v, s_red, a.partials + part * 3);
}

static int box_bulk_enabled() {
  static const int v = [] {
    const char* e = std::getenv("SSK_BOX_BULK");
    return e ? std::atoi(e) : 1;
  }();
  return v;
}

template <typename TIN, int S, int R>
static int launch_block_t(const BoxArgs& a, dim3 grid, cudaStream_t st) {
  if (box_bulk_enabled()) {
    const bool fast = !(a.want & (SSK_MAP_TERMS | SSK_MAP_STATS)) && !a.wsums && a.fast_ok;
    auto fn = fast ? box_bulk_kernel<TIN, S, R, true> : box_bulk_kernel<TIN, S, R, false>;
    const size_t smem = bulk_smem_bytes<TIN, S>();
    if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
      return SSK_E_CUDA;
    fn<<<grid, 128, smem, st>>>(a);
  } else {
    box_block_kernel<TIN, S, R><<<grid, 128, 0, st>>>(a);
  }
  note_launch();
  return cudaGetLastError() == cudaSuccess ? SSK_OK : SSK_E_CUDA;
}

template <typename TIN>
static int launch_block_dtype(const BoxArgs& a, dim3 grid, cudaStream_t st) {
  const int S = a.s, R = a.k / a.s;
  if (S == 4 && R == 1) return launch_block_t<TIN, 4, 1>(a, grid, st);
  if (S == 4 && R == 2) return launch_block_t<TIN, 4, 2>(a, grid, st);
  if (S == 4 && R == 3) return launch_block_t<TIN, 4, 3>(a, grid, st);
  if (S == 2 && R == 1) return launch_block_t<TIN, 2, 1>(a, grid, st);
  if (S == 2 && R == 2) return launch_block_t<TIN, 2, 2>(a, grid, st);
  if (S == 2 && R == 3) return launch_block_t<TIN, 2, 3>(a, grid, st);
  if (S == 2 && R == 4) return launch_block_t<TIN, 2, 4>(a, grid, st);
  if (S == 2 && R == 5) return launch_block_t<TIN, 2, 5>(a, grid, st);
  if (S == 8 && R == 1) return launch_block_t<TIN, 8, 1>(a, grid, st);
  if (S == 8 && R == 2) return launch_block_t<TIN, 8, 2>(a, grid, st);
  return SSK_E_SHAPE;
}

bool box_block_supported(int dtype, int k, int s, bool wide, double stored_max) {
  if (wide || (dtype != SSK_U8 && dtype != SSK_U16) || s < 2 || k % s != 0) return false;
  if ((double)s * s / 2.0 * stored_max >= 65536.0) return false;  // packed u16 half-sums must not carry
  const int R = k / s;
  if (s == 4) return R >= 1 && R <= 3;
  if (s == 2) return R >= 1 && R <= 5;
  if (s == 8) return R >= 1 && R <= 2;
  return false;
}

int launch_box_block(const BoxArgs& a, dim3 grid, cudaStream_t st) {
  return a.dtype == SSK_U8 ? launch_block_dtype<uint8_t>(a, grid, st) : launch_block_dtype<uint16_t>(a, grid, st);
}

}  // namespace ssk
