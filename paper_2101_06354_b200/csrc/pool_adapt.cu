// Spatial pooling family and resolution adaptation on the device.
//
//  * pooling (src/pooling.py:157-243): every SPATIAL_KINDS pooler over a batch
//    of quality maps.  Sums run in float64 with a fixed-order, geometry-only
//    reduction tree (run-to-run reproducible); order statistics are exact (a
//    radix select on order-preserving bit patterns), so np.percentile's
//    'linear' rule is reproduced bit for bit.
//  * box_downsample (src/adaptation.py:93-110): integer-factor block means with
//    partial trailing blocks, the resampler of every ScalePolicy.
#include <cmath>
#include <cstring>
#include <type_traits>

#include "common.cuh"
#include "kernels.h"

namespace ssk {
namespace {

constexpr int PL_THREADS = 256;
constexpr int SEL_BITS = 11;
constexpr int SEL_BINS = 1 << SEL_BITS;
constexpr int MAX_RANKS = 6;  // fns: three quartiles x (lower, upper) order statistic
constexpr int NC1 = 5;        // pass-1 partials: sum, min, max, f1, f2

struct PoolArgs {
  const unsigned char* vals;
  const unsigned char* aux;
  long long rp, fp, arp, afp;  // elements
  int n, h, w, nblk;           // nblk row ranges (blocks) per map
  int flat;                    // rows contiguous (pitch == width) in values and aux: flat index loop
  double cnt;                  // h * w
  int kind;
  double p, o, a, b, ps, rs;
  int nranks, nq;
  long long rank[MAX_RANKS];   // quantile i uses ranks 2i (lower) and 2i+1 (upper)
  double gamma[MAX_RANKS / 2];
  int pass2;
  double* part1;               // [n][nblk][NC1]
  double* part2;               // [n][nblk]
  unsigned long long* sel;     // [n][MAX_RANKS][2]: key prefix, remaining rank
  unsigned int* hist;          // [n][MAX_RANKS][SEL_BINS]
  double* out;
  double* mean;
};

// order-preserving unsigned keys (-0.0 folded onto +0.0 first)
template <typename T>
struct Keys;
template <>
struct Keys<float> {
  using K = uint32_t;
  static constexpr int B = 32;
  __device__ static K key(float v) {
    const uint32_t u = __float_as_uint(__fadd_rn(v, 0.0f));
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
  }
  __device__ static double value(unsigned long long k) {
    const uint32_t kk = (uint32_t)k;
    return (double)__uint_as_float((kk & 0x80000000u) ? (kk & 0x7fffffffu) : ~kk);
  }
};
template <>
struct Keys<double> {
  using K = unsigned long long;
  static constexpr int B = 64;
  __device__ static K key(double v) {
    const unsigned long long u = (unsigned long long)__double_as_longlong(__dadd_rn(v, 0.0));
    return (u & 0x8000000000000000ull) ? ~u : (u | 0x8000000000000000ull);
  }
  __device__ static double value(unsigned long long k) {
    return __longlong_as_double((long long)((k & 0x8000000000000000ull) ? (k & 0x7fffffffffffffffull) : ~k));
  }
};

// x ** p with numpy's fast scalar-power cases (1, 2, 0.5) done exactly
__device__ __forceinline__ double powp(double x, double p) {
  if (p == 1.0) return x;
  if (p == 2.0) return __dmul_rn(x, x);
  if (p == 0.5) return __dsqrt_rn(x);
  return pow(x, p);
}

// np.percentile 'linear' interpolation (numpy/lib/_function_base_impl.py _lerp)
__device__ __forceinline__ double np_lerp(double lo, double hi, double t) {
  const double d = __dsub_rn(hi, lo);
  return t >= 0.5 ? __dsub_rn(hi, __dmul_rn(d, __dsub_rn(1.0, t))) : __dadd_rn(lo, __dmul_rn(d, t));
}

// Visit the elements of row range `blk` of one map: f(load(value offset), value offset,
// aux offset, slot 0..3), block-strided.  Contiguous maps (the usual [gh][gw] planes) take a flat
// index loop that issues four independent loads before using any of them: one
// outstanding load per thread leaves these streaming passes latency-bound.
template <int NT = PL_THREADS, typename L, typename F>
__device__ __forceinline__ void for_range(const PoolArgs& a, int blk, L&& load, F&& f) {
  const int r0 = (int)((long long)blk * a.h / a.nblk);
  const int r1 = (int)((long long)(blk + 1) * a.h / a.nblk);
  if (a.flat) {
    const long long e1 = (long long)r1 * a.w;
    long long i = (long long)r0 * a.w + threadIdx.x;
    for (; i + 3 * NT < e1; i += 4 * NT) {
      const auto v0 = load(i), v1 = load(i + NT), v2 = load(i + 2 * NT), v3 = load(i + 3 * NT);
      f(v0, i, i, 0);
      f(v1, i + NT, i + NT, 1);
      f(v2, i + 2 * NT, i + 2 * NT, 2);
      f(v3, i + 3 * NT, i + 3 * NT, 3);
    }
    for (; i < e1; i += NT) f(load(i), i, i, 0);
    return;
  }
  const long long total = (long long)(r1 - r0) * a.w;
  const int dr = NT / a.w, dc = NT % a.w;
  int row = r0 + (int)(threadIdx.x / a.w), col = (int)(threadIdx.x % a.w);
  for (long long i = threadIdx.x; i < total; i += NT) {
    const long long vo = (long long)row * a.rp + col;
    f(load(vo), vo, (long long)row * a.arp + col, 0);
    row += dr;
    col += dc;
    if (col >= a.w) {
      col -= a.w;
      ++row;
    }
  }
}

__device__ __forceinline__ double warp_min(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Fixed-order fold of one component of a frame's per-block partials by one warp
// (identical result in every caller: lane-strided sums then an xor tree).
__device__ double fold_sum(const double* part, int nblk, int ncomp, int c) {
  const int lane = threadIdx.x & 31;
  double s = 0.0;
  for (int i = lane; i < nblk; i += 32) s += part[(long long)i * ncomp + c];
  return warp_sum(s);
}

template <typename T>
__device__ double rank_value(const PoolArgs& a, int frame, int r) {
  return Keys<T>::value(a.sel[((long long)frame * MAX_RANKS + r) * 2]);
}

// per-element work of the two passes
template <typename T>
__device__ __forceinline__ void pass1_elem(const PoolArgs& a, const T* ab, double v, long long ao, double& sum,
                                           double& mn, double& mx, double& f1, double& f2) {
  sum += v;
  mn = fmin(mn, v);
  mx = fmax(mx, v);
  if (a.kind == SSK_POOL_DW) {
    const double wt = powp(__dsub_rn(1.0, v), a.p);
    f1 += wt;
    f2 += __dmul_rn(wt, v);
  } else if (a.kind == SSK_POOL_MINK) {
    f1 += powp(__dsub_rn(1.0, v), a.p);
  } else if (a.kind == SSK_POOL_LW) {
    const double mu = (double)ab[ao];
    const double wt = a.b == 0.0 ? (mu >= a.a ? 1.0 : 0.0) : fmin(fmax(__ddiv_rn(__dsub_rn(mu, a.a), a.b), 0.0), 1.0);
    f1 += __dmul_rn(wt, v);
  }
}

__device__ __forceinline__ double pass2_elem(const PoolArgs& a, double v, double c) {
  if (a.kind == SSK_POOL_COV) {
    const double d = __dsub_rn(v, c);
    return __dmul_rn(d, d);
  }
  if (a.kind == SSK_POOL_MD) return powp(fabs(__dsub_rn(v, c)), a.p);
  return v <= c ? __ddiv_rn(v, a.rs) : v;  // pp
}

template <typename T>
__device__ __forceinline__ const T* frame_vals(const PoolArgs& a, int frame) {
  return reinterpret_cast<const T*>(a.vals) + (long long)frame * a.fp;
}
template <typename T>
__device__ __forceinline__ const T* frame_aux(const PoolArgs& a, int frame) {
  return a.aux ? reinterpret_cast<const T*>(a.aux) + (long long)frame * a.afp : nullptr;
}

// pooled score from the folded sums (src/pooling.py:157-243 semantics)
template <typename T>
__device__ void finish(const PoolArgs& a, int frame, double sum, double mn, double mx, double f1, double f2,
                       double s2) {
  const double mean = __ddiv_rn(sum, a.cnt);
  double r = mean;
  switch (a.kind) {
    case SSK_POOL_COV:
      r = mean == 0.0 ? NAN : __ddiv_rn(__dsqrt_rn(__ddiv_rn(s2, a.cnt)), mean);
      break;
    case SSK_POOL_MD: {
      const double inner = powp(__ddiv_rn(s2, a.cnt), __ddiv_rn(1.0, a.p));
      r = a.o == 1.0 ? inner : pow(inner, a.o);
      break;
    }
    case SSK_POOL_FNS: {
      double q[3];
      for (int i = 0; i < 3; ++i)
        q[i] = np_lerp(rank_value<T>(a, frame, 2 * i), rank_value<T>(a, frame, 2 * i + 1), a.gamma[i]);
      r = __ddiv_rn(__dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(mn, q[0]), q[1]), q[2]), mx), 5.0);
      break;
    }
    case SSK_POOL_DW:
      r = f1 == 0.0 ? mean : __ddiv_rn(f2, f1);
      break;
    case SSK_POOL_MINK:
    case SSK_POOL_LW:
      r = __ddiv_rn(f1, a.cnt);
      break;
    case SSK_POOL_PP:
      r = (a.ps <= 0.0 || a.rs == 1.0) ? mean : __ddiv_rn(s2, a.cnt);
      break;
    case SSK_POOL_PCTL:
      r = np_lerp(rank_value<T>(a, frame, 0), rank_value<T>(a, frame, 1), a.gamma[0]);
      break;
    default:
      break;
  }
  a.out[frame] = r;
  if (a.mean) a.mean[frame] = mean;
}

// ---------------------------------------------------------------------------
// pass 1: sum, min, max and the kind's own sums
// ---------------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(PL_THREADS) pool_pass1_kernel(const __grid_constant__ PoolArgs a) {
  __shared__ double red[PL_THREADS / 32][NC1];
  const int frame = blockIdx.y, blk = blockIdx.x;
  if (blk == 0 && (int)threadIdx.x < a.nranks) {
    unsigned long long* s = a.sel + ((long long)frame * MAX_RANKS + threadIdx.x) * 2;
    s[0] = 0ull;
    s[1] = (unsigned long long)a.rank[threadIdx.x];
  }
  const T* vb = frame_vals<T>(a, frame);
  const T* ab = frame_aux<T>(a, frame);
  double sum = 0.0, mn = INFINITY, mx = -INFINITY, f1 = 0.0, f2 = 0.0;
  for_range(
      a, blk, [&](long long o) { return (double)vb[o]; },
      [&](double v, long long, long long ao, int) { pass1_elem<T>(a, ab, v, ao, sum, mn, mx, f1, f2); });
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  sum = warp_sum(sum);
  mn = warp_min(mn);
  mx = warp_max(mx);
  f1 = warp_sum(f1);
  f2 = warp_sum(f2);
  if (lane == 0) {
    red[warp][0] = sum;
    red[warp][1] = mn;
    red[warp][2] = mx;
    red[warp][3] = f1;
    red[warp][4] = f2;
  }
  __syncthreads();
  if (threadIdx.x < NC1) {
    const int c = threadIdx.x;
    double r = red[0][c];
    for (int wi = 1; wi < PL_THREADS / 32; ++wi)
      r = c == 1 ? fmin(r, red[wi][c]) : (c == 2 ? fmax(r, red[wi][c]) : r + red[wi][c]);
    a.part1[((long long)frame * a.nblk + blk) * NC1 + c] = r;
  }
}

// ---------------------------------------------------------------------------
// pass 2: sums around a per-map centre (mean for cov/md, the percentile cutoff for pp)
// ---------------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(PL_THREADS) pool_pass2_kernel(const __grid_constant__ PoolArgs a) {
  __shared__ double red[PL_THREADS / 32];
  __shared__ double centre_s;
  const int frame = blockIdx.y, blk = blockIdx.x;
  if (threadIdx.x < 32) {
    const double s = fold_sum(a.part1 + (long long)frame * a.nblk * NC1, a.nblk, NC1, 0);
    if (threadIdx.x == 0) {
      centre_s = a.kind == SSK_POOL_PP ? np_lerp(rank_value<T>(a, frame, 0), rank_value<T>(a, frame, 1), a.gamma[0])
                                       : __ddiv_rn(s, a.cnt);
    }
  }
  __syncthreads();
  const double c = centre_s;
  double acc = 0.0;
  const T* vb = frame_vals<T>(a, frame);
  for_range(
      a, blk, [&](long long o) { return (double)vb[o]; },
      [&](double v, long long, long long, int) { acc += pass2_elem(a, v, c); });
  acc = warp_sum(acc);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double r = red[0];
    for (int wi = 1; wi < PL_THREADS / 32; ++wi) r += red[wi];
    a.part2[(long long)frame * a.nblk + blk] = r;
  }
}

// ---------------------------------------------------------------------------
// radix select: histogram of the next SEL_BITS-wide digit of the keys that
// match each rank's prefix so far, then one block per map picks the digits
// ---------------------------------------------------------------------------
// Ranks whose key prefixes agree so far share one histogram (all of them in the first
// pass): rep[r] = first rank with the same prefix above bit `hi`.
template <typename K>
__device__ __forceinline__ int prefix_rep(const unsigned long long* pre, int r, int hi, int bits) {
  if (hi >= bits) return 0;
  for (int q = 0; q < r; ++q)
    if (((K)pre[q] >> hi) == ((K)pre[r] >> hi)) return q;
  return r;
}

template <typename T>
__global__ void __launch_bounds__(PL_THREADS) select_hist_kernel(const __grid_constant__ PoolArgs a, int hi,
                                                                 int width) {
  extern __shared__ unsigned int sh[];  // [nranks][SEL_BINS]
  __shared__ unsigned long long pre[MAX_RANKS];
  __shared__ int reps[MAX_RANKS], nrep;
  const int frame = blockIdx.y, blk = blockIdx.x;
  using K = typename Keys<T>::K;
  if ((int)threadIdx.x < a.nranks) pre[threadIdx.x] = a.sel[((long long)frame * MAX_RANKS + threadIdx.x) * 2];
  __syncthreads();
  if (threadIdx.x == 0) {
    int m = 0;
    for (int r = 0; r < a.nranks; ++r)
      if (prefix_rep<K>(pre, r, hi, Keys<T>::B) == r) reps[m++] = r;
    nrep = m;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nrep * SEL_BINS; i += PL_THREADS) sh[reps[i / SEL_BINS] * SEL_BINS + i % SEL_BINS] = 0u;
  __syncthreads();
  const int shift = hi - width;
  const K mask = (K)((1u << width) - 1u);
  const bool first = hi >= Keys<T>::B;
  const int nu = nrep;
  const T* vb = frame_vals<T>(a, frame);
  // quality maps crowd into a few leading digits (values near 1): when a whole warp's
  // candidates fall into one bin, one shared atomic adds the warp's count
  const unsigned lane = threadIdx.x & 31;
  for_range(a, blk, [&](long long o) { return vb[o]; }, [&](T raw, long long, long long, int) {
    const K key = Keys<T>::key(raw);
    const unsigned d = (unsigned)((key >> shift) & mask);
    const unsigned active = __activemask();
    const int leader = __ffs(active) - 1;
    const unsigned d0 = __shfl_sync(active, d, leader);
    for (int u = 0; u < nu; ++u) {
      const int r = reps[u];
      const bool hit = first || (key >> hi) == ((K)pre[r] >> hi);
      const unsigned hits = __ballot_sync(active, hit);
      if (!hits) continue;
      if (__all_sync(active, !hit || d == d0)) {
        if ((int)lane == leader) atomicAdd(&sh[r * SEL_BINS + d0], (unsigned)__popc(hits));
      } else if (hit) {
        atomicAdd(&sh[r * SEL_BINS + d], 1u);
      }
    }
  });
  __syncthreads();
  unsigned int* g = a.hist + (long long)frame * MAX_RANKS * SEL_BINS;
  for (int i = threadIdx.x; i < nrep * SEL_BINS; i += PL_THREADS) {
    const int j = reps[i / SEL_BINS] * SEL_BINS + i % SEL_BINS;
    const unsigned c = sh[j];
    if (c) atomicAdd(&g[j], c);
  }
}

template <typename T>
__global__ void __launch_bounds__(PL_THREADS) select_pick_kernel(const __grid_constant__ PoolArgs a, int shift,
                                                                 int hi) {
  __shared__ unsigned long long wtot[PL_THREADS / 32];
  __shared__ unsigned long long pre[MAX_RANKS];
  __shared__ int rep[MAX_RANKS];
  constexpr int PER = SEL_BINS / PL_THREADS;  // 8 bins per thread
  const int frame = blockIdx.x, t = threadIdx.x, lane = t & 31, warp = t >> 5;
  // histogram owner of every rank, from the prefixes before this digit is appended
  if (t < a.nranks) pre[t] = a.sel[((long long)frame * MAX_RANKS + t) * 2];
  __syncthreads();
  if (t < a.nranks) rep[t] = prefix_rep<typename Keys<T>::K>(pre, t, hi, Keys<T>::B);
  __syncthreads();
  for (int r = 0; r < a.nranks; ++r) {
    unsigned int* h = a.hist + ((long long)frame * MAX_RANKS + rep[r]) * SEL_BINS;
    unsigned long long* st = a.sel + ((long long)frame * MAX_RANKS + r) * 2;
    unsigned c[PER];
    unsigned long long s = 0;
#pragma unroll
    for (int j = 0; j < PER; ++j) {
      c[j] = h[t * PER + j];
      s += c[j];
    }
    // block exclusive scan of the per-thread totals (bins are in key order)
    unsigned long long incl = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    if (lane == 31) wtot[warp] = incl;
    // every thread reads the residual rank before the barrier: the owning thread
    // rewrites st[1] below, and no other thread may see the new value
    const unsigned long long k = st[1];
    SSK_JITTER(300);
    __syncthreads();
    SSK_JITTER(301);
    unsigned long long base = 0;
    for (int wi = 0; wi < warp; ++wi) base += wtot[wi];
    const unsigned long long excl = base + incl - s;
    if (s > 0 && k >= excl && k < excl + s) {
      unsigned long long cum = excl;
#pragma unroll
      for (int j = 0; j < PER; ++j) {
        if (k < cum + c[j]) {
          st[0] |= (unsigned long long)(t * PER + j) << shift;
          st[1] = k - cum;
          break;
        }
        cum += c[j];
      }
    }
    __syncthreads();
  }
  // clear every histogram for the next digit (shared ones are read by several ranks above)
  for (int i = t; i < a.nranks * SEL_BINS; i += PL_THREADS)
    a.hist[(long long)frame * MAX_RANKS * SEL_BINS + i] = 0u;
}

// ---------------------------------------------------------------------------
// finalize: one warp per map
// ---------------------------------------------------------------------------
template <typename T>
__global__ void pool_finalize_kernel(const __grid_constant__ PoolArgs a) {
  const int frame = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (frame >= a.n) return;
  const double* p1 = a.part1 + (long long)frame * a.nblk * NC1;
  const double sum = fold_sum(p1, a.nblk, NC1, 0);
  double mn = INFINITY, mx = -INFINITY;
  for (int i = lane; i < a.nblk; i += 32) {
    mn = fmin(mn, p1[(long long)i * NC1 + 1]);
    mx = fmax(mx, p1[(long long)i * NC1 + 2]);
  }
  mn = warp_min(mn);
  mx = warp_max(mx);
  const double f1 = fold_sum(p1, a.nblk, NC1, 3);
  const double f2 = fold_sum(p1, a.nblk, NC1, 4);
  const double s2 = a.pass2 ? fold_sum(a.part2 + (long long)frame * a.nblk, a.nblk, 1, 0) : 0.0;
  if (lane == 0) finish<T>(a, frame, sum, mn, mx, f1, f2, s2);
}

// ---------------------------------------------------------------------------
// small maps (one block per map, no order statistics): both passes and the
// final combination in one launch
// ---------------------------------------------------------------------------
constexpr int PS_THREADS = 512;

template <typename T>
__global__ void __launch_bounds__(PS_THREADS) pool_small_kernel(const __grid_constant__ PoolArgs a) {
  __shared__ double red[PS_THREADS / 32][NC1];
  __shared__ double tot[NC1];
  const int frame = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const T* vb = frame_vals<T>(a, frame);
  const T* ab = frame_aux<T>(a, frame);
  double sum = 0.0, mn = INFINITY, mx = -INFINITY, f1 = 0.0, f2 = 0.0;
  for_range<PS_THREADS>(
      a, 0, [&](long long o) { return (double)vb[o]; },
      [&](double v, long long, long long ao, int) { pass1_elem<T>(a, ab, v, ao, sum, mn, mx, f1, f2); });
  sum = warp_sum(sum);
  mn = warp_min(mn);
  mx = warp_max(mx);
  f1 = warp_sum(f1);
  f2 = warp_sum(f2);
  if (lane == 0) {
    red[warp][0] = sum;
    red[warp][1] = mn;
    red[warp][2] = mx;
    red[warp][3] = f1;
    red[warp][4] = f2;
  }
  __syncthreads();
  if (threadIdx.x < NC1) {
    const int c = threadIdx.x;
    double r = red[0][c];
    for (int wi = 1; wi < PS_THREADS / 32; ++wi)
      r = c == 1 ? fmin(r, red[wi][c]) : (c == 2 ? fmax(r, red[wi][c]) : r + red[wi][c]);
    tot[c] = r;
  }
  __syncthreads();
  double s2 = 0.0;
  if (a.pass2) {
    const double c = __ddiv_rn(tot[0], a.cnt);
    double acc = 0.0;
    for_range<PS_THREADS>(
        a, 0, [&](long long o) { return (double)vb[o]; },
        [&](double v, long long, long long, int) { acc += pass2_elem(a, v, c); });
    acc = warp_sum(acc);
    __syncthreads();
    if (lane == 0) red[warp][0] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
      s2 = red[0][0];
      for (int wi = 1; wi < PS_THREADS / 32; ++wi) s2 += red[wi][0];
    }
  }
  if (threadIdx.x == 0) finish<T>(a, frame, tot[0], tot[1], tot[2], tot[3], tot[4], s2);
}

// ---------------------------------------------------------------------------
// box_downsample: one thread per output sample.  Integer samples: exact block
// sums.  Float samples replay np.add.reduceat's rounding (rows of the block
// first, then columns): each run is first + pairwise(rest), numpy's pairwise
// summation (< 8 terms sequential, <= 128 terms eight interleaved partials);
// longer runs (factor > 129) fall back to sequential order.
// ---------------------------------------------------------------------------
template <typename GET>
__device__ __forceinline__ double np_pairwise(int n, GET get) {
  if (n < 8 || n > 128) {
    double r = 0.0;
    for (int i = 0; i < n; ++i) r = __dadd_rn(r, get(i));
    return r;
  }
  double r[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) r[j] = get(j);
  int i = 8;
  for (; i < n - (n % 8); i += 8) {
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], get(i + j));
  }
  double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                         __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
  for (; i < n; ++i) res = __dadd_rn(res, get(i));
  return res;
}

template <typename GET>
__device__ __forceinline__ double np_reduce(int m, GET get) {
  const double first = get(0);
  return m > 1 ? __dadd_rn(first, np_pairwise(m - 1, [&](int i) { return get(i + 1); })) : first;
}

template <typename TS, typename TD>
__global__ void __launch_bounds__(128) box_downsample_kernel(const unsigned char* __restrict__ src_r,
                                                             const unsigned char* __restrict__ src_d,
                                                             long long srp, long long sfp, int h, int w, int f,
                                                             unsigned char* __restrict__ dst_r,
                                                             unsigned char* __restrict__ dst_d, long long drp,
                                                             long long dfp, int wo) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y;
  const int frame = blockIdx.z >> 1, img = blockIdx.z & 1;
  if (x >= wo) return;
  const TS* s = reinterpret_cast<const TS*>(img ? src_d : src_r) + (long long)frame * sfp;
  TD* d = reinterpret_cast<TD*>(img ? dst_d : dst_r) + (long long)frame * dfp + (long long)y * drp + x;
  const int r0 = y * f, r1 = min(r0 + f, h), c0 = x * f, c1 = min(c0 + f, w);
  double value;
  if constexpr (std::is_integral<TS>::value) {
    unsigned long long acc = 0;
    for (int r = r0; r < r1; ++r) {
      const TS* row = s + (long long)r * srp;
      for (int c = c0; c < c1; ++c) acc += row[c];
    }
    if constexpr (!std::is_floating_point<TD>::value) {
      *d = (TD)acc;
      return;
    }
    value = (double)acc;
  } else {
    value = np_reduce(c1 - c0, [&](int j) {
      return np_reduce(r1 - r0, [&](int i) { return (double)s[(long long)(r0 + i) * srp + c0 + j]; });
    });
  }
  if constexpr (std::is_floating_point<TD>::value) *d = (TD)__ddiv_rn(value, (double)((r1 - r0) * (c1 - c0)));
}

// Vector path (the resolution-adaptation hot case): integer samples, a power-of-two
// factor F that divides a 16-byte vector, frames tiled by F, 16-byte aligned rows.
// A thread owns one vector column of F input rows: F independent 16-byte loads,
// V/F block sums out.
template <typename TS, typename TD, int F>
__global__ void __launch_bounds__(128) box_down_vec_kernel(const unsigned char* __restrict__ src_r,
                                                           const unsigned char* __restrict__ src_d, long long srp,
                                                           long long sfp, int w, unsigned char* __restrict__ dst_r,
                                                           unsigned char* __restrict__ dst_d, long long drp,
                                                           long long dfp, int nvec) {
  constexpr int V = 16 / (int)sizeof(TS);
  constexpr int NO = V / F;
  const int vx = blockIdx.x * blockDim.x + threadIdx.x;
  if (vx >= nvec) return;
  const int y = blockIdx.y;
  const int frame = blockIdx.z >> 1, img = blockIdx.z & 1;
  const TS* s = reinterpret_cast<const TS*>(img ? src_d : src_r) + (long long)frame * sfp +
                (long long)(y * F) * srp + (long long)vx * V;
  uint32_t acc[NO];
#pragma unroll
  for (int j = 0; j < NO; ++j) acc[j] = 0u;
  const int nvalid = min(V, w - vx * V);  // a multiple of F (w % F == 0)
  if (nvalid == V) {
    uint4 q[F];
#pragma unroll
    for (int r = 0; r < F; ++r) q[r] = __ldg(reinterpret_cast<const uint4*>(s + (long long)r * srp));
#pragma unroll
    for (int r = 0; r < F; ++r) {
      const TS* e = reinterpret_cast<const TS*>(&q[r]);
#pragma unroll
      for (int i = 0; i < V; ++i) acc[i / F] += (uint32_t)e[i];
    }
  } else {
    for (int r = 0; r < F; ++r)
      for (int i = 0; i < nvalid; ++i) acc[i / F] += (uint32_t)s[(long long)r * srp + i];
  }
  TD* d = reinterpret_cast<TD*>(img ? dst_d : dst_r) + (long long)frame * dfp + (long long)y * drp +
          (long long)vx * NO;
  const int nout = nvalid / F;
#pragma unroll
  for (int j = 0; j < NO; ++j)
    if (j < nout) d[j] = (TD)acc[j];
}

template <typename TS, typename TD, int F>
int launch_down_vec(const ssk_planes* p, const unsigned char* sr, const unsigned char* sd, unsigned char* r,
                    unsigned char* d, long long drp, long long dfp, int ho, cudaStream_t st) {
  constexpr int V = 16 / (int)sizeof(TS);
  const int nvec = (p->w + V - 1) / V;
  const dim3 grid((nvec + 127) / 128, ho, 2 * p->n);
  box_down_vec_kernel<TS, TD, F><<<grid, 128, 0, st>>>(sr, sd, p->row_pitch, p->frame_pitch, p->w, r, d, drp, dfp,
                                                       nvec);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? SSK_OK : SSK_E_CUDA;
}

template <typename TS, typename TD>
int try_down_vec(const ssk_planes* p, int f, const unsigned char* sr, const unsigned char* sd, unsigned char* r,
                 unsigned char* d, long long drp, long long dfp, int ho, cudaStream_t st) {
  constexpr int V = 16 / (int)sizeof(TS);
  const bool aligned = !((reinterpret_cast<uintptr_t>(sr) | reinterpret_cast<uintptr_t>(sd)) & 15) &&
                       !((p->row_pitch * (long long)sizeof(TS)) & 15) && !((p->frame_pitch * (long long)sizeof(TS)) & 15);
  if (!aligned || p->h % f || p->w % f) return 1;
  switch (f) {
    case 2: return launch_down_vec<TS, TD, 2>(p, sr, sd, r, d, drp, dfp, ho, st);
    case 4: return V >= 4 ? launch_down_vec<TS, TD, (V >= 4 ? 4 : 1)>(p, sr, sd, r, d, drp, dfp, ho, st) : 1;
    case 8: return V >= 8 ? launch_down_vec<TS, TD, (V >= 8 ? 8 : 1)>(p, sr, sd, r, d, drp, dfp, ho, st) : 1;
    case 16: return V >= 16 ? launch_down_vec<TS, TD, (V >= 16 ? 16 : 1)>(p, sr, sd, r, d, drp, dfp, ho, st) : 1;
    default: return 1;
  }
}

template <typename TS>
int launch_box_downsample_t(const ssk_planes* p, int f, void* dr, void* dd, int dst_dtype, long long drp,
                            long long dfp, int ho, int wo, cudaStream_t st) {
  const dim3 grid((wo + 127) / 128, ho, 2 * p->n);
  const auto* sr = static_cast<const unsigned char*>(p->ref);
  const auto* sd = static_cast<const unsigned char*>(p->dist);
  auto* r = static_cast<unsigned char*>(dr);
  auto* d = static_cast<unsigned char*>(dd);
  if constexpr (std::is_integral<TS>::value) {
    if (dst_dtype == SSK_U16 || dst_dtype == SSK_U32) {
      const int rc = dst_dtype == SSK_U16 ? try_down_vec<TS, uint16_t>(p, f, sr, sd, r, d, drp, dfp, ho, st)
                                          : try_down_vec<TS, uint32_t>(p, f, sr, sd, r, d, drp, dfp, ho, st);
      if (rc <= 0) return rc;  // launched (or failed); 1 = not eligible, use the generic kernel
    }
  }
  switch (dst_dtype) {
    case SSK_F64:
      box_downsample_kernel<TS, double><<<grid, 128, 0, st>>>(sr, sd, p->row_pitch, p->frame_pitch, p->h, p->w, f,
                                                              r, d, drp, dfp, wo);
      break;
    case SSK_U16:
      box_downsample_kernel<TS, uint16_t><<<grid, 128, 0, st>>>(sr, sd, p->row_pitch, p->frame_pitch, p->h, p->w,
                                                                f, r, d, drp, dfp, wo);
      break;
    case SSK_U32:
      box_downsample_kernel<TS, uint32_t><<<grid, 128, 0, st>>>(sr, sd, p->row_pitch, p->frame_pitch, p->h, p->w,
                                                                f, r, d, drp, dfp, wo);
      break;
    default:
      return SSK_E_ARG;
  }
  note_launch();
  return cudaGetLastError() == cudaSuccess ? SSK_OK : SSK_E_CUDA;
}

// ---------------------------------------------------------------------------
// moment pooling: CoV / MD(p = 2) from the [n][4] sums of an SSK_WANT_Q2 pass
// (sum q, sum l, sum cs, sum q^2), one thread per frame
// ---------------------------------------------------------------------------
__global__ void pool_moments_kernel(const double* __restrict__ sums, int n, double count, int kind, double o,
                                    double* __restrict__ out, double* __restrict__ means) {
  const int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= n) return;
  const double* s = sums + (long long)f * 4;
  const double mq = __ddiv_rn(s[0], count);
  const double var = fmax(__dsub_rn(__ddiv_rn(s[3], count), __dmul_rn(mq, mq)), 0.0);
  const double sd = __dsqrt_rn(var);
  double r;
  if (kind == SSK_POOL_COV) {
    r = mq == 0.0 ? NAN : __ddiv_rn(sd, mq);
  } else {
    r = o == 1.0 ? sd : pow(sd, o);
  }
  out[f] = r;
  if (means) {
    means[(long long)f * 3] = mq;
    means[(long long)f * 3 + 1] = __ddiv_rn(s[1], count);
    means[(long long)f * 3 + 2] = __ddiv_rn(s[2], count);
  }
}

// ---- pooling plan ----
struct PoolPlan {
  PoolArgs a{};
  int passes = 0;  // radix-select digit passes (0: no order statistics)
  size_t part1 = 0, part2 = 0, sel = 0, hist = 0, total = 0;
};

inline size_t al(size_t x) { return (x + 255) / 256 * 256; }

int plan_pool(const ssk_maps* m, const ssk_pooler* pl, PoolPlan& P) {
  if (!m || !pl || !m->values) return SSK_E_ARG;
  if (m->dtype != SSK_F32 && m->dtype != SSK_F64) return SSK_E_ARG;
  if (m->n < 1 || m->n > 65535 || m->h < 1 || m->w < 1) return SSK_E_ARG;
  if (m->row_pitch < m->w || m->frame_pitch < m->row_pitch * (int64_t)m->h) return SSK_E_ARG;
  const int kind = pl->kind;
  if (kind < SSK_POOL_AM || kind > SSK_POOL_PCTL) return SSK_E_ARG;
  if ((kind == SSK_POOL_MD || kind == SSK_POOL_DW || kind == SSK_POOL_MINK) && !(pl->p > 0)) return SSK_E_ARG;
  if (kind == SSK_POOL_MD && !(pl->o > 0)) return SSK_E_ARG;
  if (kind == SSK_POOL_LW) {
    if (!(pl->b >= 0) || !m->aux) return SSK_E_ARG;
    if (m->aux_row_pitch < m->w || m->aux_frame_pitch < m->aux_row_pitch * (int64_t)m->h) return SSK_E_ARG;
  }
  if (kind == SSK_POOL_PP && !(pl->ps >= 0 && pl->ps <= 100 && pl->rs >= 1)) return SSK_E_ARG;
  if (kind == SSK_POOL_PCTL && !(pl->ps >= 0 && pl->ps <= 100)) return SSK_E_ARG;
  PoolArgs& a = P.a;
  a.vals = static_cast<const unsigned char*>(m->values);
  a.aux = static_cast<const unsigned char*>(m->aux);
  a.rp = m->row_pitch;
  a.fp = m->frame_pitch;
  a.arp = m->aux_row_pitch;
  a.afp = m->aux_frame_pitch;
  a.n = m->n;
  a.h = m->h;
  a.w = m->w;
  a.flat = (m->row_pitch == m->w && (!m->aux || m->aux_row_pitch == m->w)) ? 1 : 0;
  const long long count = (long long)m->h * m->w;
  a.cnt = (double)count;
  // one block per map up to 32K samples (single-launch small-map path), else ~16K
  // samples per block; whole rows, geometry-only (independent of the batch)
  long long nblk = count <= 32768 ? 1 : (count + 16383) / 16384;
  if (nblk > m->h) nblk = m->h;
  if (nblk > 1024) nblk = 1024;
  a.nblk = (int)(nblk < 1 ? 1 : nblk);
  a.kind = kind;
  a.p = pl->p;
  a.o = pl->o;
  a.a = pl->a;
  a.b = pl->b;
  a.ps = pl->ps;
  a.rs = pl->rs;
  // quantiles: np.percentile(v, q) 'linear': virtual index (n-1)*q/100, neighbours
  // floor / floor+1 (both clamped to n-1 at the top), gamma = index - floor
  double qs[3];
  int nq = 0;
  if (kind == SSK_POOL_FNS) {
    qs[0] = 25.0 / 100.0;
    qs[1] = 50.0 / 100.0;
    qs[2] = 75.0 / 100.0;
    nq = 3;
  } else if ((kind == SSK_POOL_PP && !(pl->ps <= 0.0 || pl->rs == 1.0)) || kind == SSK_POOL_PCTL) {
    qs[0] = pl->ps / 100.0;
    nq = 1;
  }
  a.nq = nq;
  a.nranks = 2 * nq;
  for (int i = 0; i < nq; ++i) {
    const double vi = (double)(count - 1) * qs[i];
    double lo = std::floor(vi);
    long long rlo = (long long)lo, rhi = rlo + 1;
    if (vi >= (double)(count - 1)) {
      rlo = rhi = count - 1;
      lo = -1.0;  // numpy indexes the last element as -1 here; gamma is moot (equal ends)
    }
    a.rank[2 * i] = rlo;
    a.rank[2 * i + 1] = rhi;
    a.gamma[i] = vi - lo;
  }
  a.pass2 = (kind == SSK_POOL_COV || kind == SSK_POOL_MD || (kind == SSK_POOL_PP && nq == 1)) ? 1 : 0;
  P.passes = nq ? ((m->dtype == SSK_F64 ? 64 : 32) + SEL_BITS - 1) / SEL_BITS : 0;
  P.part1 = al((size_t)a.n * a.nblk * NC1 * sizeof(double));
  P.part2 = al((size_t)a.n * a.nblk * sizeof(double));
  P.sel = al((size_t)a.n * MAX_RANKS * 2 * sizeof(unsigned long long));
  P.hist = nq ? al((size_t)a.n * MAX_RANKS * SEL_BINS * sizeof(unsigned int)) : 0;
  P.total = P.part1 + P.part2 + P.sel + P.hist;
  return SSK_OK;
}

template <typename T>
int run_pool(PoolPlan& P, cudaStream_t st) {
  PoolArgs& a = P.a;
  if (a.nblk == 1 && P.passes == 0) {
    pool_small_kernel<T><<<a.n, PS_THREADS, 0, st>>>(a);
    note_launch();
    return cudaGetLastError() == cudaSuccess ? SSK_OK : SSK_E_CUDA;
  }
  const dim3 grid(a.nblk, a.n);
  pool_pass1_kernel<T><<<grid, PL_THREADS, 0, st>>>(a);
  note_launch();
  if (P.passes) {
    if (cudaMemsetAsync(a.hist, 0, P.hist, st) != cudaSuccess) return SSK_E_CUDA;
    const int B = sizeof(T) * 8;
    const size_t smem = (size_t)a.nranks * SEL_BINS * sizeof(unsigned int);
    if (cudaFuncSetAttribute(select_hist_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
        cudaSuccess)
      return SSK_E_CUDA;
    // histogram blocks cover ~64K samples each: every block zeroes and flushes whole
    // 2048-bin histograms, so fewer, longer blocks amortise that fixed cost
    PoolArgs as = a;
    long long sb = ((long long)a.h * a.w + 65535) / 65536;
    as.nblk = (int)(sb < 1 ? 1 : (sb > a.h ? a.h : sb));
    const dim3 sgrid(as.nblk, a.n);
    for (int hi = B; hi > 0; hi -= SEL_BITS) {
      const int width = hi < SEL_BITS ? hi : SEL_BITS;
      select_hist_kernel<T><<<sgrid, PL_THREADS, smem, st>>>(as, hi, width);
      select_pick_kernel<T><<<a.n, PL_THREADS, 0, st>>>(a, hi - width, hi);
      note_launch(2);
    }
  }
  if (a.pass2) {
    pool_pass2_kernel<T><<<grid, PL_THREADS, 0, st>>>(a);
    note_launch();
  }
  pool_finalize_kernel<T><<<(a.n * 32 + 127) / 128, 128, 0, st>>>(a);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? SSK_OK : SSK_E_CUDA;
}

}  // namespace
}  // namespace ssk

using namespace ssk;

extern "C" {

int ssk_box_downsample(const ssk_planes* src, int factor, void* d_dst_ref, void* d_dst_dist, int dst_dtype,
                       int64_t dst_row_pitch, int64_t dst_frame_pitch, void* stream) {
  if (!src || !src->ref || !src->dist || !d_dst_ref || !d_dst_dist) return SSK_E_ARG;
  if (esize_of(src->dtype) == 0 || src->n < 1 || src->n > 32767 || src->h < 1 || src->w < 1) return SSK_E_ARG;
  if (src->row_pitch < src->w || src->frame_pitch < src->row_pitch * (int64_t)src->h) return SSK_E_ARG;
  if (factor < 1 || factor > 4096) return SSK_E_ARG;
  const int ho = (src->h + factor - 1) / factor, wo = (src->w + factor - 1) / factor;
  if (ho > 65535 || dst_row_pitch < wo || dst_frame_pitch < dst_row_pitch * (int64_t)ho) return SSK_E_ARG;
  const bool integer = src->dtype == SSK_U8 || src->dtype == SSK_U16 || src->dtype == SSK_U32;
  if (dst_dtype == SSK_U16 || dst_dtype == SSK_U32) {
    if (!integer || src->h % factor || src->w % factor) return SSK_E_ARG;
    const double stored_max = (std::ldexp(1.0, src->bit_depth) - 1.0) * std::ldexp(1.0, src->scale_log2);
    const double lim = dst_dtype == SSK_U16 ? 65535.0 : 4294967295.0;
    if ((double)factor * factor * stored_max > lim) return SSK_E_ARG;
  } else if (dst_dtype != SSK_F64) {
    return SSK_E_ARG;
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  switch (src->dtype) {
    case SSK_U8:
      return launch_box_downsample_t<uint8_t>(src, factor, d_dst_ref, d_dst_dist, dst_dtype, dst_row_pitch,
                                              dst_frame_pitch, ho, wo, st);
    case SSK_U16:
      return launch_box_downsample_t<uint16_t>(src, factor, d_dst_ref, d_dst_dist, dst_dtype, dst_row_pitch,
                                               dst_frame_pitch, ho, wo, st);
    case SSK_U32:
      return launch_box_downsample_t<uint32_t>(src, factor, d_dst_ref, d_dst_dist, dst_dtype, dst_row_pitch,
                                               dst_frame_pitch, ho, wo, st);
    case SSK_F32:
      return launch_box_downsample_t<float>(src, factor, d_dst_ref, d_dst_dist, dst_dtype, dst_row_pitch,
                                            dst_frame_pitch, ho, wo, st);
    case SSK_F64:
      return launch_box_downsample_t<double>(src, factor, d_dst_ref, d_dst_dist, dst_dtype, dst_row_pitch,
                                             dst_frame_pitch, ho, wo, st);
    default:
      return SSK_E_ARG;
  }
}

int ssk_pool_moments(const double* d_sums, int n, double count, const ssk_pooler* pool, double* d_out,
                     double* d_means, void* stream) {
  if (!d_sums || !d_out || !pool || n < 1 || !(count > 0)) return SSK_E_ARG;
  const bool md2 = pool->kind == SSK_POOL_MD && pool->p == 2.0 && pool->o > 0;
  if (pool->kind != SSK_POOL_COV && !md2) return SSK_E_ARG;
  pool_moments_kernel<<<(n + 127) / 128, 128, 0, static_cast<cudaStream_t>(stream)>>>(d_sums, n, count, pool->kind,
                                                                                     pool->o, d_out, d_means);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? SSK_OK : SSK_E_CUDA;
}

size_t ssk_pool_workspace_bytes(const ssk_maps* m, const ssk_pooler* pool) {
  PoolPlan P;
  if (plan_pool(m, pool, P) != SSK_OK) return 0;
  return P.total;
}

int ssk_pool_spatial(const ssk_maps* m, const ssk_pooler* pool, double* d_out, double* d_mean, void* d_workspace,
                     size_t workspace_bytes, void* stream) {
  PoolPlan P;
  const int rc = plan_pool(m, pool, P);
  if (rc) return rc;
  if (!d_out) return SSK_E_ARG;
  if (!d_workspace || workspace_bytes < P.total) return SSK_E_WORKSPACE;
  char* ws = static_cast<char*>(d_workspace);
  P.a.part1 = reinterpret_cast<double*>(ws);
  P.a.part2 = reinterpret_cast<double*>(ws + P.part1);
  P.a.sel = reinterpret_cast<unsigned long long*>(ws + P.part1 + P.part2);
  P.a.hist = P.hist ? reinterpret_cast<unsigned int*>(ws + P.part1 + P.part2 + P.sel) : nullptr;
  P.a.out = d_out;
  P.a.mean = d_mean;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  return m->dtype == SSK_F64 ? run_pool<double>(P, st) : run_pool<float>(P, st);
}

}  // extern "C"
