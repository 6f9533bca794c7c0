// numpy-order sums for the per-map pooling API (pool_spatial, mssim): bit-identical to
// the reference's numpy reductions.
//
// np.mean / np.sum / np.std of a contiguous float64 array reduce with numpy's pairwise
// summation (numpy/_core/src/umath/loops_utils.h.src, PW_BLOCKSIZE = 128): a node of n
// elements is summed sequentially (n < 8), with eight interleaved accumulators combined as
// ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) plus a sequential tail (n <= 128), or split at
// n2 = n/2 rounded down to a multiple of 8 into two halves added left + right; the
// reduction starts from 0.0 (tools/ and tests/ pin the emulation against numpy).  Every
// pooler of src/pooling.py:157-243 is an elementwise fp64 expression of the map followed
// by such a reduction, then scalar arithmetic; this kernel evaluates the expression with
// numpy's elementwise semantics (IEEE ops in the same order; `**` with numpy's fast scalar
// powers) and the reduction in numpy's order, so the host's final scalar step sees the
// very same sums the reference computes.
//
// The recursion's top d levels (d <= 15) are a complete binary tree (every node there has
// more than 128 elements): pass 1 gives each of the 2^d depth-d subtrees of a map to one
// thread, which sums it with the sequential recursion; pass 2 (one block per map) combines
// the tree level by level, left + right, exactly as the recursion would.
#include "common.cuh"
#include "kernels.h"

namespace ssk {
namespace {

constexpr int PX_THREADS = 1024;
constexpr int PX_MAX_DEPTH = 15;                                  // <= 32768 subtrees per map
constexpr int PX_PER_THREAD = (1 << (PX_MAX_DEPTH - 1)) / PX_THREADS;  // pairs per thread, widest level

struct ExactArgs {
  const unsigned char* values;
  const unsigned char* aux;
  int f32;                 // values / aux stored as float32 (widened exactly)
  int n, h, w;
  long long row_pitch, frame_pitch, aux_row_pitch, aux_frame_pitch;  // elements
  int expr;
  double p, a, b;
  const double* c;         // per-map centre (nullable)
  double* out;
};

// x ** p with numpy's fast scalar-power cases; small integer exponents correctly rounded
// through double-double products (numpy calls libm pow, correctly rounded in practice)
__device__ __forceinline__ void dd_mul(double ah, double al, double bh, double bl, double& rh, double& rl) {
  const double p = ah * bh;
  const double e = fma(ah, bh, -p);
  const double t = e + (ah * bl + al * bh);
  rh = p + t;
  rl = t - (rh - p);
}
__device__ double np_power(double x, double p) {
  if (p == 2.0) return __dmul_rn(x, x);
  if (p == 1.0) return x;
  if (p == 0.5) return __dsqrt_rn(x);
  if (p == -1.0) return __drcp_rn(x);
  if (p == 0.0) return 1.0;
  if (p == floor(p) && p >= 3.0 && p <= 64.0 && isfinite(x)) {
    int k = (int)p;
    double rh = 1.0, rl = 0.0, bh = x, bl = 0.0;
    while (k) {
      if (k & 1) dd_mul(rh, rl, bh, bl, rh, rl);
      k >>= 1;
      if (k) dd_mul(bh, bl, bh, bl, bh, bl);
    }
    return rh + rl;
  }
  return pow(x, p);
}

struct Elem {
  const ExactArgs* a;
  const unsigned char* v;
  const unsigned char* x;  // aux
  double c;
  __device__ double load(const unsigned char* base, long long off) const {
    return a->f32 ? (double)reinterpret_cast<const float*>(base)[off] : reinterpret_cast<const double*>(base)[off];
  }
  __device__ double operator()(long long i) const {
    const long long r = i / a->w, col = i - r * a->w;
    const double v0 = load(v, r * a->row_pitch + col);
    switch (a->expr) {
      case SSK_PW_V: return v0;
      case SSK_PW_SQDEV: {
        const double d = __dsub_rn(v0, c);
        return __dmul_rn(d, d);
      }
      case SSK_PW_ABSDEV_P: return np_power(fabs(__dsub_rn(v0, c)), a->p);
      case SSK_PW_ONEMINUS_P: return np_power(__dsub_rn(1.0, v0), a->p);
      case SSK_PW_DW_NUM: return __dmul_rn(np_power(__dsub_rn(1.0, v0), a->p), v0);
      case SSK_PW_PP: return v0 <= c ? __ddiv_rn(v0, a->p) : v0;
      case SSK_PW_LW: {
        const double mu = load(x, r * a->aux_row_pitch + col);
        double wgt;
        if (a->b == 0.0) {
          wgt = mu >= a->a ? 1.0 : 0.0;
        } else {
          wgt = __ddiv_rn(__dsub_rn(mu, a->a), a->b);
          wgt = fmin(fmax(wgt, 0.0), 1.0);  // np.clip(., 0, 1)
        }
        return __dmul_rn(wgt, v0);
      }
      default: return 0.0;
    }
  }
};

// numpy's pairwise_sum over elements [off, off + n)
__device__ double pairwise(const Elem& f, long long off, long long n) {
  if (n < 8) {
    double res = 0.0;
    for (long long i = 0; i < n; ++i) res = __dadd_rn(res, f(off + i));
    return res;
  }
  if (n <= 128) {
    double r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = f(off + j);
    long long i = 8;
    for (; i < n - (n % 8); i += 8) {
#pragma unroll
      for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], f(off + i + j));
    }
    double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                           __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    for (; i < n; ++i) res = __dadd_rn(res, f(off + i));
    return res;
  }
  long long n2 = n / 2;
  n2 -= n2 % 8;
  return __dadd_rn(pairwise(f, off, n2), pairwise(f, off + n2, n - n2));
}

// depth of the complete top tree: every node above it has more than 128 elements
__host__ __device__ inline int top_depth(long long n) {
  int d = 0;
  while (d < PX_MAX_DEPTH && (n >> (d + 1)) > 256) ++d;
  return d;
}

// pass 1: thread t < 2^d of a map sums its depth-d subtree (descend: bit lv of t picks the half)
__global__ void __launch_bounds__(256) pairwise_leaves_kernel(const __grid_constant__ ExactArgs a, double* ws,
                                                              long long ws_stride) {
  const int map = blockIdx.y;
  const long long n = (long long)a.h * a.w;
  const int d = top_depth(n);
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (1LL << d)) return;
  Elem f{&a, a.values + (long long)map * a.frame_pitch * (a.f32 ? 4 : 8),
         a.aux ? a.aux + (long long)map * a.aux_frame_pitch * (a.f32 ? 4 : 8) : nullptr, a.c ? a.c[map] : 0.0};
  long long off = 0, len = n;
  for (int lv = d - 1; lv >= 0; --lv) {
    long long n2 = len / 2;
    n2 -= n2 % 8;
    if ((t >> lv) & 1) {
      off += n2;
      len -= n2;
    } else {
      len = n2;
    }
  }
  ws[map * ws_stride + t] = pairwise(f, off, len);
}

// pass 2: one block per map combines the top tree level by level, left + right, in place
__global__ void __launch_bounds__(PX_THREADS) pairwise_combine_kernel(const __grid_constant__ ExactArgs a,
                                                                      double* ws, long long ws_stride) {
  const int map = blockIdx.x;
  const int d = top_depth((long long)a.h * a.w);
  double* v = ws + map * ws_stride;
  for (long long width = (1LL << d) >> 1; width >= 1; width >>= 1) {
    // read every pair of this level before anyone overwrites the front of the array
    double sums[PX_PER_THREAD];
    int k = 0;
    for (long long j = threadIdx.x; j < width; j += PX_THREADS, ++k) sums[k] = __dadd_rn(v[2 * j], v[2 * j + 1]);
    __syncthreads();
    k = 0;
    for (long long j = threadIdx.x; j < width; j += PX_THREADS, ++k) v[j] = sums[k];
    __syncthreads();
  }
  if (threadIdx.x == 0) a.out[map] = __dadd_rn(0.0, v[0]);  // np.add.reduce starts from 0.0
}

}  // namespace

size_t pairwise_workspace_bytes(const ssk_maps* m) {
  return (size_t)m->n * ((size_t)1 << top_depth((long long)m->h * m->w)) * sizeof(double);
}

int launch_pairwise_maps(const ssk_maps* m, int expr, double p, double a, double b, const double* d_c,
                         double* d_out, void* d_ws, cudaStream_t st) {
  ExactArgs x{};
  x.values = static_cast<const unsigned char*>(m->values);
  x.aux = static_cast<const unsigned char*>(m->aux);
  x.f32 = m->dtype == SSK_F32;
  x.n = m->n;
  x.h = m->h;
  x.w = m->w;
  x.row_pitch = m->row_pitch;
  x.frame_pitch = m->frame_pitch;
  x.aux_row_pitch = m->aux_row_pitch;
  x.aux_frame_pitch = m->aux_frame_pitch;
  x.expr = expr;
  x.p = p;
  x.a = a;
  x.b = b;
  x.c = d_c;
  x.out = d_out;
  const long long leaves = 1LL << top_depth((long long)m->h * m->w);
  double* ws = static_cast<double*>(d_ws);
  pairwise_leaves_kernel<<<dim3((unsigned)((leaves + 255) / 256), (unsigned)m->n), 256, 0, st>>>(x, ws, leaves);
  note_launch();
  if (cudaGetLastError() != cudaSuccess) return SSK_E_CUDA;
  pairwise_combine_kernel<<<m->n, PX_THREADS, 0, st>>>(x, ws, leaves);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? SSK_OK : SSK_E_CUDA;
}

}  // namespace ssk
