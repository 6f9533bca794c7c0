// Colorimetric similarity models on the device (src/color.py:27-371):
//   ssk_color_convert  BT.709 RGB <-> YCbCr (4:2:0 nearest upsampling), luma,
//                      HSV hue plane, CIELAB embedding -- float64 planes out,
//                      numpy's expression order replayed with IEEE intrinsics
//   ssk_qssim          quaternion SSIM (qssim, src/color.py:181-256): twelve
//                      windowed means per anchor in the reference's (m, n)
//                      accumulation order, then the quaternion modulus terms
//   ssk_delta_e        CIELAB difference with the opponent-space chroma
//                      smoothing (delta_e_map / cmssim weights, :263-334),
//                      sampled at the window centres of an SSIM grid
#include <cmath>
#include <cstring>

#include "common.cuh"
#include "kernels.h"

namespace ssk {
namespace {

constexpr double KR = 0.213, KG = 0.715, KB = 0.072;
constexpr double CB_SCALE = 0.539, CR_SCALE = 0.635;
__constant__ double c_rgb2xyz[9] = {0.4124564, 0.3575761, 0.1804375, 0.2126729, 0.7151522,
                                    0.0721750, 0.0193339, 0.1191920, 0.9503041};
__constant__ double c_xyz2q[9] = {0.279, 0.72, -0.107, -0.449, 0.29, -0.077, 0.086, -0.59, 0.501};
__constant__ double c_q2xyz[9] = {0.6204, -1.8704, -0.1553, 1.3661, 0.9316, 0.4339, 1.5013, 1.4176, 2.5331};
__constant__ double c_d65[3] = {0.95047, 1.0, 1.08883};
constexpr int SMOOTH_K = 13;  // _smooth: sigma 2, 13 taps, reflect padding (src/color.py:263-273)

struct ColorIn {
  const unsigned char* ch[3];
  long long rp[3], fp[3];  // elements
  int dtype, space, sub420, n, h, w;
  double peak;
};

__device__ __forceinline__ double sample_at(const unsigned char* base, int dtype, long long idx) {
  switch (dtype) {
    case SSK_U8: return (double)base[idx];
    case SSK_U16: return (double)reinterpret_cast<const uint16_t*>(base)[idx];
    case SSK_F32: return (double)reinterpret_cast<const float*>(base)[idx];
    default: return reinterpret_cast<const double*>(base)[idx];
  }
}

// channel c at luma-grid pixel (y, x); 4:2:0 chroma by nearest upsampling (repeat 2x2)
__device__ __forceinline__ double chan(const ColorIn& in, int c, int f, int y, int x) {
  if (c > 0 && in.sub420) {
    y >>= 1;
    x >>= 1;
  }
  return sample_at(in.ch[c], in.dtype, (long long)f * in.fp[c] + (long long)y * in.rp[c] + x);
}

__device__ __forceinline__ double clip(double v, double lo, double hi) { return fmin(fmax(v, lo), hi); }

// BT.709 YCbCr (offset L/2) -> RGB, clamped (ycbcr_bt709_to_rgb, src/color.py:76-89)
__device__ __forceinline__ void ycc_to_rgb(double y, double cb, double cr, double peak, double& r, double& g,
                                           double& b) {
  const double half = __ddiv_rn(peak, 2.0);
  const double bb = __dadd_rn(__ddiv_rn(__dsub_rn(cb, half), CB_SCALE), y);
  const double rr = __dadd_rn(__ddiv_rn(__dsub_rn(cr, half), CR_SCALE), y);
  const double gg = __ddiv_rn(__dsub_rn(__dsub_rn(y, __dmul_rn(KR, rr)), __dmul_rn(KB, bb)), KG);
  r = clip(rr, 0.0, peak);
  g = clip(gg, 0.0, peak);
  b = clip(bb, 0.0, peak);
}

__device__ __forceinline__ double luma709(double r, double g, double b) {
  return __dadd_rn(__dadd_rn(__dmul_rn(KR, r), __dmul_rn(KG, g)), __dmul_rn(KB, b));
}

// RGB of pixel (y, x) as float64 (converting YCbCr frames first)
__device__ __forceinline__ void rgb_at(const ColorIn& in, int f, int y, int x, double& r, double& g, double& b) {
  const double c0 = chan(in, 0, f, y, x), c1 = chan(in, 1, f, y, x), c2 = chan(in, 2, f, y, x);
  if (in.space == SSK_SPACE_YCBCR) {
    ycc_to_rgb(c0, c1, c2, in.peak, r, g, b);
  } else {
    r = c0;
    g = c1;
    b = c2;
  }
}

// numpy float mod (npy_divmod): sign follows the divisor
__device__ __forceinline__ double np_mod(double a, double m) {
  double r = fmod(a, m);
  if (r != 0.0) {
    if ((m < 0) != (r < 0)) r = __dadd_rn(r, m);
  } else {
    r = copysign(0.0, m);
  }
  return r;
}

// HSV hue scaled to [0, L] (hue_plane, src/color.py:341-362)
__device__ __forceinline__ double hue_of(double r, double g, double b, double peak) {
  const double mx = fmax(fmax(r, g), b), mn = fmin(fmin(r, g), b);
  const double d = __dsub_rn(mx, mn);
  double h;
  if (d == 0.0) {
    h = 0.0;
  } else if (mx == r) {
    h = np_mod(__ddiv_rn(__dsub_rn(g, b), d), 6.0);
  } else if (mx == g) {
    h = __dadd_rn(__ddiv_rn(__dsub_rn(b, r), d), 2.0);
  } else {
    h = __dadd_rn(__ddiv_rn(__dsub_rn(r, g), d), 4.0);
  }
  h = __dmul_rn(h, 60.0);
  return __dmul_rn(__ddiv_rn(h, 360.0), peak);
}

__device__ __forceinline__ void mat3(const double* m, double a, double b, double c, double& o0, double& o1,
                                     double& o2) {
  o0 = __dadd_rn(__dadd_rn(__dmul_rn(m[0], a), __dmul_rn(m[1], b)), __dmul_rn(m[2], c));
  o1 = __dadd_rn(__dadd_rn(__dmul_rn(m[3], a), __dmul_rn(m[4], b)), __dmul_rn(m[5], c));
  o2 = __dadd_rn(__dadd_rn(__dmul_rn(m[6], a), __dmul_rn(m[7], b)), __dmul_rn(m[8], c));
}

__device__ __forceinline__ double lab_f(double t) {
  constexpr double d = 6.0 / 29.0;
  return t > d * d * d ? cbrt(t) : __dadd_rn(__ddiv_rn(t, 3.0 * d * d), 4.0 / 29.0);
}

__device__ __forceinline__ void xyz_to_lab(double x, double y, double z, double& L, double& A, double& B) {
  const double fx = lab_f(__ddiv_rn(x, c_d65[0])), fy = lab_f(__ddiv_rn(y, c_d65[1])),
               fz = lab_f(__ddiv_rn(z, c_d65[2]));
  L = __dsub_rn(__dmul_rn(116.0, fy), 16.0);
  A = __dmul_rn(500.0, __dsub_rn(fx, fy));
  B = __dmul_rn(200.0, __dsub_rn(fy, fz));
}

// ---------------------------------------------------------------------------
// conversions: one thread per pixel, float64 planes out
// ---------------------------------------------------------------------------
__global__ void color_convert_kernel(const __grid_constant__ ColorIn in, int op, double* __restrict__ out,
                                     long long orp, long long ofp) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y;
  const int f = blockIdx.z;
  if (x >= in.w) return;
  double* o = out + (long long)f * ofp + (long long)y * orp + x;
  const long long pp = (long long)in.h * orp;  // plane pitch
  switch (op) {
    case SSK_CONV_RGB: {
      double r, g, b;
      rgb_at(in, f, y, x, r, g, b);
      o[0] = r;
      o[pp] = g;
      o[2 * pp] = b;
      break;
    }
    case SSK_CONV_YCBCR: {
      const double c0 = chan(in, 0, f, y, x), c1 = chan(in, 1, f, y, x), c2 = chan(in, 2, f, y, x);
      if (in.space == SSK_SPACE_YCBCR) {
        o[0] = c0;
        o[pp] = c1;
        o[2 * pp] = c2;
      } else {
        const double half = __ddiv_rn(in.peak, 2.0);
        const double yy = luma709(c0, c1, c2);
        o[0] = yy;
        o[pp] = __dadd_rn(__dmul_rn(CB_SCALE, __dsub_rn(c2, yy)), half);
        o[2 * pp] = __dadd_rn(__dmul_rn(CR_SCALE, __dsub_rn(c0, yy)), half);
      }
      break;
    }
    case SSK_CONV_LUMA: {
      if (in.space == SSK_SPACE_YCBCR) {
        o[0] = chan(in, 0, f, y, x);
      } else {
        o[0] = luma709(chan(in, 0, f, y, x), chan(in, 1, f, y, x), chan(in, 2, f, y, x));
      }
      break;
    }
    case SSK_CONV_HUE: {
      double r, g, b;
      rgb_at(in, f, y, x, r, g, b);
      o[0] = hue_of(r, g, b, in.peak);
      break;
    }
    case SSK_CONV_LAB_EMBED: {  // qssim's 'lab' embedding: CIELAB * L / 100
      double r, g, b, X, Y, Z, L, A, B;
      rgb_at(in, f, y, x, r, g, b);
      mat3(c_rgb2xyz, __ddiv_rn(r, in.peak), __ddiv_rn(g, in.peak), __ddiv_rn(b, in.peak), X, Y, Z);
      xyz_to_lab(X, Y, Z, L, A, B);
      const double sc = __ddiv_rn(in.peak, 100.0);
      o[0] = __dmul_rn(L, sc);
      o[pp] = __dmul_rn(A, sc);
      o[2 * pp] = __dmul_rn(B, sc);
      break;
    }
    default:
      break;
  }
}

// ---------------------------------------------------------------------------
// qssim: one thread per anchor; the twelve windowed means accumulate
// (1/k^2) * value in the (m, n) order of _sliding_weighted_sums
// (src/stats.py:155-164), so each mean is bit-identical to the reference's
// ---------------------------------------------------------------------------
struct QArgs {
  const double* e1;  // [n][3][h][rp]
  const double* e2;
  long long rp, pp, fp;
  int n, h, w, k, s, gh, gw;
  double wgt, c1, c2;
  double* partials;  // [n][blocks][1]
};

__global__ void __launch_bounds__(128) qssim_kernel(const __grid_constant__ QArgs a) {
  __shared__ double red[4];
  const int ac = blockIdx.x * 32 + (threadIdx.x & 31);
  const int ar = blockIdx.y * 4 + (threadIdx.x >> 5);
  const int f = blockIdx.z;
  double val = 0.0;
  if (ac < a.gw && ar < a.gh) {
    const double* p1 = a.e1 + (long long)f * a.fp + (long long)(ar * a.s) * a.rp + ac * a.s;
    const double* p2 = a.e2 + (long long)f * a.fp + (long long)(ar * a.s) * a.rp + ac * a.s;
    double m1[3] = {0, 0, 0}, m2[3] = {0, 0, 0}, ed = 0, ei = 0, ej = 0, ek = 0, q1 = 0, q2 = 0;
    const double c = a.wgt;
    for (int m = 0; m < a.k; ++m) {
      for (int nn = 0; nn < a.k; ++nn) {
        const long long o = (long long)m * a.rp + nn;
        const double r1 = p1[o], g1 = p1[o + a.pp], b1 = p1[o + 2 * a.pp];
        const double r2 = p2[o], g2 = p2[o + a.pp], b2 = p2[o + 2 * a.pp];
        m1[0] = __dadd_rn(m1[0], __dmul_rn(c, r1));
        m1[1] = __dadd_rn(m1[1], __dmul_rn(c, g1));
        m1[2] = __dadd_rn(m1[2], __dmul_rn(c, b1));
        m2[0] = __dadd_rn(m2[0], __dmul_rn(c, r2));
        m2[1] = __dadd_rn(m2[1], __dmul_rn(c, g2));
        m2[2] = __dadd_rn(m2[2], __dmul_rn(c, b2));
        const double dot = __dadd_rn(__dadd_rn(__dmul_rn(r1, r2), __dmul_rn(g1, g2)), __dmul_rn(b1, b2));
        const double ci = -__dsub_rn(__dmul_rn(g1, b2), __dmul_rn(b1, g2));
        const double cj = -__dsub_rn(__dmul_rn(b1, r2), __dmul_rn(r1, b2));
        const double ck = -__dsub_rn(__dmul_rn(r1, g2), __dmul_rn(g1, r2));
        const double s1 = __dadd_rn(__dadd_rn(__dmul_rn(r1, r1), __dmul_rn(g1, g1)), __dmul_rn(b1, b1));
        const double s2 = __dadd_rn(__dadd_rn(__dmul_rn(r2, r2), __dmul_rn(g2, g2)), __dmul_rn(b2, b2));
        ed = __dadd_rn(ed, __dmul_rn(c, dot));
        ei = __dadd_rn(ei, __dmul_rn(c, ci));
        ej = __dadd_rn(ej, __dmul_rn(c, cj));
        ek = __dadd_rn(ek, __dmul_rn(c, ck));
        q1 = __dadd_rn(q1, __dmul_rn(c, s1));
        q2 = __dadd_rn(q2, __dmul_rn(c, s2));
      }
    }
    const double mdot = __dadd_rn(__dadd_rn(__dmul_rn(m1[0], m2[0]), __dmul_rn(m1[1], m2[1])), __dmul_rn(m1[2], m2[2]));
    const double mi = -__dsub_rn(__dmul_rn(m1[1], m2[2]), __dmul_rn(m1[2], m2[1]));
    const double mj = -__dsub_rn(__dmul_rn(m1[2], m2[0]), __dmul_rn(m1[0], m2[2]));
    const double mk = -__dsub_rn(__dmul_rn(m1[0], m2[1]), __dmul_rn(m1[1], m2[0]));
    const double n1 = __dadd_rn(__dadd_rn(__dmul_rn(m1[0], m1[0]), __dmul_rn(m1[1], m1[1])), __dmul_rn(m1[2], m1[2]));
    const double n2 = __dadd_rn(__dadd_rn(__dmul_rn(m2[0], m2[0]), __dmul_rn(m2[1], m2[1])), __dmul_rn(m2[2], m2[2]));
    const double var1 = __dsub_rn(q1, n1), var2 = __dsub_rn(q2, n2);
    const double cw = __dsub_rn(ed, mdot), cvi = __dsub_rn(ei, mi), cvj = __dsub_rn(ej, mj), cvk = __dsub_rn(ek, mk);
    auto sq = [](double v) { return __dmul_rn(v, v); };
    const double a1 = __dadd_rn(__dmul_rn(2.0, mdot), a.c1);
    const double num1 = __dsqrt_rn(__dadd_rn(__dadd_rn(__dadd_rn(sq(a1), sq(__dmul_rn(2.0, mi))), sq(__dmul_rn(2.0, mj))),
                                             sq(__dmul_rn(2.0, mk))));
    const double den1 = __dadd_rn(__dadd_rn(n1, n2), a.c1);
    const double a2 = __dadd_rn(__dmul_rn(2.0, cw), a.c2);
    const double num2 = __dsqrt_rn(__dadd_rn(__dadd_rn(__dadd_rn(sq(a2), sq(__dmul_rn(2.0, cvi))), sq(__dmul_rn(2.0, cvj))),
                                             sq(__dmul_rn(2.0, cvk))));
    const double den2 = __dadd_rn(__dadd_rn(var1, var2), a.c2);
    val = __dmul_rn(__ddiv_rn(num1, den1), __ddiv_rn(num2, den2));
  }
  val = warp_sum(val);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = val;
  __syncthreads();
  if (threadIdx.x == 0) {
    const long long part = ((long long)f * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
    a.partials[part * 3] = ((red[0] + red[1]) + red[2]) + red[3];  // [n][parts][3] layout, slot 0
  }
}

// ---------------------------------------------------------------------------
// delta-E: opponent planes -> separable smoothing (reflect) -> Lab at the
// window centres of an SSIM grid
// ---------------------------------------------------------------------------
// q planes per side: [n][3][h][w] float64 (q0 unsmoothed, q1 / q2 smoothed in place via tmp)
// to_q = 0 (no smoothing): the planes hold XYZ itself, like _rgb_frame_to_lab without the opponent step
__global__ void opponent_kernel(const __grid_constant__ ColorIn in, double* __restrict__ q, long long pp,
                                long long fp, int to_q) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y, f = blockIdx.z;
  if (x >= in.w) return;
  double r, g, b, X, Y, Z, q0, q1, q2;
  rgb_at(in, f, y, x, r, g, b);
  mat3(c_rgb2xyz, __ddiv_rn(r, in.peak), __ddiv_rn(g, in.peak), __ddiv_rn(b, in.peak), X, Y, Z);
  if (to_q) {
    mat3(c_xyz2q, X, Y, Z, q0, q1, q2);
  } else {
    q0 = X;
    q1 = Y;
    q2 = Z;
  }
  double* o = q + (long long)f * fp + (long long)y * in.w + x;
  o[0] = q0;
  o[pp] = q1;
  o[2 * pp] = q2;
}

struct SmoothTaps {
  double g[SMOOTH_K];
};

__device__ __forceinline__ int reflect(int i, int n) {
  if (n == 1) return 0;
  const int period = 2 * (n - 1);
  i %= period;
  if (i < 0) i += period;
  return i < n ? i : period - i;
}

// one smoothing pass (vertical: dir 0, horizontal: dir 1) over planes 1 and 2:
// out = sum_m g[m] * v[reflect(i + m - pad)] accumulated from 0 in m order, like
// Python's sum() over the shifted slices
__global__ void smooth_kernel(const double* __restrict__ src, double* __restrict__ dst, int h, int w, long long pp,
                              long long fp, int dir, const __grid_constant__ SmoothTaps taps) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y;
  const int f = blockIdx.z >> 1, plane = 1 + (blockIdx.z & 1);
  if (x >= w) return;
  const double* s = src + (long long)f * fp + plane * pp;
  double acc = 0.0;
  constexpr int pad = (SMOOTH_K - 1) / 2;
#pragma unroll
  for (int m = 0; m < SMOOTH_K; ++m) {
    const double v = dir == 0 ? s[(long long)reflect(y + m - pad, h) * w + x] : s[(long long)y * w + reflect(x + m - pad, w)];
    acc = __dadd_rn(acc, __dmul_rn(taps.g[m], v));
  }
  dst[(long long)f * fp + plane * pp + (long long)y * w + x] = acc;
}

struct DeArgs {
  const double* q1;  // smoothed opponent planes of ref / dist, [n][3][h][w]
  const double* q2;
  long long pp, fp;
  int n, h, w, gh, gw, k, s, smooth, mode;
  double* out;       // [n][gh][gw]
  long long orp, ofp;
};

__device__ __forceinline__ void lab_from_q(const double* q, long long pp, long long idx, int from_q, double& L,
                                           double& A, double& B) {
  double X = q[idx], Y = q[idx + pp], Z = q[idx + 2 * pp];
  if (from_q) mat3(c_q2xyz, q[idx], q[idx + pp], q[idx + 2 * pp], X, Y, Z);
  xyz_to_lab(X, Y, Z, L, A, B);
}

__global__ void delta_e_kernel(const __grid_constant__ DeArgs a) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  const int r = blockIdx.y, f = blockIdx.z;
  if (c >= a.gw) return;
  const int ctr = (a.k - 1) / 2;
  const long long idx = (long long)f * a.fp + (long long)(r * a.s + ctr) * a.w + (c * a.s + ctr);
  double L1, A1, B1, L2, A2, B2;
  lab_from_q(a.q1, a.pp, idx, a.smooth, L1, A1, B1);
  lab_from_q(a.q2, a.pp, idx, a.smooth, L2, A2, B2);
  const double dl = __dsub_rn(L1, L2), da = __dsub_rn(A1, A2), db = __dsub_rn(B1, B2);
  const double de = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(dl, dl), __dmul_rn(da, da)), __dmul_rn(db, db)));
  // mode 1: the cmssim weight before clamping, 1 - dE / 45
  a.out[(long long)f * a.ofp + (long long)r * a.orp + c] = a.mode ? __dsub_rn(1.0, __ddiv_rn(de, 45.0)) : de;
}

int make_color_in(const ssk_color* c, ColorIn& in) {
  if (!c || !c->ch[0] || !c->ch[1] || !c->ch[2]) return SSK_E_ARG;
  if (c->dtype != SSK_U8 && c->dtype != SSK_U16 && c->dtype != SSK_F32 && c->dtype != SSK_F64) return SSK_E_ARG;
  if (c->space != SSK_SPACE_RGB && c->space != SSK_SPACE_YCBCR) return SSK_E_ARG;
  if (c->subsampling != 0 && c->subsampling != 1) return SSK_E_ARG;
  if (c->subsampling == 1 && c->space != SSK_SPACE_YCBCR) return SSK_E_ARG;
  if (c->n < 1 || c->n > 65535 || c->h < 1 || c->w < 1 || c->h > 65535) return SSK_E_ARG;
  if (c->bit_depth < 1 || c->bit_depth > 16) return SSK_E_ARG;
  for (int i = 0; i < 3; ++i) {
    const int hh = (i && c->subsampling) ? (c->h + 1) / 2 : c->h;
    const int ww = (i && c->subsampling) ? (c->w + 1) / 2 : c->w;
    if (c->row_pitch[i] < ww || c->frame_pitch[i] < c->row_pitch[i] * (int64_t)hh) return SSK_E_ARG;
    in.ch[i] = static_cast<const unsigned char*>(c->ch[i]);
    in.rp[i] = c->row_pitch[i];
    in.fp[i] = c->frame_pitch[i];
  }
  in.dtype = c->dtype;
  in.space = c->space;
  in.sub420 = c->subsampling;
  in.n = c->n;
  in.h = c->h;
  in.w = c->w;
  in.peak = std::ldexp(1.0, c->bit_depth) - 1.0;
  return SSK_OK;
}

inline size_t al(size_t x) { return (x + 255) / 256 * 256; }

}  // namespace
}  // namespace ssk

using namespace ssk;

extern "C" {

int ssk_color_convert(const ssk_color* src, int op, double* d_out, int64_t out_row_pitch, int64_t out_frame_pitch,
                      void* stream) {
  ColorIn in;
  int rc = make_color_in(src, in);
  if (rc) return rc;
  if (op < SSK_CONV_RGB || op > SSK_CONV_LAB_EMBED || !d_out) return SSK_E_ARG;
  const int planes = (op == SSK_CONV_LUMA || op == SSK_CONV_HUE) ? 1 : 3;
  if (out_row_pitch < in.w || out_frame_pitch < out_row_pitch * (int64_t)in.h * planes) return SSK_E_ARG;
  const dim3 grid((in.w + 127) / 128, in.h, in.n);
  color_convert_kernel<<<grid, 128, 0, static_cast<cudaStream_t>(stream)>>>(in, op, d_out, out_row_pitch,
                                                                            out_frame_pitch);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? SSK_OK : SSK_E_CUDA;
}

size_t ssk_qssim_workspace_bytes(int n, int h, int w, int k, int stride) {
  if (n < 1 || k < 1 || stride < 1 || k > h || k > w) return 0;
  const int gh = (h - k) / stride + 1, gw = (w - k) / stride + 1;
  return al((size_t)n * ((gw + 31) / 32) * ((gh + 3) / 4) * 3 * sizeof(double));
}

int ssk_qssim(const double* d_emb_ref, const double* d_emb_dist, int n, int h, int w, int64_t row_pitch,
              int64_t frame_pitch, int k, int stride, double c1, double c2, double* d_means, void* d_workspace,
              size_t workspace_bytes, void* stream) {
  if (!d_emb_ref || !d_emb_dist || !d_means || n < 1 || n > 65535 || h < 1 || w < 1) return SSK_E_ARG;
  if (k < 1 || stride < 1) return SSK_E_ARG;
  if (k > h || k > w) return SSK_E_WINDOW;
  if (row_pitch < w || frame_pitch < 3 * row_pitch * (int64_t)h) return SSK_E_ARG;
  const size_t need = ssk_qssim_workspace_bytes(n, h, w, k, stride);
  if (!d_workspace || workspace_bytes < need) return SSK_E_WORKSPACE;
  QArgs a{};
  a.e1 = d_emb_ref;
  a.e2 = d_emb_dist;
  a.rp = row_pitch;
  a.pp = row_pitch * h;
  a.fp = frame_pitch;
  a.n = n;
  a.h = h;
  a.w = w;
  a.k = k;
  a.s = stride;
  a.gh = (h - k) / stride + 1;
  a.gw = (w - k) / stride + 1;
  a.wgt = 1.0 / ((double)k * (double)k);  // np.full((k, k), 1.0 / (k * k))
  a.c1 = c1;
  a.c2 = c2;
  a.partials = static_cast<double*>(d_workspace);
  const dim3 grid((a.gw + 31) / 32, (a.gh + 3) / 4, n);
  if (grid.y > 65535) return SSK_E_ARG;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  qssim_kernel<<<grid, 128, 0, st>>>(a);
  note_launch();
  if (cudaGetLastError() != cudaSuccess) return SSK_E_CUDA;
  return launch_reduce_partials(a.partials, (int)(grid.x * grid.y), n, 1, (double)a.gh * (double)a.gw, d_means, 1,
                                0, 0, st);
}

size_t ssk_delta_e_workspace_bytes(int n, int h, int w) {
  if (n < 1 || h < 1 || w < 1) return 0;
  return 3 * al((size_t)n * 3 * h * w * sizeof(double));
}

int ssk_delta_e(const ssk_color* ref, const ssk_color* dist, int smooth, int k, int stride, int mode, double* d_out,
                int64_t out_row_pitch, int64_t out_frame_pitch, void* d_workspace, size_t workspace_bytes,
                void* stream) {
  ColorIn a, b;
  int rc = make_color_in(ref, a);
  if (rc) return rc;
  rc = make_color_in(dist, b);
  if (rc) return rc;
  if (a.n != b.n || a.h != b.h || a.w != b.w || a.peak != b.peak) return SSK_E_ARG;
  if (k < 1 || stride < 1 || (mode != 0 && mode != 1) || !d_out) return SSK_E_ARG;
  if (k > a.h || k > a.w) return SSK_E_WINDOW;
  const int gh = (a.h - k) / stride + 1, gw = (a.w - k) / stride + 1;
  if (out_row_pitch < gw || out_frame_pitch < out_row_pitch * (int64_t)gh) return SSK_E_ARG;
  const size_t one = al((size_t)a.n * 3 * a.h * a.w * sizeof(double));
  if (!d_workspace || workspace_bytes < 3 * one) return SSK_E_WORKSPACE;
  char* ws = static_cast<char*>(d_workspace);
  double* q1 = reinterpret_cast<double*>(ws);
  double* q2 = reinterpret_cast<double*>(ws + one);
  double* tmp = reinterpret_cast<double*>(ws + 2 * one);
  const long long pp = (long long)a.h * a.w, fp = 3 * pp;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const dim3 grid((a.w + 127) / 128, a.h, a.n);
  opponent_kernel<<<grid, 128, 0, st>>>(a, q1, pp, fp, smooth ? 1 : 0);
  opponent_kernel<<<grid, 128, 0, st>>>(b, q2, pp, fp, smooth ? 1 : 0);
  note_launch(2);
  if (smooth) {
    // _smooth's taps: the centre row of gaussian_kernel(2, 13) (outer(g, g) / its sum),
    // renormalised to sum 1
    SmoothTaps t{};
    double g[SMOOTH_K], outer = 0.0, row[SMOOTH_K], rs = 0.0;
    for (int i = 0; i < SMOOTH_K; ++i) {
      const double c = (double)i - (SMOOTH_K - 1) / 2.0;
      g[i] = std::exp(-(c * c) / (2.0 * 2.0 * 2.0));
    }
    for (int i = 0; i < SMOOTH_K; ++i)
      for (int j = 0; j < SMOOTH_K; ++j) outer += g[i] * g[j];
    for (int i = 0; i < SMOOTH_K; ++i) {
      row[i] = (g[(SMOOTH_K - 1) / 2] * g[i]) / outer;
      rs += row[i];
    }
    for (int i = 0; i < SMOOTH_K; ++i) t.g[i] = row[i] / rs;
    const dim3 sg2((a.w + 127) / 128, a.h, 2 * a.n);
    for (double* q : {q1, q2}) {
      smooth_kernel<<<sg2, 128, 0, st>>>(q, tmp, a.h, a.w, pp, fp, 0, t);
      smooth_kernel<<<sg2, 128, 0, st>>>(tmp, q, a.h, a.w, pp, fp, 1, t);
      note_launch(2);
    }
  }
  DeArgs d{};
  d.q1 = q1;
  d.q2 = q2;
  d.pp = pp;
  d.fp = fp;
  d.n = a.n;
  d.h = a.h;
  d.w = a.w;
  d.gh = gh;
  d.gw = gw;
  d.k = k;
  d.s = stride;
  d.smooth = smooth ? 1 : 0;
  d.mode = mode;
  d.out = d_out;
  d.orp = out_row_pitch;
  d.ofp = out_frame_pitch;
  delta_e_kernel<<<dim3((gw + 127) / 128, gh, a.n), 128, 0, st>>>(d);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? SSK_OK : SSK_E_CUDA;
}

}  // extern "C"
