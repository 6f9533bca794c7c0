// C ABI entry points (include/ssimk.h): argument validation, launch planning,
// workspace carving and the MS-SSIM level loop.  Host-side C++; no allocation
// inside the calls (all scratch comes from the caller's workspace).
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <utility>

#include "common.cuh"
#include "kernels.h"

namespace ssk {
namespace gk {
int gauss_ws_level();
}
}  // namespace ssk
namespace ssk {
namespace gk {
int gauss_ws_level() {
  static const int v = [] {
    const char* e = std::getenv("SSK_GAUSS_WS");  // warp-specialised K1 (default on; 0 = classic)
    return e ? std::atoi(e) : 1;
  }();
  return v;
}
int gauss_persist_level() {
  static const int v = [] {
    const char* e = std::getenv("SSK_GAUSS_PERSIST");  // persistent wide u8 K1 (default on; 0 = one tile per CTA)
    return e ? std::atoi(e) : 1;
  }();
  return v;
}
int gauss_narrow_ws() {
  static const int v = [] {
    const char* e = std::getenv("SSK_NARROW_WS");  // 1 = warp-specialised kernel for 128-column strips
    return e ? std::atoi(e) : 0;
  }();
  return v;
}
int gauss_l0_classic() {
  static const int v = [] {
    const char* e = std::getenv("SSK_L0_CLASSIC");  // wide u8 frames on the classic kernel, 2 CTAs/SM (0 = persistent warp-specialised)
    return e ? std::atoi(e) : 1;
  }();
  return v;
}
int sm_count() {
  static int cached[64] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
  if (!cached[dev]) {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    cached[dev] = n > 0 ? n : 148;
  }
  return cached[dev];
}
}  // namespace gk

static std::atomic<unsigned long long> g_launches{0};
// SSK_FUSED_L1=0 restores the separate pyramid pass for level 1 (A/B switch)
static int fused_l1_enabled() {
  static const int v = [] {
    const char* e = std::getenv("SSK_FUSED_L1");
    return e ? std::atoi(e) : 1;
  }();
  return v;
}
void note_launch(int count) { g_launches.fetch_add((unsigned long long)count); }
int probe_fp32(double seconds, double* tflops, cudaStream_t st);

namespace {

constexpr size_t kAlign = 256;
inline size_t align_up(size_t x, size_t a = kAlign) { return (x + a - 1) / a * a; }

struct Plan {
  bool gauss = false;
  bool generic = false;  // Gaussian wider than 31 taps: the fp64 generic-K kernel (K1g)
  bool strided = false;  // strided Gaussian scores: the anchor-only kernel (K1s)
  bool box_block = false;
  bool box_int = false;
  bool wide = false;
  dim3 grid, block;
  int gh = 0, gw = 0;
  size_t nparts_per_frame = 0;
  GaussArgs ga{};
  GaussGenericArgs gg{};
  BoxArgs ba{};
};

// normalised 1-D Gaussian g/sum(g) in fp64 (gaussian_kernel, src/stats.py:41-44)
void build_taps(double sigma, int k, double* out) {
  double sum = 0.0;
  for (int i = 0; i < k; ++i) {
    const double c = (double)i - (k - 1) / 2.0;
    out[i] = std::exp(-(c * c) / (2.0 * sigma * sigma));
    sum += out[i];
  }
  for (int i = 0; i < k; ++i) out[i] /= sum;
}

bool taps_given(const ssk_window* win) {
  for (int i = 0; i < 32; ++i)
    if (win->taps[i] != 0.0f) return true;
  return false;
}

int check_planes(const ssk_planes* p) {
  if (!p || !p->ref || !p->dist) return SSK_E_ARG;
  const int es = esize_of(p->dtype);
  if (es == 0) return SSK_E_ARG;
  if (p->n < 1 || p->h < 1 || p->w < 1 || p->n > 65535) return SSK_E_ARG;
  if (p->row_pitch < p->w || p->frame_pitch < p->row_pitch * (int64_t)p->h) return SSK_E_ARG;
  if (p->bit_depth < 8 || p->bit_depth > 16 || p->scale_log2 < 0 || p->scale_log2 > 40)
    return SSK_E_ARG;
  if ((reinterpret_cast<uintptr_t>(p->ref) & 15) || (reinterpret_cast<uintptr_t>(p->dist) & 15) ||
      ((p->row_pitch * es) & 15) || ((p->frame_pitch * es) & 15))
    return SSK_E_ALIGN;
  return SSK_OK;
}

int check_window(const ssk_planes* p, const ssk_window* win) {
  if (!win || win->k < 1 || win->stride < 1) return SSK_E_ARG;
  if (win->shape == SSK_GAUSS) {
    if (win->k < 3 || (win->k % 2) == 0 || win->k > SSK_GAUSS_MAX_K) return SSK_E_SHAPE;
    if (p->dtype == SSK_F64) return SSK_E_ARG;
    const bool sigma_ok = std::isfinite(win->sigma) && win->sigma > 0.0;
    if (win->k > 31 || !taps_given(win)) {
      if (!sigma_ok) return SSK_E_ARG;  // nothing to build the window from
    } else {
      // caller's taps: finite, non-negative (a tiny sigma underflows the outer taps to 0,
      // as in the reference), exactly symmetric, normalised, zero past k
      double sum = 0.0;
      for (int i = 0; i < 32; ++i) {
        const float t = win->taps[i];
        if (i >= win->k) {
          if (t != 0.0f) return SSK_E_ARG;
          continue;
        }
        if (!std::isfinite(t) || !(t >= 0.0f) || t != win->taps[win->k - 1 - i]) return SSK_E_ARG;
        sum += t;
      }
      if (std::fabs(sum - 1.0) > 1e-5) return SSK_E_ARG;
    }
  } else if (win->shape != SSK_RECT) {
    return SSK_E_ARG;
  }
  if (win->k > p->h || win->k > p->w) return SSK_E_WINDOW;
  return SSK_OK;
}

int plan_ssim(const ssk_planes* p, const ssk_window* win, int want, Plan& pl) {
  int rc = check_planes(p);
  if (rc) return rc;
  rc = check_window(p, win);
  if (rc) return rc;
  const int k = win->k, s = win->stride;
  const int es = esize_of(p->dtype);
  pl.gh = grid_extent(p->h, k, s);
  pl.gw = grid_extent(p->w, k, s);
  const double L = std::ldexp(1.0, p->bit_depth) - 1.0;
  const double stored_max = L * std::ldexp(1.0, p->scale_log2);

  if (win->shape == SSK_GAUSS && (k > 31 || (want & SSK_MAP_F64))) {
    pl.gauss = pl.generic = true;
    pl.ga.vcols = 0;  // never joins the fused / multi-level launches
    GaussGenericArgs& g = pl.gg;
    g.ref = static_cast<const unsigned char*>(p->ref);
    g.dist = static_cast<const unsigned char*>(p->dist);
    g.row_pitch_b = p->row_pitch * es;
    g.frame_pitch_b = p->frame_pitch * es;
    g.dtype = p->dtype;
    g.esize = es;
    g.n = p->n;
    g.h = p->h;
    g.w = p->w;
    g.k = k;
    g.stride = s;
    g.ho = p->h - k + 1;
    g.wo = p->w - k + 1;
    g.gh = pl.gh;
    g.gw = pl.gw;
    g.seg_rows = 64;
    g.scale = (p->dtype == SSK_F32) ? 1.0 : std::ldexp(1.0, -p->scale_log2);
    g.c1 = win->c1;
    g.c2 = win->c2;
    g.want = want;
    g.map_plane = (long long)pl.gh * pl.gw;
    g.map_frame = g.map_plane * ((want & SSK_MAP_STATS) ? 5 : 3);
    g.map_f64 = (want & SSK_MAP_F64) ? 1 : 0;
    if (win->sigma > 0.0) {
      build_taps(win->sigma, k, g.taps);
    } else {  // caller's fp32 taps (k <= 31), widened
      for (int i = 0; i < k; ++i) g.taps[i] = (double)win->taps[i];
    }
    if (gauss_generic_grid(g.ho, g.wo, p->n, g.seg_rows, &pl.grid)) return SSK_E_ARG;
    pl.nparts_per_frame = (size_t)pl.grid.x * pl.grid.y;
    return SSK_OK;
  }
  if (win->shape == SSK_GAUSS) {
    pl.gauss = true;
    GaussArgs& a = pl.ga;
    a.ref = static_cast<const unsigned char*>(p->ref);
    a.dist = static_cast<const unsigned char*>(p->dist);
    a.row_pitch_b = p->row_pitch * es;
    a.frame_pitch_b = p->frame_pitch * es;
    a.dtype = p->dtype;
    a.esize = es;
    a.n = p->n;
    a.h = p->h;
    a.w = p->w;
    a.ho = p->h - k + 1;
    a.wo = p->w - k + 1;
    a.gh = pl.gh;
    a.gw = pl.gw;
    a.stride = s;
    // wide strips (256 V columns, 1 CTA/SM) for 8-bit frames under the warp-specialised
    // kernel: V-halo overhead 250/240 instead of 122/112 and fewer idle H threads
    // (16-bit frames too since the classic kernel took over the wide strips, r2: 10-bit 1080p
    // scores 101.7 k pairs/s on 256-column strips vs 91.8 k on 128-column ones; SSK_WIDE_U16=0
    // restores the narrow strips)
    static const int wide_u16 = [] {
      const char* e = std::getenv("SSK_WIDE_U16");
      return e ? std::atoi(e) : 1;
    }();
    // coarse pyramid levels (u16 scaled sums): wide strips on the classic multi-level kernel
    static const int levels_wide = [] {
      const char* e = std::getenv("SSK_LEVELS_WIDE");  // default on; 0 = 128-column strips
      return e ? std::atoi(e) : 1;
    }();
    const bool coarse_wide = p->dtype == SSK_U16 && p->scale_log2 > 0 && levels_wide;
    const bool wide_ok = p->dtype == SSK_U8 || (p->dtype == SSK_U16 && (wide_u16 || coarse_wide));
    const bool maps = (want & (SSK_MAP_TERMS | SSK_MAP_STATS)) != 0;  // maps: classic kernel only
    static const int wide_min_wo = [] {  // narrowest output width that gets 256-column strips
      const char* e = std::getenv("SSK_WIDE_MIN_WO");
      return e ? std::atoi(e) : 480;
    }();
    // below that width: wide strips where they cover the row with no more V columns than
    // narrow ones (one 240-column strip vs two or three of 112, or two vs four / five):
    // 480 x 480 frames 0.113 -> 0.097 ms per 64 pairs, 352 x 288 0.177 -> 0.163 ms per 256
    const int tw_w = gauss_tw(k, 256), tw_n = gauss_tw(k, 128);
    const bool cols_ok = tw_w > 0 && tw_n > 0 &&
                         (long long)((a.wo + tw_w - 1) / tw_w) * 256 <= (long long)((a.wo + tw_n - 1) / tw_n) * 128;
    a.vcols = (gk::gauss_ws_level() >= 1 && wide_ok && !maps && k <= 17 &&
               (a.wo >= wide_min_wo || cols_ok || coarse_wide)) ? 256 : 128;
    const int tw = gauss_tw(k, a.vcols);
    const int nstrips = (a.wo + tw - 1) / tw;
    // Segments depend on the frame geometry only (never on the batch size), so a
    // frame's fp32 partial sums -- and hence its score -- are bit-identical
    // however frames are batched or sharded.
    static const int coarse_seg = [] {  // target rows per segment of the coarse levels
      const char* e = std::getenv("SSK_LEVEL_SEG");
      return e ? std::max(16, std::atoi(e)) : 128;
    }();
    static const int base_seg = [] {  // target rows per segment of full-resolution frames
      const char* e = std::getenv("SSK_BASE_SEG");
      return e ? std::max(16, std::atoi(e)) : 128;
    }();
    const int seg_target = (p->scale_log2 > 0) ? coarse_seg : base_seg;
    int nseg = (a.ho + seg_target - 1) / seg_target;
    a.seg_rows = (a.ho + nseg - 1) / nseg;
    if (a.vcols == 256) a.seg_rows += a.seg_rows & 1;  // even: segments own whole 2x2 pyramid blocks
    nseg = (a.ho + a.seg_rows - 1) / a.seg_rows;
    const float shift = (float)std::ldexp(1.0, p->bit_depth - 1);
    const double scale = std::ldexp(1.0, -p->scale_log2);
    a.conv_scale = (p->dtype == SSK_F32) ? 1.0f : (float)scale;
    if (p->dtype == SSK_U8 || p->dtype == SSK_U16)
      a.conv_bias = (float)(-(8388608.0 * scale + shift));
    else
      a.conv_bias = -shift;
    a.shift = shift;
    a.c1 = (float)win->c1;
    a.c2 = (float)win->c2;
    a.one = 1.0f;
    a.want = want;
    // x' = m * 2^-scale with |m| <= 2^(bd+scale) (per-tile shift anywhere in [0, L]): x'^2 is
    // exact in fp32 when m^2 fits 24 bits
    a.exact_sq = (p->dtype != SSK_F32 && p->bit_depth + p->scale_log2 <= 12) ? 1 : 0;
    if (taps_given(win)) {
      std::memcpy(a.taps, win->taps, sizeof(a.taps));
    } else {  // sigma only: the fp64 taps rounded to fp32
      double t[32];
      build_taps(win->sigma, k, t);
      for (int i = 0; i < 32; ++i) a.taps[i] = i < k ? (float)t[i] : 0.0f;
    }
    pl.grid = dim3(nstrips, nseg, (p->n + 1) / 2);  // two frames per CTA (packed fp32 pairs)
    pl.nparts_per_frame = (size_t)nstrips * nseg;
    a.map_plane = (long long)pl.gh * pl.gw;
    a.map_frame = a.map_plane * ((want & SSK_MAP_STATS) ? 5 : 3);
    // strided score launches on 8/16-bit samples: the anchor-only kernel (K1s); map
    // launches stay on K1 (strided maps == dense maps at [::s, ::s], bit-exact)
    static const int stride_fast = [] {
      const char* e = std::getenv("SSK_STRIDE_FAST");  // default on; 0 = K1 with anchor masking
      return e ? std::atoi(e) : 1;
    }();
    if (!maps && stride_fast && gauss_stride_supported(p->dtype, k, s)) {
      pl.strided = true;
      a.vcols = 0;  // never joins the fused / multi-level launches
      const int twa = gauss_stride_twa(k, s, es);
      const int sx = (pl.gw + twa - 1) / twa;
      int sseg = (pl.gh + 23) / 24;  // ~24 anchor rows per segment (geometry only)
      a.seg_rows = (pl.gh + sseg - 1) / sseg;
      sseg = (pl.gh + a.seg_rows - 1) / a.seg_rows;
      if (sseg > 65535) return SSK_E_ARG;
      pl.grid = dim3(sx, sseg, (p->n + 1) / 2);
      pl.nparts_per_frame = (size_t)sx * sseg;
    }
    return SSK_OK;
  }

  BoxArgs& a = pl.ba;
  a.ref = static_cast<const unsigned char*>(p->ref);
  a.dist = static_cast<const unsigned char*>(p->dist);
  a.row_pitch_b = p->row_pitch * es;
  a.frame_pitch_b = p->frame_pitch * es;
  a.dtype = p->dtype;
  a.esize = es;
  a.n = p->n;
  a.h = p->h;
  a.w = p->w;
  a.k = k;
  a.s = s;
  a.gh = pl.gh;
  a.gw = pl.gw;
  a.sscale1 = std::ldexp(1.0, -p->scale_log2);
  a.sscale2 = std::ldexp(1.0, -2 * p->scale_log2);
  a.area = (double)k * (double)k;
  a.area_i = k * k;
  a.c1i = (float)(win->c1 * a.area * a.area * std::ldexp(1.0, 2 * p->scale_log2));
  a.c2i = (float)(win->c2 * a.area * a.area * std::ldexp(1.0, 2 * p->scale_log2));
  a.c1d = win->c1 * a.area * a.area * std::ldexp(1.0, 2 * p->scale_log2);
  a.c2d = win->c2 * a.area * a.area * std::ldexp(1.0, 2 * p->scale_log2);
  a.fast_ok = (a.area * a.area * stored_max * stored_max < 4.0e15) ? 1 : 0;
  int ex = 0;
  const double fr = std::frexp(a.area, &ex);
  a.area_pow2 = (fr == 0.5) ? 1 : 0;
  a.inv_area = 1.0 / a.area;
  a.c1 = win->c1;
  a.c2 = win->c2;
  a.want = want;
  a.map_plane = (long long)pl.gh * pl.gw;
  a.map_frame = a.map_plane * ((want & SSK_MAP_STATS) ? 5 : 3);
  a.wsums = nullptr;
  const bool integer = p->dtype == SSK_U8 || p->dtype == SSK_U16 || p->dtype == SSK_U32;
  // (q^2 sums are produced by the running-sum kernel only)
  if (integer && !(want & SSK_WANT_Q2) &&
      box_block_supported(p->dtype, k, s, (double)k * k * stored_max * stored_max >= 4294967296.0, stored_max)) {
    // stride divides the window: block-sum kernel (warps of 248 new columns, ~16 anchor rows per
    // segment: enough independent warps to keep HBM busy even for a handful of frames)
    pl.box_block = true;
    int seg_anchors = 16;
    long long nseg = (pl.gh + seg_anchors - 1) / seg_anchors;
    seg_anchors = (int)((pl.gh + nseg - 1) / nseg);
    a.seg_anchors = seg_anchors;
    nseg = (pl.gh + seg_anchors - 1) / seg_anchors;
    const int nwarps = (p->w + 247) / 248;
    pl.grid = dim3((nwarps + 3) / 4, (unsigned)nseg, p->n);
    if (nseg > 65535) return SSK_E_ARG;
    pl.nparts_per_frame = (size_t)pl.grid.x * pl.grid.y;
    return SSK_OK;
  }
  if (integer && k <= BX_THREADS) {
    pl.box_int = true;
    pl.wide = (double)k * k * stored_max * stored_max >= 4294967296.0;
    const int max_delta = 16 / es - 1;  // strips stage from a 16-byte aligned column
    a.na = (BX_THREADS - max_delta - k) / s + 1;
    const int nstrips = a.na > 0 ? (pl.gw + a.na - 1) / a.na : 0;
    int vr = 32 / s;
    vr = vr < 1 ? 1 : (vr > 8 ? 8 : vr);
    a.ch = vr * s;
    a.in_pitch = BX_THREADS * es + 16;
    a.nslot = (k + s - 1) / s + 1;
    // geometry-only segmentation (~256 input rows; shorter segments, down to ~48 rows,
    // when a frame would otherwise give fewer than 32 CTAs), independent of the batch size
    int seg_rows = 256;
    while (seg_rows > 48 && (long long)nstrips * ((pl.gh + (seg_rows + s - 1) / s - 1) / ((seg_rows + s - 1) / s)) < 32)
      seg_rows /= 2;
    int seg_anchors = (seg_rows + s - 1) / s;
    if (seg_anchors < 1) seg_anchors = 1;
    long long nseg = (pl.gh + seg_anchors - 1) / seg_anchors;
    seg_anchors = (int)((pl.gh + nseg - 1) / nseg);
    a.seg_anchors = seg_anchors;
    nseg = (pl.gh + seg_anchors - 1) / seg_anchors;
    if (nseg > 65535) return SSK_E_ARG;
    // short segments: stage at most ~half a segment per chunk (less shared memory per
    // CTA -> more resident CTAs to hide the staging latency)
    const int vr_seg = (seg_anchors + 1) / 2;
    if (vr > vr_seg) a.ch = (vr_seg < 1 ? 1 : vr_seg) * s;
    pl.grid = dim3(nstrips, (unsigned)nseg, p->n);
    pl.nparts_per_frame = (size_t)nstrips * nseg;
    if (a.na < 1 || box_smem_bytes(a, pl.wide) > 227 * 1024) {
      pl.box_int = false;  // extreme strides: fall through to the direct kernel
    } else {
      return SSK_OK;
    }
  }
  pl.block = dim3(32, 4);
  pl.grid = dim3((pl.gw + 31) / 32, (pl.gh + 3) / 4, p->n);
  if (pl.grid.y > 65535) return SSK_E_ARG;
  pl.nparts_per_frame = (size_t)pl.grid.x * pl.grid.y;
  return SSK_OK;
}

size_t partial_bytes(const Plan& pl, int n) { return align_up(pl.nparts_per_frame * n * 3 * sizeof(double)); }

int run_plan(Plan& pl, double* partials, void* maps, long long* wsums, cudaStream_t st) {
  if (pl.generic) {
    pl.gg.partials = partials;
    pl.gg.maps = maps;
    return launch_gauss_generic(pl.gg, pl.grid, st);
  }
  if (pl.strided) {
    pl.ga.partials = partials;
    pl.ga.maps = nullptr;
    return launch_gauss_stride(pl.ga, pl.grid, pl.ga.h - pl.ga.ho + 1, st);
  }
  if (pl.gauss) {
    pl.ga.partials = partials;
    pl.ga.maps = maps;
    return launch_gauss(pl.ga, pl.grid, pl.ga.h - pl.ga.ho + 1, st);
  }
  pl.ba.partials = partials;
  pl.ba.maps = static_cast<double*>(maps);
  pl.ba.wsums = wsums;
  if (pl.box_block) return launch_box_block(pl.ba, pl.grid, st);
  if (pl.box_int) return launch_box_int(pl.ba, pl.grid, pl.wide, st);
  return launch_box_float(pl.ba, pl.grid, pl.block, st);
}

// ---- MS-SSIM pyramid layout ----
struct Level {
  ssk_planes planes;
  size_t offset_r = 0, offset_d = 0;  // workspace offsets (level >= 1)
};

// Sample type of the scaled integer pyramid: one type for every level >= 1 (the one
// the deepest level needs), so the whole pyramid is produced by one kernel.
int level_dtype(const ssk_planes* p, int deepest) {
  if (p->dtype == SSK_F32) return SSK_F32;
  if (p->dtype == SSK_F64) return SSK_F64;
  const double mx = (std::ldexp(1.0, p->bit_depth) - 1.0) * std::ldexp(1.0, p->scale_log2 + 2 * deepest);
  return mx <= 65535.0 ? SSK_U16 : SSK_U32;
}

int plan_pyramid(const ssk_planes* p, const ssk_window* win, int levels, Level* lv, size_t* pyr_bytes) {
  size_t off = 0;
  lv[0].planes = *p;
  for (int l = 1; l < levels; ++l) {
    const ssk_planes& prev = lv[l - 1].planes;
    ssk_planes q = prev;
    q.h = prev.h / 2;
    q.w = prev.w / 2;
    if (q.h < 1 || q.w < 1) return SSK_E_TOO_SMALL;
    q.dtype = level_dtype(p, levels - 1);
    if (q.dtype == SSK_U16 || q.dtype == SSK_U32) q.scale_log2 = p->scale_log2 + 2 * l;
    const int es = esize_of(q.dtype);
    q.row_pitch = (int64_t)(align_up((size_t)q.w * es, 16) / es);
    q.frame_pitch = q.row_pitch * q.h;
    const size_t bytes = align_up((size_t)q.frame_pitch * es * q.n);
    lv[l].offset_r = off;
    off += bytes;
    lv[l].offset_d = off;
    off += bytes;
    lv[l].planes = q;
  }
  (void)win;
  *pyr_bytes = off;
  return SSK_OK;
}

}  // namespace
}  // namespace ssk

using namespace ssk;

extern "C" {

int ssk_abi_version(void) { return SSK_ABI_VERSION; }

const char* ssk_strerror(int code) {
  switch (code) {
    case SSK_OK: return "ok";
    case SSK_E_ARG: return "invalid argument";
    case SSK_E_WINDOW: return "window larger than the image";
    case SSK_E_SHAPE: return "unsupported window shape/size for this engine";
    case SSK_E_WORKSPACE: return "workspace too small";
    case SSK_E_ALIGN: return "planes must be 16-byte aligned with 16-byte row/frame pitches";
    case SSK_E_CUDA: return "CUDA error";
    case SSK_E_LEVELS: return "too many scales for the image size";
    case SSK_E_TOO_SMALL: return "plane too small to downsample";
    default: return "unknown error";
  }
}

size_t ssk_ssim_workspace_bytes(const ssk_planes* p, const ssk_window* win) {
  // enough for any `want`: map launches run on narrower strips (more partials) than
  // score-only launches, a Σq² launch (rect only) may pick the per-window kernel (more
  // partials than the block kernel) and fp64 Gaussian maps run the generic kernel's
  // 64-column tiles, so take the largest of the plans
  size_t bytes = 0;
  for (const int want : {SSK_WANT_Q | SSK_WANT_L | SSK_WANT_CS, SSK_WANT_Q | SSK_MAP_TERMS,
                         SSK_WANT_Q | SSK_WANT_Q2, SSK_WANT_Q | SSK_MAP_TERMS | SSK_MAP_F64}) {
    Plan pl;
    if (plan_ssim(p, win, want, pl)) return 0;
    bytes = std::max(bytes, partial_bytes(pl, p->n) * (pl.gauss ? 1 : 2));  // rect: room for q^2
  }
  return bytes;
}

int ssk_ssim(const ssk_planes* p, const ssk_window* win, int want, double* d_sums, void* d_maps,
             void* d_workspace, size_t workspace_bytes, void* stream) {
  Plan pl;
  const int rc = plan_ssim(p, win, want, pl);
  if (rc) return rc;
  if (!d_sums) return SSK_E_ARG;
  if ((want & (SSK_MAP_TERMS | SSK_MAP_STATS)) && !d_maps) return SSK_E_ARG;
  const bool q2 = (want & SSK_WANT_Q2) != 0;
  if (q2 && pl.gauss) return SSK_E_SHAPE;
  const size_t one = partial_bytes(pl, p->n);
  if (!d_workspace || workspace_bytes < one * (q2 ? 2 : 1)) return SSK_E_WORKSPACE;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  double* partials = static_cast<double*>(d_workspace);
  double* partials2 = q2 ? reinterpret_cast<double*>(static_cast<char*>(d_workspace) + one) : nullptr;
  pl.ba.partials2 = partials2;
  int e = run_plan(pl, partials, d_maps, nullptr, st);
  if (e) return e;
  const int cols = q2 ? 4 : 3;
  e = launch_reduce_partials(partials, (int)pl.nparts_per_frame, p->n, 3, 1.0, d_sums, cols, 0, 0, st);
  if (e || !q2) return e;
  return launch_reduce_partials(partials2, (int)pl.nparts_per_frame, p->n, 1, 1.0, d_sums, 4, 3, 0, st);
}

int ssk_box_window_sums(const ssk_planes* p, int k, int stride, int64_t* d_out, void* d_workspace,
                        size_t workspace_bytes, void* stream) {
  if (!d_out || !p) return SSK_E_ARG;
  if (p->dtype == SSK_F32 || p->dtype == SSK_F64) return SSK_E_ARG;
  ssk_window win{};
  win.shape = SSK_RECT;
  win.k = k;
  win.stride = stride;
  win.c1 = 1.0;
  win.c2 = 1.0;
  Plan pl;
  const int rc = plan_ssim(p, &win, SSK_WANT_Q, pl);
  if (rc) return rc;
  if (!d_workspace || workspace_bytes < partial_bytes(pl, p->n)) return SSK_E_WORKSPACE;
  return run_plan(pl, static_cast<double*>(d_workspace), nullptr, reinterpret_cast<long long*>(d_out),
                  static_cast<cudaStream_t>(stream));
}

int ssk_integral_tables(const ssk_planes* p, void* d_out, void* stream) {
  const int rc = check_planes(p);
  if (rc) return rc;
  if (!d_out) return SSK_E_ARG;
  return launch_integral(static_cast<const unsigned char*>(p->ref),
                         static_cast<const unsigned char*>(p->dist), p->dtype, p->row_pitch,
                         p->frame_pitch, p->n, p->h, p->w, d_out, static_cast<cudaStream_t>(stream));
}

int ssk_downsample(const ssk_planes* src, void* d_dst_ref, void* d_dst_dist, int dst_dtype,
                   int64_t dst_row_pitch, int64_t dst_frame_pitch, void* stream) {
  if (!src || !src->ref || !src->dist || !d_dst_ref || !d_dst_dist) return SSK_E_ARG;
  if (esize_of(src->dtype) == 0 || esize_of(dst_dtype) == 0 || src->n < 1) return SSK_E_ARG;
  if (src->h < 2 || src->w < 2) return SSK_E_TOO_SMALL;
  const int es = esize_of(src->dtype), ed = esize_of(dst_dtype);
  if ((reinterpret_cast<uintptr_t>(src->ref) & 15) || (reinterpret_cast<uintptr_t>(src->dist) & 15) ||
      ((src->row_pitch * es) & 15) || ((src->frame_pitch * es) & 15) ||
      (reinterpret_cast<uintptr_t>(d_dst_ref) & 15) || (reinterpret_cast<uintptr_t>(d_dst_dist) & 15) ||
      ((dst_row_pitch * ed) & 15) || ((dst_frame_pitch * ed) & 15))
    return SSK_E_ALIGN;
  return launch_downsample(static_cast<const unsigned char*>(src->ref),
                           static_cast<const unsigned char*>(src->dist), src->dtype, src->row_pitch,
                           src->frame_pitch, src->n, src->h, src->w,
                           static_cast<unsigned char*>(d_dst_ref), static_cast<unsigned char*>(d_dst_dist),
                           dst_dtype, dst_row_pitch, dst_frame_pitch, static_cast<cudaStream_t>(stream));
}

size_t ssk_msssim_workspace_bytes(const ssk_planes* p, const ssk_window* win, int levels) {
  if (!p || levels < 1 || levels > 16) return 0;
  Level lv[16];
  size_t pyr = 0;
  if (plan_pyramid(p, win, levels, lv, &pyr)) return 0;
  size_t parts = 0;
  for (int l = 0; l < levels; ++l) {
    ssk_planes q = lv[l].planes;
    if (l > 0) q.ref = q.dist = reinterpret_cast<const void*>(kAlign);  // lives in the workspace
    Plan pl;
    if (plan_ssim(&q, win, SSK_WANT_Q | SSK_WANT_L | SSK_WANT_CS, pl)) return 0;
    parts += partial_bytes(pl, p->n);
  }
  return pyr + parts;
}

int ssk_msssim(const ssk_planes* p, const ssk_window* win, int levels, const double* exponents,
               int aggregation, double* d_level_means, double* d_scores, double* d_ssim_means,
               void* d_workspace, size_t workspace_bytes, void* stream) {
  int rc = check_planes(p);
  if (rc) return rc;
  if (!win || !d_level_means || levels < 1 || levels > 16) return SSK_E_ARG;
  if (aggregation < 0 || aggregation > 2 || (aggregation && !exponents)) return SSK_E_ARG;
  if ((std::min(p->h, p->w) >> (levels - 1)) < win->k) return SSK_E_LEVELS;
  const size_t need = ssk_msssim_workspace_bytes(p, win, levels);
  if (need == 0) return SSK_E_ARG;
  if (!d_workspace || workspace_bytes < need) return SSK_E_WORKSPACE;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  unsigned char* ws = static_cast<unsigned char*>(d_workspace);
  Level lv[16];
  size_t pyr = 0;
  rc = plan_pyramid(p, win, levels, lv, &pyr);
  if (rc) return rc;
  for (int l = 1; l < levels; ++l) {
    lv[l].planes.ref = ws + lv[l].offset_r;
    lv[l].planes.dist = ws + lv[l].offset_d;
  }

  // per-level plans (the pyramid levels' geometry is known before any launch)
  FinalizeArgs fa{};
  fa.levels = levels;
  fa.n = p->n;
  fa.aggregation = aggregation;
  fa.level_means = d_level_means;
  fa.scores = d_scores;
  fa.ssim_sums = d_ssim_means;
  for (int l = 0; l < levels; ++l) fa.exps[l] = aggregation ? exponents[l] : 0.0;
  size_t part_off = pyr;
  Plan plans[16];
  for (int l = 0; l < levels; ++l) {
    const bool last = l == levels - 1;
    int want = last ? SSK_WANT_Q : SSK_WANT_CS;
    if (l == 0 && d_ssim_means) want |= SSK_WANT_Q | SSK_WANT_L | SSK_WANT_CS;
    rc = plan_ssim(&lv[l].planes, win, want, plans[l]);
    if (rc) return rc;
    fa.partials[l] = reinterpret_cast<const double*>(ws + part_off);
    fa.nparts[l] = (int)plans[l].nparts_per_frame;
    fa.count[l] = (double)plans[l].gh * (double)plans[l].gw;
    if (plans[l].gauss) {
      plans[l].ga.partials = reinterpret_cast<double*>(ws + part_off);
      plans[l].ga.maps = nullptr;
    }
    part_off += partial_bytes(plans[l], p->n);
  }

  // level 1 fused into the level-0 pass: the wide warp-specialised u8 kernel's producers
  // write the 2x2 sums of the rows they stage anyway (one HBM read of level 0 less)
  const bool fuse_l1 = levels >= 2 && plans[0].gauss && plans[0].ga.vcols == 256 && p->dtype == SSK_U8 &&
                       lv[1].planes.dtype == SSK_U16 && fused_l1_enabled();
  if (fuse_l1) {
    GaussArgs& g0 = plans[0].ga;
    g0.l1_ref = static_cast<unsigned short*>(const_cast<void*>(lv[1].planes.ref));
    g0.l1_dist = static_cast<unsigned short*>(const_cast<void*>(lv[1].planes.dist));
    g0.l1_rp = lv[1].planes.row_pitch;
    g0.l1_fp = lv[1].planes.frame_pitch;
    g0.l1_h = lv[1].planes.h;
    g0.l1_w = lv[1].planes.w;
    rc = run_plan(plans[0], const_cast<double*>(fa.partials[0]), nullptr, nullptr, st);
    if (rc) return rc;
  }

  // 1) the pyramid: up to four levels per pass over the previous top level
  for (int base = fuse_l1 ? 1 : 0; base + 1 < levels;) {
    const int nl = std::min(GS_MAX_LEVELS, levels - 1 - base);
    const ssk_planes& s = lv[base].planes;
    PyramidArgs pa{};
    pa.src_r = static_cast<const unsigned char*>(s.ref);
    pa.src_d = static_cast<const unsigned char*>(s.dist);
    pa.src_rp = s.row_pitch;
    pa.src_fp = s.frame_pitch;
    for (int i = 0; i < nl; ++i) {
      const ssk_planes& d = lv[base + 1 + i].planes;
      pa.dst_r[i] = const_cast<unsigned char*>(static_cast<const unsigned char*>(d.ref));
      pa.dst_d[i] = const_cast<unsigned char*>(static_cast<const unsigned char*>(d.dist));
      pa.dst_rp[i] = d.row_pitch;
      pa.dst_fp[i] = d.frame_pitch;
      pa.hl[i] = d.h;
      pa.wl[i] = d.w;
    }
    rc = launch_pyramid(pa, s.dtype, lv[base + 1].planes.dtype, nl, p->n, st);
    if (rc) return rc;
    base += nl;
  }

  // 2) SSIM per level: level 0 alone (input type, unless already run fused), the
  //    coarser levels batched
  for (int l = fuse_l1 ? 1 : 0; l < levels;) {
    // coarse levels go to the multi-level kernel: 128-column strips, or 256-column strips
    // for u16 levels planned wide (classic kernel, 2 CTAs/SM); one launch per strip width
    auto multi = [&](int i) {
      return i > 0 && plans[i].gauss &&
             (plans[i].ga.vcols == GS_THREADS || (plans[i].ga.vcols == 256 && plans[i].ga.dtype == SSK_U16));
    };
    if (!multi(l)) {  // level 0 and wide u8 / non-Gaussian levels launch alone
      rc = run_plan(plans[l], const_cast<double*>(fa.partials[l]), nullptr, nullptr, st);
      if (rc) return rc;
      ++l;
      continue;
    }
    // Longest tiles first (LPT): every frame pair's tiles of the tallest segments are
    // dispatched before any shorter ones, so the short tiles of the small levels fill
    // the last wave instead of trailing behind it.
    int order[GS_MAX_LEVELS], nl = 0;
    const int vcols = plans[l].ga.vcols;
    while (l < levels && nl < GS_MAX_LEVELS && multi(l) && plans[l].ga.vcols == vcols) order[nl++] = l++;
    for (int i = 1; i < nl; ++i)
      for (int j = i; j > 0 && plans[order[j]].ga.seg_rows > plans[order[j - 1]].ga.seg_rows; --j)
        std::swap(order[j], order[j - 1]);
    GaussLevels gl{};
    gl.npairs = (p->n + 1) / 2;
    long long ctas = 0;
    for (int i = 0; i < nl; ++i) {
      const Plan& pl = plans[order[i]];
      gl.lv[i] = pl.ga;
      gl.cta_off[i] = (int)ctas;
      gl.nstrips[i] = (int)pl.grid.x;
      gl.nseg[i] = (int)pl.grid.y;
      ctas += (long long)pl.grid.x * pl.grid.y * gl.npairs;
    }
    gl.nlev = nl;
    if (ctas > 0x7fffffffLL) return SSK_E_ARG;
    rc = launch_gauss_levels(gl, dim3((unsigned)ctas, 1, 1), win->k, gl.lv[0].dtype, st);
    if (rc) return rc;
  }

  // 3) per-frame means, level-0 SSIM sums and the combined score
  return launch_msssim_finalize(fa, st);
}

}  // extern "C"

namespace {

int plan_volume(const ssk_volume* v, const ssk_window* win, int want, Plan& pl) {
  if (!v || !v->planes || !win || v->h < 1 || v->w < 1 || v->depth < 1 || v->pitch < v->w) return SSK_E_ARG;
  if (win->shape != SSK_RECT) return SSK_E_SHAPE;
  if (win->k < 1 || win->stride < 1) return SSK_E_ARG;
  if (win->k > v->h || win->k > v->w) return SSK_E_WINDOW;
  const int k = win->k, s = win->stride;
  BoxArgs& a = pl.ba;
  a = BoxArgs{};
  a.n = 1;
  a.h = v->h;
  a.w = v->w;
  a.k = k;
  a.s = s;
  a.esize = 1;
  a.dtype = SSK_U8;
  pl.gh = a.gh = grid_extent(v->h, k, s);
  pl.gw = a.gw = grid_extent(v->w, k, s);
  a.sscale1 = a.sscale2 = 1.0;
  a.area = (double)k * (double)k * (double)v->depth;
  int ex = 0;
  a.area_pow2 = std::frexp(a.area, &ex) == 0.5 ? 1 : 0;
  a.inv_area = 1.0 / a.area;
  a.c1 = win->c1;
  a.c2 = win->c2;
  // integer-domain score epilogue (box_fast_terms) over the exact temporal window sums:
  // exact while area^2 * max_sample^2 < 2^52 (samples <= 16 bits)
  a.area_i = (int)(k * k * v->depth);
  a.c1d = win->c1 * a.area * a.area;
  a.c2d = win->c2 * a.area * a.area;
  a.fast_ok = (a.area * a.area * 65535.0 * 65535.0 < 4.0e15) ? 1 : 0;
  a.want = want;
  a.map_plane = (long long)pl.gh * pl.gw;
  a.map_frame = a.map_plane * ((want & SSK_MAP_STATS) ? 5 : 3);
  a.mom = static_cast<const long long*>(v->planes);
  a.mom_rp = v->pitch;
  a.mom_plane = v->pitch * v->h;
  if (!v->is_float && k <= BX_THREADS - 15) {
    pl.box_int = true;
    pl.wide = true;
    a.na = (BX_THREADS - 15 - k) / s + 1;
    const int nstrips = (pl.gw + a.na - 1) / a.na;
    int vr = 32 / s;
    vr = vr < 1 ? 1 : (vr > 8 ? 8 : vr);
    a.ch = vr * s;
    a.in_pitch = 16;  // no staging for moment planes
    a.nslot = (k + s - 1) / s + 1;
    // a volume is scored one frame at a time: cut the frame into enough segments for
    // ~4 CTAs per SM of a B200 (592 CTAs; a constant, so results depend on the geometry
    // only), between 16 and 256 rows per segment
    const int lo = std::max(1, (16 + s - 1) / s), hi = (256 + s - 1) / s;
    int seg_anchors = (int)std::min<long long>(hi, std::max<long long>(lo, (pl.gh * (long long)nstrips + 591) / 592));
    long long nseg = (pl.gh + seg_anchors - 1) / seg_anchors;
    seg_anchors = (int)((pl.gh + nseg - 1) / nseg);
    a.seg_anchors = seg_anchors;
    nseg = (pl.gh + seg_anchors - 1) / seg_anchors;
    pl.grid = dim3(nstrips, (unsigned)nseg, 1);
    pl.nparts_per_frame = (size_t)nstrips * nseg;
    return SSK_OK;
  }
  pl.box_int = false;
  pl.block = dim3(32, 4);
  pl.grid = dim3((pl.gw + 31) / 32, (pl.gh + 3) / 4, 1);
  pl.nparts_per_frame = (size_t)pl.grid.x * pl.grid.y;
  return SSK_OK;
}

}  // namespace

extern "C" {

int ssk_volume_update(const ssk_volume* v, const void* new_ref, const void* new_dist, const void* old_ref,
                      const void* old_dist, int dtype, int64_t src_row_pitch, int mode, void* stream) {
  if (!v || !v->planes || !new_ref || !new_dist || mode < 0 || mode > 2) return SSK_E_ARG;
  if (mode == 2 && (!old_ref || !old_dist)) return SSK_E_ARG;
  if (src_row_pitch < v->w) return SSK_E_ARG;
  return launch_volume_update(v->planes, v->is_float, v->pitch * v->h, v->pitch, new_ref, new_dist, old_ref,
                              old_dist, dtype, src_row_pitch, v->h, v->w, mode, static_cast<cudaStream_t>(stream));
}

int ssk_volume_refresh(const ssk_volume* v, const void* const* refs, const void* const* dists, int count,
                       int dtype, int64_t src_row_pitch, void* stream) {
  if (!v || !v->planes || !v->is_float || !refs || !dists) return SSK_E_ARG;
  return launch_volume_refresh(v->planes, v->pitch * v->h, v->pitch, refs, dists, count, dtype, src_row_pitch,
                               v->h, v->w, static_cast<cudaStream_t>(stream));
}

size_t ssk_volume_workspace_bytes(const ssk_volume* v, const ssk_window* win) {
  Plan pl;
  if (plan_volume(v, win, SSK_WANT_Q | SSK_WANT_L | SSK_WANT_CS, pl)) return 0;
  return partial_bytes(pl, 1);
}

int ssk_volume_ssim(const ssk_volume* v, const ssk_window* win, int want, double* d_sums, void* d_maps,
                    void* d_workspace, size_t workspace_bytes, void* stream) {
  Plan pl;
  const int rc = plan_volume(v, win, want, pl);
  if (rc) return rc;
  if (!d_sums || ((want & (SSK_MAP_TERMS | SSK_MAP_STATS)) && !d_maps)) return SSK_E_ARG;
  if (!d_workspace || workspace_bytes < partial_bytes(pl, 1)) return SSK_E_WORKSPACE;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  double* partials = static_cast<double*>(d_workspace);
  pl.ba.partials = partials;
  pl.ba.maps = static_cast<double*>(d_maps);
  int e = pl.box_int ? launch_box_moments(pl.ba, pl.grid, st)
                     : launch_volume_direct(pl.ba, static_cast<const double*>(v->planes), pl.grid, pl.block, st);
  if (e) return e;
  return launch_reduce_partials(partials, (int)pl.nparts_per_frame, 1, 3, 1.0, d_sums, 3, 0, 0, st);
}

int ssk_stats_from_sums(const double* d_s1, const double* d_s2, const double* d_q1, const double* d_q2,
                        const double* d_p12, int64_t count, double area, double* d_out, void* stream) {
  if (!d_s1 || !d_s2 || !d_q1 || !d_q2 || !d_p12 || !d_out || count < 0 || !(area > 0.0)) return SSK_E_ARG;
  return launch_stats_from_sums(d_s1, d_s2, d_q1, d_q2, d_p12, count, area, d_out,
                                static_cast<cudaStream_t>(stream));
}

int ssk_term_maps(const double* d_mu1, const double* d_mu2, const double* d_var1, const double* d_var2,
                  const double* d_cov, int64_t count, double c1, double c2, double* d_out, void* stream) {
  if (!d_mu1 || !d_mu2 || !d_var1 || !d_var2 || !d_cov || !d_out || count < 0) return SSK_E_ARG;
  return launch_term_maps(d_mu1, d_mu2, d_var1, d_var2, d_cov, count, c1, c2, d_out,
                          static_cast<cudaStream_t>(stream));
}

int ssk_divide(const double* d_x, int64_t count, double divisor, double* d_out, void* stream) {
  if (!d_x || !d_out || count < 0) return SSK_E_ARG;
  return launch_divide(d_x, count, divisor, d_out, static_cast<cudaStream_t>(stream));
}

size_t ssk_pairwise_workspace_bytes(const ssk_maps* m) {
  if (!m || m->n < 1 || m->h < 1 || m->w < 1) return 0;
  return pairwise_workspace_bytes(m);
}

int ssk_pairwise_sum(const ssk_maps* m, int expr, double p, double a, double b, const double* d_c, double* d_out,
                     void* d_workspace, size_t workspace_bytes, void* stream) {
  if (!m || !m->values || !d_out || m->n < 1 || m->h < 1 || m->w < 1 || m->n > 65535) return SSK_E_ARG;
  if (m->dtype != SSK_F32 && m->dtype != SSK_F64) return SSK_E_ARG;
  if (m->row_pitch < m->w || m->frame_pitch < m->row_pitch * (int64_t)m->h) return SSK_E_ARG;
  if (expr < SSK_PW_V || expr > SSK_PW_LW) return SSK_E_ARG;
  if ((expr == SSK_PW_SQDEV || expr == SSK_PW_ABSDEV_P || expr == SSK_PW_PP) && !d_c) return SSK_E_ARG;
  if (expr == SSK_PW_LW && (!m->aux || m->aux_row_pitch < m->w)) return SSK_E_ARG;
  if (!d_workspace || workspace_bytes < pairwise_workspace_bytes(m)) return SSK_E_WORKSPACE;
  return launch_pairwise_maps(m, expr, p, a, b, d_c, d_out, d_workspace, static_cast<cudaStream_t>(stream));
}

uint64_t ssk_launch_count(void) { return g_launches.load(); }

int ssk_host_register(void* ptr, size_t bytes, int read_only) {
  if (!ptr || !bytes) return SSK_E_ARG;
  const unsigned flags = cudaHostRegisterPortable | (read_only ? cudaHostRegisterReadOnly : 0u);
  const cudaError_t e = cudaHostRegister(ptr, bytes, flags);
  if (e != cudaSuccess) {
    (void)cudaGetLastError();  // not sticky: clear it so later launch checks do not see it
    return -1000 - (int)e;     // SSK_E_CUDA family; the cudaError_t is recoverable for diagnostics
  }
  return SSK_OK;
}

int ssk_host_unregister(void* ptr) {
  if (!ptr) return SSK_E_ARG;
  if (cudaHostUnregister(ptr) != cudaSuccess) {
    (void)cudaGetLastError();
    return SSK_E_CUDA;
  }
  return SSK_OK;
}

int ssk_probe_fp32_tflops(double seconds, double* tflops, void* stream) {
  if (!tflops || seconds <= 0) return SSK_E_ARG;
  return probe_fp32(seconds, tflops, static_cast<cudaStream_t>(stream));
}

}  // extern "C"
