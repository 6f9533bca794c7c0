/*
 * ssimk.h — C ABI of the B200-native SSIM engine (libssimk.so).
 *
 * This is the drop-in boundary for the hot path of the reference package
 * `ssimkit` (arXiv 2101.06354, /root/reference/pkg/src/ssimkit).  The reference
 * has no FFI: its only dispatch seam is the `engine` string of
 * `local_statistics` (src/stats.py:205-261, engine resolution :223-228).  Each
 * entry point below replaces one numpy routine on that path; the replaced
 * reference code is cited beside it.  INTEGRATION.md shows the ctypes binding
 * a ssimkit maintainer would add behind that seam.
 *
 * Conventions
 *  - Every pointer named `d_*` (and every pointer inside ssk_planes) is a
 *    DEVICE pointer owned by the caller; nothing is allocated inside a call.
 *    Scratch comes from a caller-provided workspace sized by the matching
 *    *_workspace_bytes query.
 *  - Calls are asynchronous on `stream` (a cudaStream_t / CUstream passed as
 *    void*; NULL = legacy default stream) and re-entrant (no global mutable
 *    state apart from a monotonically increasing launch counter).
 *  - Return value: 0 on success, a negative SSK_E* code otherwise
 *    (ssk_strerror gives the text).  Argument errors are detected before any
 *    launch; the Python layer maps them onto the reference's exception classes
 *    (src/errors.py).
 *  - Geometry follows the reference exactly (valid region only, anchor (0,0),
 *    window cell (r,c) covers rows [r*s, r*s+k) and cols [c*s, c*s+k);
 *    grid = ((H-k)//s + 1, (W-k)//s + 1); src/stats.py:130-164).
 */
#ifndef SSIMK_H
#define SSIMK_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SSK_ABI_VERSION 9

/* sample storage types */
enum {
  SSK_U8 = 1,  /* uint8  samples (8-bit luma)                               */
  SSK_U16 = 2, /* uint16 samples (9..16-bit luma, or a scaled pyramid level) */
  SSK_U32 = 3, /* uint32 samples (scaled pyramid levels of deep inputs)      */
  SSK_F32 = 4, /* float32 samples                                           */
  SSK_F64 = 5  /* float64 samples (downsample only)                         */
};

/* window shapes (WindowSpec.shape, src/config.py:31-75) */
enum { SSK_RECT = 1, SSK_GAUSS = 2 };

/* what a scoring call produces */
enum {
  SSK_WANT_Q = 1,      /* per-frame sum of q = l*cs                           */
  SSK_WANT_L = 2,      /* per-frame sum of l                                  */
  SSK_WANT_CS = 4,     /* per-frame sum of cs                                 */
  SSK_MAP_TERMS = 8,   /* write the l, cs, q maps (3 planes per frame)        */
  SSK_MAP_STATS = 16,  /* write mu1, mu2, var1, var2, cov (5 planes per frame) */
  SSK_WANT_Q2 = 32,    /* rect windows: also the per-frame sum of q^2, d_sums is then
                          [n][4] (CoV / MD(2) pooling without a map, src/pooling.py:157-166) */
  SSK_MAP_F64 = 64     /* Gaussian windows: maps (and sums) from the fp64 kernel, maps stored
                          as float64 -- the reference's own precision, for the map API
                          (ssim_map / local_statistics); without it Gaussian maps are the
                          fp32 kernel's, stored as float32 */
};

/* error codes */
enum {
  SSK_OK = 0,
  SSK_E_ARG = -1,          /* bad argument (null pointer, bad enum, bad size)   */
  SSK_E_WINDOW = -2,       /* window larger than the image                      */
  SSK_E_SHAPE = -3,        /* unsupported window/engine combination             */
  SSK_E_WORKSPACE = -4,    /* workspace too small                               */
  SSK_E_ALIGN = -5,        /* base pointer / pitch not 16-byte aligned          */
  SSK_E_CUDA = -6,         /* CUDA launch or runtime error                      */
  SSK_E_LEVELS = -7,       /* too many scales for the image (TooManyLevels)     */
  SSK_E_TOO_SMALL = -8     /* cannot downsample (TooSmall)                      */
};

/*
 * A batch of n reference/distorted frame pairs of identical geometry.
 * Pointers must be 16-byte aligned and row_pitch*sizeof(sample) a multiple
 * of 16 (the Python layer pads when a caller's tensor is not).
 * Sample value = stored value * 2^-scale_log2 (scale_log2 = 2*s for a scaled
 * integer pyramid level s, whose stored values are sums of 4^s samples).
 */
typedef struct ssk_planes {
  const void* ref;
  const void* dist;
  int32_t dtype;        /* SSK_U8 / SSK_U16 / SSK_U32 / SSK_F32             */
  int32_t scale_log2;   /* 0 for ordinary planes                            */
  int32_t n, h, w;      /* frames, rows, columns                            */
  int32_t bit_depth;    /* of the source samples (8..16); selects shift L/2 */
  int64_t row_pitch;    /* elements between rows                            */
  int64_t frame_pitch;  /* elements between frames                          */
} ssk_planes;

/* Window (WindowSpec) plus the SSIM constants (SsimConfig.c1/.c2,
 * src/config.py:267-285).  Gaussian windows (gaussian_kernel, src/stats.py:30-44,
 * applied separably with the normalised 1-D taps g/sum(g)) are given EITHER by
 *   sigma > 0 and taps[] all zero: the library builds the taps itself (any odd
 *     k >= 3 up to SSK_GAUSS_MAX_K), or by
 *   taps[0..k-1] (k <= 31): the caller's normalised taps, validated -- every tap
 *     finite and >= 0, taps[i] == taps[k-1-i] exactly, sum within 1e-5 of 1 --
 *     else SSK_E_ARG (sigma, if also given, is then only informative).
 * Windows wider than 31 taps need sigma (they run the generic fp64 kernel). */
#define SSK_GAUSS_MAX_K 255
typedef struct ssk_window {
  int32_t shape;    /* SSK_RECT or SSK_GAUSS                               */
  int32_t k;        /* window size (gauss: odd, 3..255; rect: 1..4096)     */
  int32_t stride;   /* >= 1                                                */
  int32_t _pad;
  double c1, c2;    /* (k1*L)^2, (k2*L)^2                                  */
  double sigma;     /* gauss: Gaussian sigma (> 0), see above              */
  float taps[32];   /* gauss, k <= 31: normalised 1-D taps, or all zero    */
} ssk_window;

/* ------------------------------------------------------------------------ */

int ssk_abi_version(void);
const char* ssk_strerror(int code);

/* Workspace for ssk_ssim / ssk_msssim over this batch geometry. */
size_t ssk_ssim_workspace_bytes(const ssk_planes* p, const ssk_window* win);
size_t ssk_msssim_workspace_bytes(const ssk_planes* p, const ssk_window* win, int levels);

/*
 * Fused local statistics + SSIM terms + mean-pooling reduction for a batch.
 * Replaces local_statistics (src/stats.py:205-261: _sliding_weighted_sums
 * :155-164 for Gaussian windows, build_integral_set/_grid_window_sums
 * :96-141 for rect windows), stats_from_sums (:185-202),
 * term_maps_from_stats (src/ssim.py:31-46) and mssim (src/ssim.py:55-65).
 *   d_sums  : [n][3] float64, per-frame (sum q, sum l, sum cs) over the grid
 *             (only the components selected by `want` are meaningful).
 *   d_maps  : optional; SSK_MAP_TERMS -> [n][3][gh][gw] (l, cs, q),
 *             SSK_MAP_STATS -> [n][5][gh][gw] (mu1, mu2, var1, var2, cov);
 *             float32 for Gaussian windows (float64 with SSK_MAP_F64), float64 for
 *             rect windows.
 * Rect windows on integer samples use exact integer window sums (the
 * integral engine's int64 arithmetic, src/stats.py:101-103) and a float64
 * epilogue in the reference's operation order, so their maps are
 * bit-identical to the reference.
 */
int ssk_ssim(const ssk_planes* p, const ssk_window* win, int want,
             double* d_sums, void* d_maps, void* d_workspace, size_t workspace_bytes,
             void* stream);

/*
 * Exact integer window sums for a rect window on integer samples:
 * d_out [n][5][gh][gw] int64 = the five grids
 * _grid_window_sums(build_integral_set(ref, dist).table(t), k, s)
 * for t in (sum1, sum2, sq1, sq2, prod) (src/stats.py:96-141), bit-exact.
 */
int ssk_box_window_sums(const ssk_planes* p, int k, int stride, int64_t* d_out,
                        void* d_workspace, size_t workspace_bytes, void* stream);
/* workspace: ssk_ssim_workspace_bytes(p, rect window k/stride) */

/*
 * Summed-area tables (src/stats.py:66-71, build_integral_set :96-116):
 * d_out [n][5][h+1][w+1], int64 for integer samples (exact) or float64.
 */
int ssk_integral_tables(const ssk_planes* p, void* d_out, void* stream);

/*
 * 2x2 mean pyramid step (dyadic_downsample, src/multiscale.py:19-33).
 * Integer inputs produce stored sums of 4 (dst scale_log2 = src + 2, exact);
 * float inputs produce ((a00+a01)+a10)+a11)/4 in their own precision.
 * dst: [n][h/2][w/2] with the given pitch, dtype dst_dtype.
 */
int ssk_downsample(const ssk_planes* src, void* d_dst_ref, void* d_dst_dist, int dst_dtype,
                   int64_t dst_row_pitch, int64_t dst_frame_pitch, void* stream);

/*
 * Whole MS-SSIM pyramid for a batch (scale_scores + combine_scale_scores,
 * src/multiscale.py:36-74).  One pass builds every pyramid level (exact scaled
 * integers for integer samples), one fused SSIM pass per sample type scores
 * the levels, and one finalize kernel writes
 *   d_level_means [n][levels] float64: mean(cs) for levels < L-1, mean(l*cs)
 *                 at the coarsest level;
 *   d_scores      [n] (nullable): the combined score, aggregation 1 = product
 *                 of max(s, 0)^e, 2 = sum of e*s, with `exponents` (host array,
 *                 `levels` entries, already renormalised for sum/fast4 as
 *                 MultiscaleSpec.effective_exponents does); aggregation 0 = none;
 *   d_ssim_means  [n][3] (nullable): level-0 (mean q, mean l, mean cs) -- the
 *                 plain SSIM record (score, l_mean, cs_mean) of the same pass
 *                 (scale 0 is shared).
 */
int ssk_msssim(const ssk_planes* p, const ssk_window* win, int levels, const double* exponents,
               int aggregation, double* d_level_means, double* d_scores, double* d_ssim_means,
               void* d_workspace, size_t workspace_bytes, void* stream);

/*
 * SSIM-3D rolling volumes (src/spatiotemporal.py:28-207).  The caller owns the
 * five temporal-sum planes [5][h][pitch] (x, y, x^2, y^2, xy summed over the
 * last `depth` frame pairs): int64 for integer samples (exact, no drift, so the
 * reference's periodic refresh is a no-op) or float64 for float samples.
 */
typedef struct ssk_volume {
  void* planes;
  int32_t is_float;     /* 0: int64 planes (u8/u16 frames), 1: float64 planes (f64 frames) */
  int32_t h, w;
  int32_t depth;        /* frames currently summed (1..Kt)                  */
  int64_t pitch;        /* elements between rows of one plane               */
} ssk_volume;

/* mode 0: planes = terms(new); 1: planes += terms(new);
 * 2: planes = planes - terms(old) + terms(new)  (RollingVolume.push, :60-97).
 * Frames: device [h][src_row_pitch] of `dtype` (SSK_U8/SSK_U16 for int64 planes,
 * SSK_F64 for float64 planes). */
int ssk_volume_update(const ssk_volume* v, const void* new_ref, const void* new_dist, const void* old_ref,
                      const void* old_dist, int dtype, int64_t src_row_pitch, int mode, void* stream);
/* float64 planes only: recompute from `count` buffered frame pairs, oldest first
 * (RollingVolume._refresh / direct_sums, :99-115); refs/dists: HOST arrays of
 * device pointers, count <= 64. */
int ssk_volume_refresh(const ssk_volume* v, const void* const* refs, const void* const* dists, int count,
                       int dtype, int64_t src_row_pitch, void* stream);
size_t ssk_volume_workspace_bytes(const ssk_volume* v, const ssk_window* win);
/* k x k x depth window SSIM over the volume (RollingVolume.local_statistics +
 * ssim3d_map, :116-149): rect windows only; area = k*k*depth.  d_sums [1][3]
 * as in ssk_ssim; optional float64 maps (SSK_MAP_TERMS / SSK_MAP_STATS). */
int ssk_volume_ssim(const ssk_volume* v, const ssk_window* win, int want, double* d_sums, void* d_maps,
                    void* d_workspace, size_t workspace_bytes, void* stream);

/*
 * Resolution adaptation: integer-factor block averaging
 * (box_downsample, src/adaptation.py:93-110).  Output (ceil(h/f), ceil(w/f));
 * trailing partial blocks average over their actual size.
 *   dst_dtype SSK_F64: sum / (rows*cols) with one IEEE division -- bit-identical
 *                      to the reference for integer samples (exact sums);
 *   dst_dtype SSK_U16 / SSK_U32: the exact block sums of integer samples (the
 *                      caller must have h % f == 0 and w % f == 0; for a power
 *                      of two f the result is a scaled plane with
 *                      scale_log2 = src scale_log2 + 2*log2(f)).
 */
int ssk_box_downsample(const ssk_planes* src, int factor, void* d_dst_ref, void* d_dst_dist, int dst_dtype,
                       int64_t dst_row_pitch, int64_t dst_frame_pitch, void* stream);

/*
 * Spatial pooling of a batch of quality maps on the device
 * (pool_spatial, src/pooling.py:157-243).  Kinds follow SPATIAL_KINDS (:29).
 * Order statistics (fns quartiles, pp cutoff) are exact: a radix select on
 * the values' order-preserving bit patterns, interpolated with numpy's
 * 'linear' percentile rule (virtual index n*q + (1 - q) - 1, lerp flipped at
 * gamma >= 0.5), so they equal np.percentile bit for bit.
 */
enum {
  SSK_POOL_AM = 0,   /* mean                                                */
  SSK_POOL_COV = 1,  /* std / mean (NaN result for a zero mean: ZeroMeanCoV) */
  SSK_POOL_MD = 2,   /* (mean |v - mean|^p)^(1/p) ^ o                        */
  SSK_POOL_FNS = 3,  /* (min + Q1 + median + Q3 + max) / 5                    */
  SSK_POOL_DW = 4,   /* sum((1-v)^p v) / sum((1-v)^p), mean if all v == 1    */
  SSK_POOL_MINK = 5, /* mean (1-v)^p                                          */
  SSK_POOL_LW = 6,   /* mean w(mu) v, w = [mu >= a] (b == 0) or clip((mu-a)/b) */
  SSK_POOL_PP = 7,   /* mean of v/rs below the ps-th percentile, v above     */
  SSK_POOL_PCTL = 8  /* np.percentile(v, ps) itself (pp's cutoff; exact)     */
};

typedef struct ssk_maps {
  const void* values;        /* device quality values                                    */
  const void* aux;           /* device mean-luminance map (SSK_POOL_LW only), else NULL  */
  int32_t dtype;             /* SSK_F32 or SSK_F64 (values and aux)                      */
  int32_t n, h, w;           /* maps, rows, columns                                      */
  int64_t row_pitch, frame_pitch;          /* elements                                   */
  int64_t aux_row_pitch, aux_frame_pitch;  /* elements                                   */
} ssk_maps;

typedef struct ssk_pooler {
  int32_t kind;              /* SSK_POOL_*                                               */
  int32_t _pad;
  double p, o;               /* md / dw / mink exponent, md outer exponent               */
  double a, b;               /* lw lower luminance limit, ramp length                    */
  double ps, rs;             /* pp percentile, down-weighting divisor                    */
} ssk_pooler;

/* numpy-order sums for the per-map pooling API: for each of the n maps (row-major
 * flattened, as pool_spatial's v.reshape(-1)), the sum of an elementwise fp64 expression in
 * np.add.reduce's pairwise order (PW_BLOCKSIZE 128, starting from 0.0) -- bit-identical to
 * the reference's numpy reductions on the same values (src/pooling.py:157-243):
 *   SSK_PW_V            v
 *   SSK_PW_SQDEV        (v - c)^2                 np.std's second pass (c = the mean)
 *   SSK_PW_ABSDEV_P     |v - c| ** p              md
 *   SSK_PW_ONEMINUS_P   (1 - v) ** p              mink, dw's total
 *   SSK_PW_DW_NUM       ((1 - v) ** p) * v        dw
 *   SSK_PW_PP           v <= c ? v / p : v        pp (c = the cutoff, p = rs)
 *   SSK_PW_LW           w(aux) * v                lw: w = aux >= a (b == 0), else
 *                                                 clip((aux - a) / b, 0, 1)
 * d_c: per-map centre [n] (NULL when unused).  `** p` follows numpy's fast scalar powers
 * (2, 1, 0.5, -1, 0); integer p in [3, 64] is computed in double-double and rounded once
 * (libm pow's correctly rounded result in practice); other p use CUDA pow (<= 2 ulp).
 * Workspace: ssk_pairwise_workspace_bytes(m). */
enum { SSK_PW_V = 0, SSK_PW_SQDEV = 1, SSK_PW_ABSDEV_P = 2, SSK_PW_ONEMINUS_P = 3, SSK_PW_DW_NUM = 4,
       SSK_PW_PP = 5, SSK_PW_LW = 6 };
size_t ssk_pairwise_workspace_bytes(const ssk_maps* m);
int ssk_pairwise_sum(const ssk_maps* m, int expr, double p, double a, double b, const double* d_c, double* d_out,
                     void* d_workspace, size_t workspace_bytes, void* stream);

size_t ssk_pool_workspace_bytes(const ssk_maps* m, const ssk_pooler* pool);
/* CoV / MD(p = 2, o) pooling without a map, from the [n][4] per-frame sums of an
 * ssk_ssim(..., SSK_WANT_Q2) pass over `count` windows (one-pass variance,
 * ~1e-11 relative to numpy's two-pass std); d_out [n]; d_means [n][3]
 * (nullable) = mean q, mean l, mean cs. */
int ssk_pool_moments(const double* d_sums, int n, double count, const ssk_pooler* pool, double* d_out,
                     double* d_means, void* stream);
/* d_out [n] pooled scores; d_mean [n] (nullable) the plain mean of each map. */
int ssk_pool_spatial(const ssk_maps* m, const ssk_pooler* pool, double* d_out, double* d_mean,
                     void* d_workspace, size_t workspace_bytes, void* stream);

/*
 * Colorimetric models (src/color.py:27-371): qssim, cmssim, hssim and the
 * conversions they need.  A color frame batch is three device planes per
 * frame; 4:2:0 chroma planes are ceil(h/2) x ceil(w/2) and are upsampled by
 * nearest neighbour (upsample_chroma, :92-101) where a model needs co-sited
 * channels.
 */
enum { SSK_SPACE_RGB = 1, SSK_SPACE_YCBCR = 2 };
enum {
  SSK_CONV_RGB = 1,       /* -> R, G, B (YCbCr input: inverse BT.709, clamped, :76-89)   */
  SSK_CONV_YCBCR = 2,     /* -> Y, Cb, Cr 4:4:4 (RGB input: forward BT.709, :64-73)      */
  SSK_CONV_LUMA = 3,      /* -> luma_of (:104-108)                                       */
  SSK_CONV_HUE = 4,       /* -> hue_plane scaled to [0, L] (:341-362)                     */
  SSK_CONV_LAB_EMBED = 5  /* -> CIELAB * L/100, qssim's 'lab' embedding (:172-178)        */
};

typedef struct ssk_color {
  const void* ch[3];           /* device planes (R,G,B or Y,Cb,Cr)                     */
  int32_t dtype;               /* SSK_U8 / SSK_U16 / SSK_F32 / SSK_F64                  */
  int32_t space;               /* SSK_SPACE_RGB / SSK_SPACE_YCBCR                       */
  int32_t subsampling;         /* 0 = 4:4:4, 1 = 4:2:0 (YCbCr only)                     */
  int32_t n, h, w;             /* frames, luma rows, luma columns                       */
  int32_t bit_depth;           /* L = 2^bit_depth - 1                                   */
  int64_t row_pitch[3];        /* elements, per channel                                 */
  int64_t frame_pitch[3];
} ssk_color;

/* float64 planes out: d_out[f * out_frame_pitch + plane * h * out_row_pitch + y * out_row_pitch + x]. */
int ssk_color_convert(const ssk_color* src, int op, double* d_out, int64_t out_row_pitch, int64_t out_frame_pitch,
                      void* stream);

/* Quaternion SSIM (qssim, :181-256) of two float64 embeddings [n][3][h][row_pitch]
 * (frame_pitch elements between frames), rect k x k window, stride; d_means [n]. */
size_t ssk_qssim_workspace_bytes(int n, int h, int w, int k, int stride);
int ssk_qssim(const double* d_emb_ref, const double* d_emb_dist, int n, int h, int w, int64_t row_pitch,
              int64_t frame_pitch, int k, int stride, double c1, double c2, double* d_means, void* d_workspace,
              size_t workspace_bytes, void* stream);

/* CIELAB difference (delta_e_map, :290-296; smooth = opponent-space chroma
 * smoothing) sampled at the centres of the k/stride window grid:
 * d_out [n][gh][gw]; mode 0 = dE, mode 1 = 1 - dE/45 (cmssim's weight before
 * the clamp to [0, 1], :299-334).  k = stride = 1 gives the full map. */
size_t ssk_delta_e_workspace_bytes(int n, int h, int w);
int ssk_delta_e(const ssk_color* ref, const ssk_color* dist, int smooth, int k, int stride, int mode, double* d_out,
                int64_t out_row_pitch, int64_t out_frame_pitch, void* d_workspace, size_t workspace_bytes,
                void* stream);

/* Page-lock an existing host range (e.g. a memory-mapped media file) so frame planes
 * are DMA'd straight to the device with no staging copy; read_only for read-only
 * mappings.  0, or -1000 - cudaError_t when the driver refuses (the error is
 * cleared, nothing else is affected). */
int ssk_host_register(void* ptr, size_t bytes, int read_only);
int ssk_host_unregister(void* ptr);

/* Elementwise fp64 map arithmetic of the public API, in the reference's operation order
 * (bit-identical to numpy on the same inputs).  Device pointers, `count` elements each:
 *   ssk_stats_from_sums: stats_from_sums (src/stats.py:185-202); d_out [5][count] =
 *     mu1, mu2, var1, var2 (clamped at 0), cov (not clamped), from window sums over `area`;
 *   ssk_term_maps: term_maps_from_stats (src/ssim.py:31-46); d_out [3][count] = l, cs, q;
 *   ssk_divide: d_out[i] = d_x[i] / divisor (IEEE division: per-frame means from sums). */
int ssk_stats_from_sums(const double* d_s1, const double* d_s2, const double* d_q1, const double* d_q2,
                        const double* d_p12, int64_t count, double area, double* d_out, void* stream);
int ssk_term_maps(const double* d_mu1, const double* d_mu2, const double* d_var1, const double* d_var2,
                  const double* d_cov, int64_t count, double c1, double c2, double* d_out, void* stream);
int ssk_divide(const double* d_x, int64_t count, double divisor, double* d_out, void* stream);

/* Number of kernels this library has launched since load (for bench.py). */
uint64_t ssk_launch_count(void);

/* Sustained FP32 FMA throughput probe (roofline denominator), TFLOP/s. */
int ssk_probe_fp32_tflops(double seconds, double* tflops, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SSIMK_H */
