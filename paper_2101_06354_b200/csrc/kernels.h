// Internal kernel argument blocks and launchers (not part of the C ABI).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace ssk {

// ---------------- K1: Gaussian window ----------------
constexpr int GS_THREADS = 128;  // one input column per thread in the V pass
constexpr int GS_VCOLS = 128;    // input columns per strip (output columns: 16-aligned 128 - (k - 1))
constexpr int GS_G = 8;          // output rows per chunk

struct GaussArgs {
  const unsigned char* ref;
  const unsigned char* dist;
  long long row_pitch_b, frame_pitch_b;  // bytes
  int dtype, esize;
  int n, h, w;
  int ho, wo;                 // dense output extents (h-k+1, w-k+1)
  int gh, gw, stride;         // anchor grid
  int seg_rows;               // output rows per segment (gridDim.y segments)
  float conv_scale, conv_bias;  // shifted sample = fma(raw_or_biased, scale, bias)
  float shift;                // added back to the means
  float c1, c2;
  float one;                  // 1.0f, opaque to ptxas: sum += v * one stays an FFMA2 whose product is never
                              // contracted with the multiply that formed v (rounding independent of `want`)
  int want;
  int exact_sq;               // shifted samples square exactly in fp32 (symmetric fast products)
  int vcols;                  // V-pass columns per CTA: 128, or 256 (wide warp-specialised u8 kernel)
  float taps[32];
  double* partials;           // [n][gridDim.y][gridDim.x][3]; gridDim.z = ceil(n / 2) frame pairs
  void* maps;                 // float32 [n][planes][gh][gw]
  long long map_plane, map_frame;
  // optional fused MS-SSIM level 1 (u16 sums of 2x2 blocks) written by the producer warps
  // of the wide warp-specialised u8 kernel from the rows they stage anyway; null = off
  unsigned short* l1_ref;
  unsigned short* l1_dist;
  long long l1_rp, l1_fp;     // elements
  int l1_h, l1_w;
};

constexpr int GS_MAX_LEVELS = 4;  // pyramid levels fused into one multi-level launch

// Several pyramid levels (same sample type) scored by one launch.
struct GaussLevels {
  GaussArgs lv[GS_MAX_LEVELS];
  int nlev;
  int npairs;                  // frame pairs (two frames per CTA)
  int cta_off[GS_MAX_LEVELS];  // first blockIdx.x of each level (level-major, then pair, then tile)
  int nstrips[GS_MAX_LEVELS];
  int nseg[GS_MAX_LEVELS];
};

int launch_gauss_levels(const GaussLevels& p, dim3 grid, int k, int dtype, cudaStream_t st);

// output columns per strip for a V pass of vc columns (16-column aligned strips)
inline int gauss_tw(int k, int vc = GS_VCOLS) { return ((vc - (k - 1)) / 16) * 16; }
int launch_gauss(const GaussArgs& a, dim3 grid, int k, cudaStream_t st);
int launch_gauss_u8(const GaussArgs& a, dim3 grid, int k, cudaStream_t st);
int launch_gauss_u16(const GaussArgs& a, dim3 grid, int k, cudaStream_t st);
int launch_gauss_u32(const GaussArgs& a, dim3 grid, int k, cudaStream_t st);
int launch_gauss_f32(const GaussArgs& a, dim3 grid, int k, cudaStream_t st);

// ---------------- numpy-order map sums for the per-map pooling API (pool_exact.cu) ----------------
size_t pairwise_workspace_bytes(const ssk_maps* m);
int launch_pairwise_maps(const ssk_maps* m, int expr, double p, double a, double b, const double* d_c,
                         double* d_out, void* d_ws, cudaStream_t st);

// ---------------- elementwise map arithmetic of the public API (aux_kernels.cu) ----------------
int launch_stats_from_sums(const double* s1, const double* s2, const double* q1, const double* q2,
                           const double* p12, long long count, double area, double* out, cudaStream_t st);
int launch_term_maps(const double* mu1, const double* mu2, const double* var1, const double* var2,
                     const double* cov, long long count, double c1, double c2, double* out, cudaStream_t st);
int launch_divide(const double* x, long long count, double divisor, double* out, cudaStream_t st);

// ---------------- K1s: strided Gaussian scores (stride >= 2, 8/16-bit, k <= 31) ----------------
bool gauss_stride_supported(int dtype, int k, int s);
int gauss_stride_twa(int k, int s, int es);  // anchor columns per strip
int launch_gauss_stride(const GaussArgs& a, dim3 grid, int k, cudaStream_t st);

// ---------------- K1g: Gaussian windows wider than 31 taps (fp64, generic K) ----------------
struct GaussGenericArgs {
  const unsigned char* ref;
  const unsigned char* dist;
  long long row_pitch_b, frame_pitch_b;  // bytes
  int dtype, esize;
  int n, h, w, k, stride;
  int ho, wo, gh, gw;
  int seg_rows;                // output rows per segment (gridDim.y segments)
  double scale;                // stored integer sample -> value (2^-scale_log2); 1 for f32
  double c1, c2;
  int want;
  double* partials;            // [n][gridDim.y][gridDim.x][3]
  void* maps;                  // [n][planes][gh][gw], float64 if map_f64 else float32
  int map_f64;
  long long map_plane, map_frame;
  double taps[255];            // normalised 1-D taps g/sum(g), built in fp64 from sigma
};
size_t gauss_generic_smem(int k);
int gauss_generic_grid(int ho, int wo, int n, int seg_rows, dim3* grid);
int launch_gauss_generic(const GaussGenericArgs& a, dim3 grid, cudaStream_t st);

// ---------------- K2: rect window ----------------
constexpr int BX_THREADS = 128;  // one input column per thread in the V pass

struct BoxArgs {
  const unsigned char* ref;
  const unsigned char* dist;
  long long row_pitch_b, frame_pitch_b;
  int dtype, esize;
  int n, h, w;
  int k, s, gh, gw;
  int na;                     // anchor columns per strip (integer kernel)
  int seg_anchors;            // anchor rows per segment (gridDim.y segments)
  int ch;                     // staged input rows per chunk (multiple of s)
  int in_pitch;               // staging row pitch, bytes
  int nslot;                  // prefix history slots
  double sscale1, sscale2;    // 2^-scale_log2, 2^-2*scale_log2 (exact rescaling of sums)
  float c1i, c2i;             // C * area^2 * 4^scale_log2: constants of the integer-domain score epilogue
  double c1d, c2d;
  int fast_ok;                // area^2 * stored_max^2 < 2^52: the integer-domain epilogue is exact in u64/f64
  int area_i;                 // k * k
  double area, inv_area;
  int area_pow2;              // area is a power of two: x/area == x*inv_area exactly
  double c1, c2;
  int want;
  double* partials;           // [n][gridDim.y][gridDim.x][3]
  double* partials2;          // optional, same layout, slot 0 = sum of q^2 (SSK_WANT_Q2)
  double* maps;               // float64 [n][planes][gh][gw]
  long long map_plane, map_frame;
  long long* wsums;           // optional int64 [n][5][gh][gw]
  const long long* mom;       // moment planes [5][h][mom_rp] (volume path), else null
  long long mom_rp, mom_plane;
};

size_t box_smem_bytes(const BoxArgs& a, bool wide);
int launch_box_int(const BoxArgs& a, dim3 grid, bool wide, cudaStream_t st);
int launch_box_moments(const BoxArgs& a, dim3 grid, cudaStream_t st);
int launch_volume_update(void* planes, int is_float, long long pp, long long prp, const void* nr, const void* nd,
                         const void* orf, const void* od, int dtype, long long srp, int h, int w, int mode,
                         cudaStream_t st);
int launch_volume_refresh(void* planes, long long pp, long long prp, const void* const* refs,
                          const void* const* dists, int count, int dtype, long long srp, int h, int w,
                          cudaStream_t st);
int launch_volume_direct(const BoxArgs& a, const double* planes, dim3 grid, dim3 block, cudaStream_t st);
int launch_box_float(const BoxArgs& a, dim3 grid, dim3 block, cudaStream_t st);
bool box_block_supported(int dtype, int k, int s, bool wide, double stored_max);
int launch_box_block(const BoxArgs& a, dim3 grid, cudaStream_t st);

// ---------------- pyramid + MS-SSIM finalize ----------------
struct PyramidArgs {
  const unsigned char* src_r;
  const unsigned char* src_d;
  long long src_rp, src_fp;                      // elements
  unsigned char* dst_r[GS_MAX_LEVELS];
  unsigned char* dst_d[GS_MAX_LEVELS];
  long long dst_rp[GS_MAX_LEVELS], dst_fp[GS_MAX_LEVELS];
  int hl[GS_MAX_LEVELS], wl[GS_MAX_LEVELS];       // dims of the produced levels 1..nl
};
int launch_pyramid(const PyramidArgs& p, int src_dtype, int dst_dtype, int nl, int n, cudaStream_t st);

constexpr int SSK_MAX_SCALES = 16;
struct FinalizeArgs {
  const double* partials[SSK_MAX_SCALES];
  int nparts[SSK_MAX_SCALES];
  double count[SSK_MAX_SCALES];
  double exps[SSK_MAX_SCALES];
  int levels, n;
  int aggregation;        // 0: level means only, 1: product, 2: sum
  double* level_means;    // [n][levels]
  double* scores;         // [n] or null
  double* ssim_sums;      // [n][3] or null: level-0 means of q, l, cs (sum / count, IEEE division)
};
int launch_msssim_finalize(const FinalizeArgs& a, cudaStream_t st);

// ---------------- helpers ----------------
int launch_reduce_partials(const double* partials, int nparts, int n, int ncomp, double divisor,
                           double* out, int out_stride, int out_offset, int comp_offset,
                           cudaStream_t st);
int launch_downsample(const unsigned char* src_r, const unsigned char* src_d, int src_dtype,
                      long long src_rp, long long src_fp, int n, int h, int w,
                      unsigned char* dst_r, unsigned char* dst_d, int dst_dtype, long long dst_rp,
                      long long dst_fp, cudaStream_t st);
int launch_integral(const unsigned char* ref, const unsigned char* dist, int dtype,
                    long long rp, long long fp, int n, int h, int w, void* out, cudaStream_t st);

}  // namespace ssk
