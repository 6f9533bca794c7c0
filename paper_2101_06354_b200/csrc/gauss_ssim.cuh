// K1: fused Gaussian-window local moments + SSIM terms + mean-pooling reduction.
//
// Replaces, for Gaussian windows, the reference's
//   _sliding_weighted_sums x5   (src/stats.py:155-164, called at :247-255)
//   stats_from_sums(area=1)     (src/stats.py:185-202)
//   term_maps_from_stats        (src/ssim.py:31-46)
//   mssim / pool_spatial("am")  (src/ssim.py:55-65, src/pooling.py:218-219)
// The 2-D kernel outer(g,g)/sum (src/stats.py:41-44) is applied separably
// with the normalised 1-D taps g/sum(g) (identical up to rounding;
// tests/test_stats.py:126-129 pins separability).
//
// Blackwell design.  One CTA = VC threads (256 for frames wide enough, else 128) = a strip
// of TW output columns (TW + K - 1 <= VC input columns) of a segment of output rows, for TWO
// frames at once: every value is carried as a packed fp32 pair (frame f, frame f+1), so the
// whole filter runs on FFMA2 / FMUL2 / FADD2 -- two FMAs per lane per issued instruction --
// without any register shuffling (the pairing is across frames, which share all addresses
// and weights).  The kernel is issue-bound (an FFMA2 holds the issue port for both of its
// cycles, tools/ubench/ffma2_forms.cu), so the design minimises instructions per output.
//   stage  : cp.async 16-B copies of G new input rows of the 4 images (ref/dist x 2 frames)
//            into a ring of raw rows, one chunk ahead of the compute, zero fill past the
//            edge; each thread's source pointer / ring slot run on from chunk to chunk.
//   V pass : thread = input column.  Score path (4 moments, sum / difference form): forms
//            a = x + y - 2c and b = x - y - d exactly (8/16-bit samples: inside the 2^23
//            integer -> float splice, one IADD3 and one FFMA2 each; c, d = the tile's rounded
//            means of (x + y) / 2 and x - y over its middle row, symmetric in ref / dist, which
//            keep E[a^2] - E[a]^2 and E[b^2] - E[b]^2 well conditioned in fp32), squares them
//            and gathers the K-tap vertical filter for G output rows (4*G packed accumulators;
//            taps in uniform registers).  Statistics maps (5 moments): x, y, x^2, y^2, xy.
//   H pass : thread = (output row, 8 adjacent columns); K-tap horizontal filter from the
//            shared-memory V rows (16-byte loads), then the SSIM epilogue on packed pairs
//            (sd_terms: 15 FMA-pipe ops and 4 reciprocals per output pair), optional map
//            stores and per-frame partial sums.
//   reduce : warp-shuffle + shared-memory block reduction into one fp64 partial per
//            (frame, CTA); a second tiny kernel folds the partials per frame in a fixed
//            order (bit-reproducible, batch-independent).
// Variants of the one body (gauss_body): the classic kernel (every thread runs V then H
// behind two CTA barriers per chunk; 2 x 256 or 4 x 128 threads per SM -- the default), the
// multi-level launch (tiles of several pyramid levels in one grid), and the warp-specialised
// kernels (producer warps V, consumer warps H over a ring of V tiles behind named barriers;
// persistent for wide u8 frames) kept as A/B alternatives (SSK_L0_CLASSIC=0, SSK_NARROW_WS=1).
// Every output value is produced by the same operation sequence whatever the
// stride, so strided grids equal dense[::s, ::s] bit-exactly
// (tests/test_stats.py:274-285).
#pragma once
#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "common.cuh"
#include "kernels.h"

namespace ssk {
namespace gk {

typedef unsigned long long u64;

__device__ __forceinline__ u64 pk(float lo, float hi) {
  u64 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ void upk(u64 v, float& lo, float& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ u64 fma2(u64 a, u64 b, u64 c) {
  u64 d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ u64 mul2(u64 a, u64 b) {
  u64 d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ u64 add2(u64 a, u64 b) {
  u64 d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ u64 sub2(u64 a, u64 b) {
  u64 d;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ float rcp_approx(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ u64 rcp2(u64 v) {
  float a, b;
  upk(v, a, b);
  return pk(rcp_approx(a), rcp_approx(b));
}
__device__ __forceinline__ u64 add_rn2(u64 a, u64 b) {  // two IEEE scalar adds, never contracted
  float a0, a1, b0, b1;
  upk(a, a0, a1);
  upk(b, b0, b1);
  return pk(__fadd_rn(a0, b0), __fadd_rn(a1, b1));
}
__device__ __forceinline__ u64 maxc_2(u64 v, float c) {
  float a, b;
  upk(v, a, b);
  return pk(fmaxf(a, c), fmaxf(b, c));
}
__device__ __forceinline__ u64 max0_2(u64 v) {
  float a, b;
  upk(v, a, b);
  return pk(fmaxf(a, 0.f), fmaxf(b, 0.f));
}

constexpr int G = GS_G;                       // output rows per chunk
#ifndef GS_NBUF
#define GS_NBUF 3                             // V tiles in flight in the warp-specialised kernel
#endif
int gauss_ws_level();                         // capi.cu: SSK_GAUSS_WS environment switch (default 1)
inline bool gauss_ws_enabled() { return gauss_ws_level() >= 1; }
#ifndef GS_MINB
#define GS_MINB (NM == 4 ? 4 : 3)  // 4 CTAs/SM measured faster than 3 with more registers
#endif
// V-row pitch in bytes for VC columns: pitch/8 odd -> a half warp's 8 rows x 2 column
// groups hit 16 distinct 8-byte bank slots
#ifndef SSK_H128
#define SSK_H128 1  // the H pass reads V values as 16-byte pairs (pitch 16 mod 128: conflict-free); 0 = 8-byte loads
#endif
__host__ __device__ constexpr int vp_of(int vc) { return SSK_H128 ? vc * 8 + 16 : vc * 8 + 8; }
__host__ __device__ constexpr int tw_of(int k, int vc) { return ((vc - (k - 1)) / 16) * 16; }
// Raw ring rows.  Warp-specialised kernels stage chunk c+1 while chunk c is read (2G + K - 1);
// the classic kernel refills the G oldest rows right after its V pass, so the G + K - 1 rows of
// a chunk suffice -- for 8-bit samples rounded up to whole groups of G rows (r2): a chunk then
// reads whole groups, each contiguous, so every row's address is one of a few per-chunk group
// bases plus an immediate (no per-row wrap select; 16-bit strips keep the exact ring, whose
// extra rows would cost them a CTA per SM).
#ifndef SSK_RING_GROUPS
#define SSK_RING_GROUPS 1
#endif
__host__ __device__ constexpr bool ring_grouped(bool ws, int es) { return SSK_RING_GROUPS && !ws && es == 1; }
__host__ __device__ constexpr int ring_rows(int k, bool ws, int es) {
  return ws ? 2 * GS_G + k - 1 : (ring_grouped(ws, es) ? (GS_G + k - 1 + GS_G - 1) / GS_G * GS_G : GS_G + k - 1);
}
// V tiles in flight: 3, except wide 16-bit strips (their doubled raw ring leaves room for 2)
__host__ __device__ constexpr int nbuf_of(int vc, int es) { return (vc == 256 && es > 1) ? 2 : GS_NBUF; }

// raw sample (as stored) -> float with the 2^23 splice for small integers
template <typename TIN>
__device__ __forceinline__ float raw_to_float(const unsigned char* p) {
  if constexpr (sizeof(TIN) == 1) {
    return __int_as_float(0x4B000000 | (unsigned)*p);
  } else if constexpr (sizeof(TIN) == 2) {
    return __int_as_float(0x4B000000 | (unsigned)*reinterpret_cast<const unsigned short*>(p));
  } else if constexpr (std::is_same<TIN, float>::value) {
    return *reinterpret_cast<const float*>(p);
  } else {
    return __uint2float_rn(*reinterpret_cast<const unsigned*>(p));
  }
}

template <typename TIN>
__device__ __forceinline__ unsigned raw_uint(const unsigned char* p) {  // 8/16-bit stored sample
  if constexpr (sizeof(TIN) == 1) return (unsigned)*p;
  else return (unsigned)*reinterpret_cast<const unsigned short*>(p);
}

// symmetric (ref <-> dist) a*a + b*b per lane: IEEE-rounded products and sum, never contracted
__device__ __forceinline__ u64 sumsq2(u64 x, u64 y) {
  float x0, x1, y0, y1;
  upk(x, x0, x1);
  upk(y, y0, y1);
  return pk(__fadd_rn(__fmul_rn(x0, x0), __fmul_rn(y0, y0)), __fadd_rn(__fmul_rn(x1, x1), __fmul_rn(y1, y1)));
}

// Sum / difference form of the 4-moment path (default).  The filters run on a = x' + y'
// and b = x - y and their squares: Sm = E[a], Dm = E[b], Var(a) = s1^2 + s2^2 + 2 s12,
// Var(b) = s1^2 + s2^2 - 2 s12, so
//   cs = (Var(a) - Var(b) + 2 C2) / (Var(a) + Var(b) + 2 C2),
//   l  = (Su^2 - Dm^2 + 2 C1) / (Su^2 + Dm^2 + 2 C1),  Su = Sm + 2 shift = mu1 + mu2.
// Swapping ref and dist negates b and Dm exactly and changes nothing else, so symmetry is
// exact without any exact-square condition; Var(b) -- the distortion's own variance -- is
// formed directly instead of through E[xy] - m1 m2, so 1 - cs of near-identical pairs loses
// no digits; and the epilogue needs 11 packed FMA-pipe ops per output pair instead of 15
// (one product op less per staged sample as well: integer samples form x + y and x - y
// inside the 2^23 splice on the ALU pipe).  SSK_SD=0 rebuilds the x / y form for A/B runs.
#ifndef SSK_SD
#define SSK_SD 1
#endif
#ifndef SSK_PROD_SYNC1
#define SSK_PROD_SYNC1 0  // 1 = one producer-internal barrier per chunk in the warp-specialised kernels (measured neutral)
#endif
#ifndef SSK_EPI_FAST
#define SSK_EPI_FAST 1  // branch-free epilogue block for interior items of score launches
#endif
constexpr unsigned long long SIGN2 = 0x8000000080000000ull;
constexpr unsigned SD_OFF = 1u << 16;  // keeps x - y + SD_OFF non-negative for 8/16-bit samples
__device__ __forceinline__ u64 neg2(u64 v) {  // folds into the consumer's operand-negate modifier
  float a, b;
  upk(v, a, b);
  return pk(-a, -b);
}
// SSIM terms of one output pair from the filtered sum / difference moments:
// Sm = E[a], Dm = E[b], Ea = E[a^2] + 2 C2, Eb = E[b^2] (a shifted by 2c, b by d, the tile's
// rounded means).  Symmetric in (ref, dist): swapping them negates Dm and dshift exactly, and
// both enter only through squares.  The variance clamp of stats_from_sums (src/stats.py:199-200) acts on
// the denominator, Var(a) + Var(b) + 2 C2 >= 2 C2.  FULL adds l (from the unshifted means:
// Su = mu1 + mu2 = Sm + 2 shift, 2 mu1 mu2 + C1 = (Su^2 - Dm^2) / 2 + C1 and
// mu1^2 + mu2^2 + C1 = (Su^2 + Dm^2) / 2 + C1, all terms >= 0) and q = l cs.
template <bool FULL>
__device__ __forceinline__ void sd_terms(const u64 Sm, const u64 Dm, const u64 Ea, const u64 Eb, const float c2x2,
                                         const u64 h2shift, const u64 dshift, const u64 twoc1_2, u64& cs, u64& l,
                                         u64& q) {
  const u64 va = fma2(neg2(Sm), Sm, Ea);  // Var(a) + 2 C2
  const u64 vb = fma2(neg2(Dm), Dm, Eb);  // Var(b) (b shifted by the tile's d: no cancellation)
  cs = mul2(add2(va, neg2(vb)), rcp2(maxc_2(add2(va, vb), c2x2)));
  q = cs;
  if constexpr (FULL) {
    const u64 Su = add2(Sm, h2shift);
    const u64 Dt = add2(Dm, dshift);  // mu1 - mu2
    const u64 H = fma2(Su, Su, twoc1_2);
    l = mul2(fma2(neg2(Dt), Dt, H), rcp2(fma2(Dt, Dt, H)));
    q = mul2(l, cs);
  }
}

// NM = 4 moments (x, y, x^2+y^2, xy) for the score/term path: sigma1^2 + sigma2^2
// only enters SSIM as a sum, so one filtered moment fewer (-20% filter FMAs);
// the variance clamp max(., 0) of stats_from_sums (src/stats.py:199-200) is then
// applied to the sum (differs from per-variance clamping only by fp32 rounding
// residue of flat windows).  NM = 5 (x, y, x^2, y^2, xy) serves the statistics
// maps of local_statistics.
// WS = warp-specialised variant: 8 warps per CTA, warps 0-3 run the V pass
// (producers) and warps 4-7 the H pass + epilogue (consumers) over a double-
// buffered V tile, synchronised by named barriers, so the two phases overlap
// instead of alternating behind CTA-wide barriers.
__device__ __forceinline__ void named_sync(int id, int count) {
  SSK_JITTER(2 * id);
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
  SSK_JITTER(2 * id + 1);
}
__device__ __forceinline__ void named_arrive(int id, int count) {
  SSK_JITTER(64 + id);
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(count) : "memory");
}

// MAPS = false compiles the map stores out (score-only kernels: smaller code, no dead branches)
// L1 = false compiles the fused pyramid-level-1 stores out (score-only persistent launches)
template <int K, typename TIN, int NM, bool WS, int VC, bool PERSIST = false, bool MAPS = true, bool L1 = true>
__device__ __forceinline__ void gauss_body(const GaussArgs& a, const int strip0, const int seg0, const int pair0,
                                           const int nstrips, const int nseg, const float (&taps)[32]) {
  constexpr int VP = vp_of(VC);
  constexpr int TW = tw_of(K, VC);
  constexpr int TWI = TW + K - 1;
  constexpr int ES = (int)sizeof(TIN);
  constexpr int RB = ((TWI * ES + 15) / 16) * 16;  // raw row bytes per image
  constexpr int NCH = RB / 16;
  // raw ring rows: the warp-specialised kernel stages chunk c+1 while chunk c is read
  // (2G + K - 1); the classic kernel refills the G oldest rows right after its V pass,
  // so the copy overlaps the H pass and the ring needs only the G + K - 1 rows of a chunk
  constexpr int RR = ring_rows(K, WS, ES);
  constexpr bool GROUPED = ring_grouped(WS, ES);
  constexpr int NH = (K + 1) / 2;
  constexpr int NP = 8 + K - 1;                     // V values read per H item
  static_assert(TWI <= VC, "strip wider than the CTA");

  constexpr int NT = WS ? 2 * VC : VC;  // threads per CTA
  extern __shared__ __align__(16) unsigned char smem[];
  unsigned char* raw = smem;                        // [RR][4][RB]
  unsigned char* vbuf0 = smem + RR * 4 * RB;        // [WS ? 2 : 1][NM][G][VP]
#ifndef SSK_TAPS_SMEM
#define SSK_TAPS_SMEM 0
#endif
#if SSK_TAPS_SMEM
  __shared__ float s_taps[32];
#endif
  __shared__ double s_red[(2 * VC / 32) * 6];

  // Warp-specialised kernels: logical thread ids swap the CTA's halves, so the producers
  // (logical 0 .. VC-1) are the hardware's upper warps.  The scheduler arbitrates eligible
  // warps highest-warp-id first: the stage that bounds the pipeline should win the issue slot
  // (measured: SSK_PROD_HI=1 is slower, 0.711 vs 0.698 ms -- the consumers keep the upper warps).
#ifndef SSK_PROD_HI
#define SSK_PROD_HI 0
#endif
  const int tid = (WS && SSK_PROD_HI) ? (int)(threadIdx.x ^ VC) : (int)threadIdx.x;
  // the tile (strip, segment, frame pair) being processed; a persistent CTA walks several
  int strip, seg, f0, f1, c0, y0, y1, in_end, nchunks, own_end, row_bytes_left;
  bool has1;
  long long fo0, fo1;  // staged images: 0 = ref f0, 1 = ref f1, 2 = dist f0, 3 = dist f1
  auto set_tile = [&](const int st, const int sg, const int pr) {
    strip = st;
    seg = sg;
    f0 = 2 * pr;
    has1 = f0 + 1 < a.n;
    f1 = has1 ? f0 + 1 : f0;
    c0 = st * TW;
    y0 = sg * a.seg_rows;
    y1 = min(y0 + a.seg_rows, a.ho);
    in_end = y1 + K - 1;
    nchunks = (y1 - y0 + G - 1) / G;
    own_end = sg == nseg - 1 ? a.h : y1;
    fo0 = (long long)f0 * a.frame_pitch_b;
    fo1 = (long long)f1 * a.frame_pitch_b;
    row_bytes_left = (a.w - c0) * ES;
  };
  const int npairs = (a.n + 1) / 2;
  const int ntiles = nstrips * nseg * npairs;
  auto tile_of = [&](const int t) { set_tile(t % nstrips, (t / nstrips) % nseg, t / (nstrips * nseg)); };
  if constexpr (PERSIST) tile_of(blockIdx.x);
  else set_tile(strip0, seg0, pair0);

  // staging (issued by the VC V-pass threads): a thread always copies the same 16-byte chunk
  // q of the same image im, of every RPP-th row, so per call the source base, the chunk's
  // validity and the ring offset are computed once and the loop is a pointer increment
  // and a ring-slot wrap (was a division / modulo chain per 16-byte item)
  constexpr int IPR = 4 * NCH;  // 16-byte items per input row (4 images)
  constexpr int RPP = VC / IPR;  // rows per pass (when IPR divides VC)
  // Running-pointer mode (r2): a tile's rows are staged strictly in order (its first G + K - 1
  // rows, then G more per chunk), so a thread's source pointer, row and ring slot simply run on
  // from call to call; the first call of a tile (r_lo == y0) derives them.  Per chunk that is
  // two copies and a handful of adds per thread -- the item loop spent ~90 instructions per
  // chunk and thread on 64-bit row-address IMADs and a modulo (7 % of the kernel's stall
  // samples sat on those IMADs, which share the FMA pipe with the filter).
#ifndef SSK_STAGE_RUNNING
#define SSK_STAGE_RUNNING 1
#endif
  const unsigned char* st_src = nullptr;
  int st_row = 0, st_slot = 0;
  auto stage_rows = [&](int r_lo, int r_hi) {
    r_hi = min(r_hi, in_end);
#ifdef SSK_STAGE_GENERIC
    constexpr bool generic_stage = true;  // A/B build: the item loop everywhere
    constexpr bool running_stage = false;
#else
    constexpr bool running_stage = SSK_STAGE_RUNNING && VC % IPR == 0;
    // (round-2 first pass, kept for SSK_STAGE_RUNNING=0: the per-call strength-reduced loop
    // won only in the score-only warp-specialised launch)
    constexpr bool generic_stage = !running_stage && (VC % IPR != 0 || !WS || L1);
#endif
    if constexpr (running_stage) {
      const int im = (tid % IPR) / NCH, q = tid % NCH;
      int valid = row_bytes_left - q * 16;
      valid = valid < 0 ? 0 : (valid > 16 ? 16 : valid);
      const long long pitch = a.row_pitch_b;
      if (r_lo == y0) {  // first rows of a tile (uniform branch)
        st_row = y0 + tid / IPR;
        st_slot = tid / IPR;
        st_src = ((im & 2) ? a.dist : a.ref) + ((im & 1) ? fo1 : fo0) + (valid ? (long long)c0 * ES + q * 16 : 0) +
                 (long long)st_row * pitch;
      }
      unsigned char* dst = raw + im * RB + q * 16;
      for (; st_row < r_hi; st_row += RPP) {
        cp_async16(dst + st_slot * 4 * RB, st_src, valid);
        st_src += RPP * pitch;
        st_slot += RPP;
        if (st_slot >= RR) st_slot -= RR;
      }
      cp_async_commit();
    } else if constexpr (generic_stage) {  // generic item loop
      const int total = (r_hi - r_lo) * IPR;
      for (int i = tid; i < total; i += VC) {
        const int rr = i / IPR;
        const int rem = i - rr * IPR;
        const int im = rem / NCH;
        const int q = rem - im * NCH;
        const int row = r_lo + rr;
        const int off = q * 16;
        int valid = row_bytes_left - off;
        valid = valid < 0 ? 0 : (valid > 16 ? 16 : valid);
        const unsigned char* rowp =
            ((im & 2) ? a.dist : a.ref) + ((im & 1) ? fo1 : fo0) + (long long)row * a.row_pitch_b;
        const unsigned char* src = valid ? rowp + (long long)c0 * ES + off : rowp;
        cp_async16(raw + (((row - y0) % RR) * 4 + im) * RB + off, src, valid);
      }
      cp_async_commit();
    } else {  // strength-reduced loop, re-derived per call
      const int im = (tid % IPR) / NCH, q = tid % NCH;
      int valid = row_bytes_left - q * 16;
      valid = valid < 0 ? 0 : (valid > 16 ? 16 : valid);
      const long long pitch = a.row_pitch_b;
      int row = r_lo + tid / IPR;
      const unsigned char* src = ((im & 2) ? a.dist : a.ref) + ((im & 1) ? fo1 : fo0) +
                                 (valid ? (long long)c0 * ES + q * 16 : 0) + (long long)row * pitch;
      unsigned char* dst = raw + im * RB + q * 16;
      int slot = (row - y0) % RR;
      for (; row < r_hi; row += RPP) {
        cp_async16(dst + slot * 4 * RB, src, valid);
        src += RPP * pitch;
        slot += RPP;
        if (slot >= RR) slot -= RR;
      }
      cp_async_commit();
    }
  };

  if (tid < VC) stage_rows(y0, y0 + G + K - 1);  // (persistent CTAs: their first tile)
#if SSK_TAPS_SMEM
  if (tid < 32) s_taps[tid] = a.taps[tid];
  __syncthreads();
  u64 w2[NH];
#pragma unroll
  for (int i = 0; i < NH; ++i) w2[i] = pk(s_taps[i], s_taps[i]);
#else
  // taps straight from the kernel arguments at a fixed offset (constant bank -> uniform
  // registers; the multi-level launch reads its first level's, every level has the same
  // window): through shared memory ptxas kept a third of them in vector registers, and an
  // FFMA2 with a register-broadcast weight issues at 2.42 cycles instead of 2.04 (tools/ubench)
  u64 w2[NH];
#pragma unroll
  for (int i = 0; i < NH; ++i) w2[i] = pk(taps[i], taps[i]);
#endif

  const u64 scale2 = pk(a.conv_scale, a.conv_scale);
  const u64 bias2 = pk(a.conv_bias, a.conv_bias);
  const u64 shift2 = pk(a.shift, a.shift);
  const u64 c1_2 = pk(a.c1, a.c1), c2_2 = pk(a.c2, a.c2);
  const u64 two2 = pk(2.f, 2.f), one2 = pk(a.one, a.one), half2 = pk(0.5f, 0.5f), mhalf2 = pk(-0.5f, -0.5f);
  const u64 twoshift2 = pk(2.f * a.shift, 2.f * a.shift);
  const u64 twoc1_2 = pk(2.f * a.c1, 2.f * a.c1), twoc2_2 = pk(2.f * a.c2, 2.f * a.c2);
  // Per-tile sample shift: instead of a fixed L/2, every tile shifts its samples by
  // c = round(mean of (x + y) / 2) over its middle input row, per frame -- symmetric in
  // ref / dist, exactly representable (an integer in stored units), and close to the local
  // level, so E[x'^2] - m^2 cancels far less in near-flat windows away from mid-gray.
  // 8/16-bit samples sum in u32; u32 pyramid levels (up to 2^24 per sample) and float
  // samples sum in fp64 (fixed shuffle order: bit-identical wherever it is recomputed).
  // vbias / hshift / h2shift carry the tile's shift into the V pass and the epilogue.
  constexpr bool TSHIFT = true;
  using TSum = typename std::conditional<ES == 4, double, unsigned>::type;
  using TDif = typename std::conditional<ES == 4, double, int>::type;  // signed sums of (x - y)
  __shared__ TSum s_tsum[2 * VC / 32][2];
  __shared__ TDif s_dsum[2 * VC / 32][2];
  u64 vbias = bias2, hshift = shift2, h2shift = twoshift2;
  // sum / difference form, integer samples: a = fma(splice(x + y), sc, abias) = (x + y) sc - 2c
  // and b = fma(splice(x - y + SD_OFF), sc, bbias) = (x - y) sc - d, both exact.  d is the
  // tile's rounded mean of x - y (rounded half away from zero, so swapping ref and dist
  // negates it exactly): Var(b) = E[b^2] - E[b]^2 then does not cancel when ref and dist
  // differ by a large offset (flat 0 vs flat 255: 6.7e-5 off in cs without it).  dshift adds
  // d back to E[b] for the luminance term.
  u64 abias = pk(2.f * a.conv_bias + 8388608.f * a.conv_scale, 2.f * a.conv_bias + 8388608.f * a.conv_scale);
  u64 bbias = pk(-(8388608.f + (float)SD_OFF) * a.conv_scale, -(8388608.f + (float)SD_OFF) * a.conv_scale);
  u64 dshift = 0ull;
  auto set_shift = [&](const TSum t0, const TSum t1, const TDif u0, const TDif u1) {  // sums over n columns
    const unsigned n = (unsigned)max(1, min(TWI, a.w - c0));
    const float sc = a.conv_scale;                        // 2^-scale_log2 (exact); 1 for floats
    if constexpr (ES == 4) {
      const float cv0 = (float)floor(t0 / (2.0 * n) + 0.5) * sc;  // integer (stored units): exact
      const float cv1 = (float)floor(t1 / (2.0 * n) + 0.5) * sc;
      const float dv0 = (float)copysign(floor(fabs(u0) / n + 0.5), u0) * sc;
      const float dv1 = (float)copysign(floor(fabs(u1) / n + 0.5), u1) * sc;
      vbias = pk(-cv0, -cv1);                             // x' = fma(x, sc, -c), one rounding
      hshift = pk(cv0, cv1);
      h2shift = pk(2.f * cv0, 2.f * cv1);
      dshift = pk(dv0, dv1);
    } else {
      const float cv0 = (float)((t0 + n) / (2u * n)) * sc;  // value units, exact
      const float cv1 = (float)((t1 + n) / (2u * n)) * sc;
      const int d0 = (int)(((unsigned)abs(u0) + n / 2u) / n), d1 = (int)(((unsigned)abs(u1) + n / 2u) / n);
      const float dv0 = (float)(u0 < 0 ? -d0 : d0) * sc, dv1 = (float)(u1 < 0 ? -d1 : d1) * sc;
      const float base = -8388608.f * sc;                   // the 2^23 splice, in value units
      const float baseb = -(8388608.f + (float)SD_OFF) * sc;
      vbias = pk(base - cv0, base - cv1);                   // exact: (2^23 + c_stored) * 2^-k
      abias = pk(base - 2.f * cv0, base - 2.f * cv1);       // exact: (2^23 + 2 c_stored) * 2^-k
      bbias = pk(baseb - dv0, baseb - dv1);                 // exact: (2^23 + SD_OFF + d_stored) * 2^-k
      hshift = pk(cv0, cv1);
      h2shift = pk(2.f * cv0, 2.f * cv1);
      dshift = pk(dv0, dv1);
    }
  };
  auto stored = [](const unsigned char* p) -> TSum {  // one stored sample, as summed
    if constexpr (ES == 1) return (unsigned)*p;
    else if constexpr (ES == 2) return (unsigned)*reinterpret_cast<const unsigned short*>(p);
    else if constexpr (std::is_same<TIN, float>::value) return (double)*reinterpret_cast<const float*>(p);
    else return (double)*reinterpret_cast<const unsigned*>(p);
  };
  auto warp_total = [](auto v) {
    if constexpr (ES == 4) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      return v;
    } else {
      return __reduce_add_sync(0xffffffffu, v);
    }
  };
  auto tile_shift = [&](const int gt, const int gs, const int wbase, auto&& gsync) {
    const int r = min(y0 + (y1 - y0) / 2 + K / 2, a.h - 1);
    TSum v0 = 0, v1 = 0;
    TDif w0 = 0, w1 = 0;
    for (int i = gt; i < TWI && c0 + i < a.w; i += gs) {
      const long long off = (long long)r * a.row_pitch_b + (long long)(c0 + i) * ES;
      const TSum xr0 = stored(a.ref + fo0 + off), yd0 = stored(a.dist + fo0 + off);
      const TSum xr1 = stored(a.ref + fo1 + off), yd1 = stored(a.dist + fo1 + off);
      v0 += xr0 + yd0;
      v1 += xr1 + yd1;
      w0 += (TDif)xr0 - (TDif)yd0;
      w1 += (TDif)xr1 - (TDif)yd1;
    }
    v0 = warp_total(v0);
    v1 = warp_total(v1);
    w0 = warp_total(w0);
    w1 = warp_total(w1);
    if ((gt & 31) == 0) {
      s_tsum[wbase + (gt >> 5)][0] = v0;
      s_tsum[wbase + (gt >> 5)][1] = v1;
      s_dsum[wbase + (gt >> 5)][0] = w0;
      s_dsum[wbase + (gt >> 5)][1] = w1;
    }
    gsync();
    TSum t0 = 0, t1 = 0;
    TDif u0 = 0, u1 = 0;
    for (int wi = 0; wi < gs / 32; ++wi) {
      t0 += s_tsum[wbase + wi][0];
      t1 += s_tsum[wbase + wi][1];
      u0 += s_dsum[wbase + wi][0];
      u1 += s_dsum[wbase + wi][1];
    }
    gsync();  // the scratch is rewritten by the next tile
    set_shift(t0, t1, u0, u1);
  };
  // Per-chunk variant for the classic kernel's map launches (same threads run the V and H
  // passes of a chunk, so nothing is handed over): the shift follows the chunk's own rows,
  // e.g. both sides of a letterbox edge inside a tile.  Reads the staged middle row.
  auto chunk_shift_smem = [&](const int c) {
    const int row = min(y0 + c * G + (G + K - 1) / 2, in_end - 1);
    const unsigned char* rp = raw + (((row - y0) % RR) * 4) * RB + tid * ES;
    TSum v0 = 0, v1 = 0;
    TDif w0 = 0, w1 = 0;
    if (tid < TWI && c0 + tid < a.w) {
      const TSum xr0 = stored(rp), yd0 = stored(rp + 2 * RB), xr1 = stored(rp + RB), yd1 = stored(rp + 3 * RB);
      v0 = xr0 + yd0;
      v1 = xr1 + yd1;
      w0 = (TDif)xr0 - (TDif)yd0;
      w1 = (TDif)xr1 - (TDif)yd1;
    }
    v0 = warp_total(v0);
    v1 = warp_total(v1);
    w0 = warp_total(w0);
    w1 = warp_total(w1);
    if ((tid & 31) == 0) {
      s_tsum[tid >> 5][0] = v0;
      s_tsum[tid >> 5][1] = v1;
      s_dsum[tid >> 5][0] = w0;
      s_dsum[tid >> 5][1] = w1;
    }
    __syncthreads();
    TSum t0 = 0, t1 = 0;
    TDif u0 = 0, u1 = 0;
    for (int wi = 0; wi < NT / 32; ++wi) {
      t0 += s_tsum[wi][0];
      t1 += s_tsum[wi][1];
      u0 += s_dsum[wi][0];
      u1 += s_dsum[wi][1];
    }
    __syncthreads();
    set_shift(t0, t1, u0, u1);
  };
  const bool full_terms = (a.want & (SSK_WANT_Q | SSK_WANT_L)) != 0;
  const bool want_maps = MAPS && (a.want & (SSK_MAP_TERMS | SSK_MAP_STATS)) != 0;
  const int s = a.stride;
  const int wo = a.wo;
  const bool exact_sq = a.exact_sq != 0;

  // per-thread running sums of q, l, cs over the tile (<= 128 outputs per thread), packed
  // fp32 pairs (frame f0, f1); widened to fp64 once per tile for the block reduction
  u64 fq = 0ull, fl = 0ull, fc = 0ull;
  auto tile_sums = [&](double* v) {
    float lo, hi;
    upk(fq, lo, hi);
    v[0] = lo;
    v[3] = hi;
    upk(fl, lo, hi);
    v[1] = lo;
    v[4] = hi;
    upk(fc, lo, hi);
    v[2] = lo;
    v[5] = hi;
  };
  const int htid = WS ? tid - VC : tid;
  const int hg = htid % G, hj = htid / G;  // H item: output row hg of the chunk, columns 8*hj..8*hj+7

  // ---------------- V pass: thread = input column ----------------
  auto vpass = [&](const int c, unsigned char* vbuf) {
    SSK_JITTER(100);
    if (tid < TWI && c0 + tid < a.w) {
      u64 acc[NM][G];
#pragma unroll
      for (int m = 0; m < NM; ++m)
#pragma unroll
        for (int r = 0; r < G; ++r) acc[m][r] = 0ull;
      // ring rows s0, s0+1, ... : one base before the wrap point, one after, so each row's
      // address is a select plus an immediate offset
      const int s0 = (c * G) % RR;
      const int wrap = RR - s0;
      const unsigned char* pa = raw + s0 * 4 * RB + tid * ES;
      const unsigned char* pb = pa - RR * 4 * RB;
      // grouped ring: the chunk's rows are groups g0, g0 + 1, ... (mod NG) of G rows each
      constexpr int NG = RR / G;
      const unsigned char* pg[GROUPED ? NG : 1];
      if constexpr (GROUPED) {
        const int g0 = c % NG;
#pragma unroll
        for (int k = 0; k < NG; ++k) {
          const int gk = g0 + k < NG ? g0 + k : g0 + k - NG;
          pg[k] = raw + gk * G * 4 * RB + tid * ES;
        }
      }
#pragma unroll
      for (int u = 0; u < G + K - 1; ++u) {
        const unsigned char* rp;
        if constexpr (GROUPED) rp = pg[u / G] + (u % G) * 4 * RB;
        else rp = (u < wrap ? pa : pb) + u * 4 * RB;
        u64 P[NM];
        if constexpr (NM == 4 && SSK_SD && ES <= 2) {
          // x + y and x - y inside the 2^23 splice (one IADD3 each), then one exact FFMA2 each
          const unsigned x0 = raw_uint<TIN>(rp), x1 = raw_uint<TIN>(rp + RB);
          const unsigned y0 = raw_uint<TIN>(rp + 2 * RB), y1 = raw_uint<TIN>(rp + 3 * RB);
          P[0] = fma2(pk(__uint_as_float(0x4B000000u + x0 + y0), __uint_as_float(0x4B000000u + x1 + y1)),
                      scale2, abias);
          P[1] = fma2(pk(__uint_as_float((0x4B000000u + SD_OFF) + x0 - y0),
                         __uint_as_float((0x4B000000u + SD_OFF) + x1 - y1)),
                      scale2, bbias);
          P[2] = mul2(P[0], P[0]);
          P[3] = mul2(P[1], P[1]);
        } else {
          const u64 X = fma2(pk(raw_to_float<TIN>(rp), raw_to_float<TIN>(rp + RB)), scale2, vbias);
          const u64 Y = fma2(pk(raw_to_float<TIN>(rp + 2 * RB), raw_to_float<TIN>(rp + 3 * RB)), scale2, vbias);
          P[0] = X;
          P[1] = Y;
          if constexpr (NM == 4 && SSK_SD) {  // float / u32 samples: rounded sum, exact antisymmetric difference
            P[0] = add2(X, Y);
            P[1] = add2(add2(X, neg2(Y)), neg2(dshift));
            P[2] = mul2(P[0], P[0]);
            P[3] = mul2(P[1], P[1]);
          } else if constexpr (NM == 4) {
            // x'^2 and y'^2 are exact in fp32 for 8-bit samples (|x'| <= 128) and for the
            // first two pyramid levels of 8-bit input (quarter / sixteenth steps), so the
            // contracted x'^2 + y'^2 is still exactly symmetric there; otherwise IEEE scalar ops
            if constexpr (sizeof(TIN) == 1) P[2] = fma2(X, X, mul2(Y, Y));
            else if (exact_sq) P[2] = fma2(X, X, mul2(Y, Y));
            else P[2] = sumsq2(X, Y);
            P[3] = mul2(X, Y);
          } else {
            P[2] = mul2(X, X);
            P[3] = mul2(Y, Y);
            P[NM - 1] = mul2(X, Y);
          }
        }
#pragma unroll
        for (int r = 0; r < G; ++r) {
          const int i = u - r;
          if (i >= 0 && i < K) {
            const u64 wi = w2[i < K - 1 - i ? i : K - 1 - i];
#pragma unroll
            for (int m = 0; m < NM; ++m) acc[m][r] = fma2(wi, P[m], acc[m][r]);
          }
        }
      }
#pragma unroll
      for (int m = 0; m < NM; ++m)
#pragma unroll
        for (int r = 0; r < G; ++r)
          *reinterpret_cast<u64*>(vbuf + (m * G + r) * VP + tid * 8) = acc[m][r];
    }
  };

  // ---------------- fused pyramid level 1 (producers, wide u8 kernel) ----------------
  // Each CTA owns input rows [y0, own_end) (the last segment also the K-1 tail rows)
  // and columns [c0, c0 + TW) (the last strip up to w); at chunk c it turns the
  // staged rows [y0 + cG, y0 + (c+1)G) -- all remaining owned rows at the last
  // chunk -- into 2x2 block sums, exactly what pyramid_kernel writes for level 1.
  auto level1 = [&](const int c) {
    const bool last_strip = strip == nstrips - 1;
    const int rlo = y0 + c * G;
    const int rhi = (c == nchunks - 1) ? own_end : min(rlo + G, own_end);
    const int yb = rlo >> 1, ye = min(rhi >> 1, a.l1_h);
    const int xb = c0 >> 1, xe = min((last_strip ? a.w : c0 + TW) >> 1, a.l1_w);
    const int nx = xe - xb, ny = ye - yb;
    if (nx <= 0 || ny <= 0) return;
    static_assert(RR % 2 == 0 && (TW + K - 1) / 2 <= 128, "level-1 item mapping");
#ifndef SSK_L1_WIDE
#define SSK_L1_WIDE 1
#endif
#if SSK_L1_WIDE
    // 8 level-1 samples per item and image (r2): two 16-byte shared loads (rows 2y, 2y+1),
    // byte-pair sums on packed 16-bit lanes, one 16-byte store (xb is a multiple of 8).
    // Item = (level-1 row, octet of columns, side): thread t < 128 owns row t / 32 (+ 4 per
    // pass), octet t % 16 and the side (ref / dist) of its half-warp, both frames -- a chunk's
    // four level-1 rows are one pass of warps 0-3 at half the instructions per sample of the
    // 4-sample items (35 -> ~20 us per 32-pair launch); warps 4-7 go straight to the V pass.
    // RR is even, so row 2y+1 sits in slot s0 + 1.
    const int no = (nx + 7) >> 3;
    const int oct = tid & 15, side = (tid >> 4) & 1;
    for (int r = tid >> 5; r < ny && oct < no && tid < 128; r += 4) {
      const int yy = yb + r, x8 = xb + 8 * oct;
      const int col = 2 * x8 - c0;
      const int s0 = (2 * yy - y0) % RR, s1 = s0 + 1;
      const int nvalid = min(8, xe - x8);
#pragma unroll
      for (int fi = 0; fi < 2; ++fi) {
        const int im = 2 * side + fi;
        if (fi && !has1) continue;
        const uint4 a0 = *reinterpret_cast<const uint4*>(raw + (s0 * 4 + im) * RB + col);
        const uint4 a1 = *reinterpret_cast<const uint4*>(raw + (s1 * 4 + im) * RB + col);
        // [b0 b1 b2 b3] -> 16-bit lanes (b0 + b1, b2 + b3); four bytes add without carry
        auto quad = [](unsigned u, unsigned v) {
          return (u & 0x00FF00FFu) + ((u >> 8) & 0x00FF00FFu) + (v & 0x00FF00FFu) + ((v >> 8) & 0x00FF00FFu);
        };
        const uint4 o = make_uint4(quad(a0.x, a1.x), quad(a0.y, a1.y), quad(a0.z, a1.z), quad(a0.w, a1.w));
        unsigned short* dst = (side ? a.l1_dist : a.l1_ref) + (long long)(fi ? f1 : f0) * a.l1_fp +
                              (long long)yy * a.l1_rp + x8;
        if (nvalid == 8) {
          *reinterpret_cast<uint4*>(dst) = o;
        } else {
          const unsigned w4[4] = {o.x, o.y, o.z, o.w};
          for (int j = 0; j < nvalid; ++j) dst[j] = (unsigned short)(w4[j >> 1] >> (16 * (j & 1)));
        }
      }
    }
#else
    // 4 level-1 samples per item: two 8-byte shared loads per image (rows 2y, 2y+1),
    // pairwise byte sums on packed 16-bit lanes, one 8-byte store (xb is a multiple of 4).
    // Item (row, quad) = (tid / 32 + k * VC / 32, tid % 32): at most 32 quads per row
    // (nx <= (TW + K - 1) / 2), so no division; RR is even, so row 2y+1 sits in slot s0 + 1.
    const int nq = (nx + 3) >> 2;
    const int q = tid & 31;
    for (int r = tid >> 5; r < ny && q < nq; r += VC >> 5) {
      const int yy = yb + r, x4 = xb + 4 * q;
      const int col = 2 * x4 - c0;
      const int s0 = (2 * yy - y0) % RR, s1 = s0 + 1;
      const int nvalid = min(4, xe - x4);
#pragma unroll
      for (int im = 0; im < 4; ++im) {
        if ((im & 1) && !has1) continue;
        const uint2 a0 = *reinterpret_cast<const uint2*>(raw + (s0 * 4 + im) * RB + col);
        const uint2 a1 = *reinterpret_cast<const uint2*>(raw + (s1 * 4 + im) * RB + col);
        // [b0 b1 b2 b3] -> 16-bit lanes (b0 + b1, b2 + b3); four rows-bytes add without carry
        const unsigned lo = (a0.x & 0x00FF00FFu) + ((a0.x >> 8) & 0x00FF00FFu) + (a1.x & 0x00FF00FFu) +
                            ((a1.x >> 8) & 0x00FF00FFu);
        const unsigned hi = (a0.y & 0x00FF00FFu) + ((a0.y >> 8) & 0x00FF00FFu) + (a1.y & 0x00FF00FFu) +
                            ((a1.y >> 8) & 0x00FF00FFu);
        unsigned short* dst = ((im & 2) ? a.l1_dist : a.l1_ref) + (long long)((im & 1) ? f1 : f0) * a.l1_fp +
                              (long long)yy * a.l1_rp + x4;
        if (nvalid == 4) {
          *reinterpret_cast<uint2*>(dst) = make_uint2(lo, hi);
        } else {
          const unsigned short v4[4] = {(unsigned short)(lo & 0xFFFF), (unsigned short)(lo >> 16),
                                        (unsigned short)(hi & 0xFFFF), (unsigned short)(hi >> 16)};
          for (int j = 0; j < nvalid; ++j) dst[j] = v4[j];
        }
      }
    }
#endif
  };

  // ---------------- H pass + epilogue: thread = (row, 8 columns) ----------------
  // K-tap horizontal filter of moment m for this thread's 8 outputs (V row hg, columns 8 hj ..)
  auto hfilter = [&](const unsigned char* vbuf, const int m, const u64 init, u64* acc8) {
#pragma unroll
    for (int jj = 0; jj < 8; ++jj) acc8[jj] = init;
#if SSK_H128
    static_assert(NP % 2 == 0, "pairs of V values");
    const ulonglong2* vr = reinterpret_cast<const ulonglong2*>(vbuf + (m * G + hg) * VP + hj * 64);
#pragma unroll
    for (int p2 = 0; p2 < NP / 2; ++p2) {
      const ulonglong2 vv = vr[p2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int p = 2 * p2 + h;
        const u64 v = h ? vv.y : vv.x;
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) {
          const int i = p - jj;
          if (i >= 0 && i < K) acc8[jj] = fma2(w2[i < K - 1 - i ? i : K - 1 - i], v, acc8[jj]);
        }
      }
    }
#else
    const u64* vr = reinterpret_cast<const u64*>(vbuf + (m * G + hg) * VP + hj * 64);
#pragma unroll
    for (int p = 0; p < NP; ++p) {
      const u64 v = vr[p];
#pragma unroll
      for (int jj = 0; jj < 8; ++jj) {
        const int i = p - jj;
        if (i >= 0 && i < K) acc8[jj] = fma2(w2[i < K - 1 - i ? i : K - 1 - i], v, acc8[jj]);
      }
    }
#endif
  };
  auto hpass = [&](const int c, const unsigned char* vbuf) {
    SSK_JITTER(101);
    const int orow = y0 + c * G + hg;
    const int ocol0 = c0 + 8 * hj;
    if (8 * hj < TW && ocol0 < wo && orow < y1 && (s == 1 || orow % s == 0)) {
      // columns of this item inside the anchor grid (all 8 for interior items at stride 1)
      const int ncol = min(8, wo - ocol0);
      u64 acc[NM][8];
#pragma unroll
      for (int m = 0; m < NM; ++m) {
        // NM = 4: the squared-sum moment starts at 2 C2 (C2 in the x / y form), so the filter
        // itself carries the constant (one add per output less)
        hfilter(vbuf, m, (NM == 4 && m == 2) ? (SSK_SD ? twoc2_2 : c2_2) : 0ull, acc[m]);
      }
      if constexpr (NM == 4 && SSK_SD && SSK_EPI_FAST) {
        // Interior items of score launches (no maps, stride 1, all 8 columns inside): one
        // branch-free block, so the eight outputs' dependent chains (FFMA2 -> MUFU -> FMUL2)
        // interleave instead of running one after another behind per-output branches.
        // (Measured: fusing the filters into the same block, each epilogue piece right after
        // the moment that completes it, is slower: 0.896 vs 0.885 ms per step.)
        if (!want_maps && s == 1 && ncol == 8) {
          const float c2x2 = 2.f * a.c2;
          u64 sq = fq, sl = fl, scs = fc;
          if (full_terms) {
#pragma unroll
            for (int jj = 0; jj < 8; ++jj) {
              u64 cs, l, q;
              sd_terms<true>(acc[0][jj], acc[1][jj], acc[2][jj], acc[3][jj], c2x2, h2shift, dshift, twoc1_2, cs, l, q);
              sq = fma2(q, one2, sq);
              sl = fma2(l, one2, sl);
              scs = fma2(cs, one2, scs);
            }
          } else {
#pragma unroll
            for (int jj = 0; jj < 8; ++jj) {
              u64 cs, l, q;
              sd_terms<false>(acc[0][jj], acc[1][jj], acc[2][jj], acc[3][jj], c2x2, h2shift, dshift, twoc1_2, cs, l, q);
              scs = fma2(cs, one2, scs);
            }
          }
          fq = sq;
          fl = sl;
          fc = scs;
          return;
        }
      }
      u64 sq = fq, sl = fl, scs = fc;
#pragma unroll
      for (int jj = 0; jj < 8; ++jj) {
        const u64 m1 = acc[0][jj], m2 = acc[1][jj];
        u64 v1, v2 = 0ull, cv = 0ull, cs, l = 0ull, q, mu1 = 0ull, mu2 = 0ull;
        if constexpr (NM == 4 && SSK_SD) {
          if (full_terms) sd_terms<true>(m1, m2, acc[2][jj], acc[3][jj], 2.f * a.c2, h2shift, dshift, twoc1_2, cs, l, q);
          else sd_terms<false>(m1, m2, acc[2][jj], acc[3][jj], 2.f * a.c2, h2shift, dshift, twoc1_2, cs, l, q);
          v1 = 0ull;
        } else {
        // Everything below is symmetric in (ref, dist): it uses only Sm = m1 + m2,
        // Dq = (m1 - m2)^2 and the exact product inside fma(m1, -m2, E[xy]).
        // exact negation by flipping the sign bits (ALU pipe, not an FMA-pipe subtract)
        const u64 nm2 = m2 ^ SIGN2;
        const u64 Sm = add2(m1, m2);
        const u64 Dm = add2(m1, nm2);  // m1 - m2 (antisymmetric; its square is symmetric)
        const u64 Dq = mul2(Dm, Dm);
        u64 den2;
        if constexpr (NM == 4) {
          // sigma1^2 + sigma2^2 = E[x^2 + y^2] - (m1^2 + m2^2), clamped as a sum, with
          // 2 (m1^2 + m2^2) = Sm^2 + Dq (no cancellation) and C2 carried by the filter:
          // den2 = max(E[x^2 + y^2] + C2 - (Sm^2 + Dq) / 2, C2)
          v1 = maxc_2(fma2(fma2(Sm, Sm, Dq), mhalf2, acc[2][jj]), a.c2);
          cv = fma2(m1, nm2, acc[3][jj]);  // cov = E[xy] - m1 m2, one rounding
          den2 = v1;
        } else {
          v1 = max0_2(sub2(acc[2][jj], mul2(m1, m1)));
          v2 = max0_2(sub2(acc[3][jj], mul2(m2, m2)));
          cv = fma2(m1, nm2, acc[NM - 1][jj]);
          den2 = add2(add2(v1, v2), c2_2);
        }
        const u64 num2 = fma2(two2, cv, c2_2);
        cs = mul2(num2, rcp2(den2));
        q = cs;
        if (full_terms) {
          // l from the unshifted means mu = m + s: with Su = mu1 + mu2 = Sm + 2s,
          // 2 mu1 mu2 + C1 = (Su^2 - Dq) / 2 + C1 and mu1^2 + mu2^2 + C1 = (Su^2 + Dq) / 2 + C1
          // (all terms >= 0: no cancellation).  The shifted form 2 Pm + 2 s Sm + 2 s^2 + C1
          // cancelled catastrophically in dark windows (m ~ -s): 3e-4 off in l at mu ~ 1.
          const u64 Su = add2(Sm, h2shift);
          const u64 H = fma2(mul2(Su, Su), half2, c1_2);
          const u64 num1 = fma2(Dq, mhalf2, H);
          const u64 den1 = fma2(Dq, half2, H);
          l = mul2(num1, rcp2(den1));
          q = mul2(l, cs);
        }
        }
        if (want_maps) {
          mu1 = add2(m1, hshift);
          mu2 = add2(m2, hshift);
        }
        const int col = ocol0 + jj;
        const bool valid = jj < ncol && (s == 1 || col % s == 0);
        if (valid) {
          // sums as explicit FFMA2 x*1 + acc: ptxas contracts a mul.f32x2 feeding an
          // add.f32x2 even with .rn, which would make a term's rounding depend on
          // whether it is also used elsewhere (i.e. on the requested outputs)
          if (full_terms) {
            sq = fma2(q, one2, sq);
            sl = fma2(l, one2, sl);
          }
          scs = fma2(cs, one2, scs);
          if (want_maps) {
            const long long idx = (long long)(orow / s) * a.gw + (col / s);
            float lo, hi;
            float* mp0 = reinterpret_cast<float*>(a.maps) + (long long)f0 * a.map_frame + idx;
            float* mp1 = reinterpret_cast<float*>(a.maps) + (long long)f1 * a.map_frame + idx;
            const bool terms = (a.want & SSK_MAP_TERMS) != 0;
            const u64 vals[5] = {terms ? l : mu1, terms ? cs : mu2, terms ? q : v1, v2, cv};
            const int nplanes = terms ? 3 : 5;
#pragma unroll
            for (int pl = 0; pl < 5; ++pl) {
              if (pl < nplanes) {
                upk(vals[pl], lo, hi);
                mp0[pl * a.map_plane] = lo;
                if (has1) mp1[pl * a.map_plane] = hi;
              }
            }
          }
        }
      }
      fq = sq;
      fl = sl;
      fc = scs;
    }
  };

  if constexpr (TSHIFT && (!WS || !PERSIST)) {  // one tile per CTA: the whole block computes it
    tile_shift(tid, NT, 0, [&] { __syncthreads(); });
  }
  if constexpr (!WS) {
    for (int c = 0; c < nchunks; ++c) {
      cp_async_wait<0>();
      __syncthreads();  // chunk c's rows landed; the previous H pass is done with the V tile
      if constexpr (TSHIFT) {
        if (want_maps) chunk_shift_smem(c);  // uniform branch
      }
      if constexpr (VC == 256 && ES == 1 && L1 && !MAPS) {
        // fused pyramid level 1 (wide u8 score launches): the chunk's G oldest rows are
        // turned into 2x2 sums before the refill below overwrites them
        if (a.l1_ref) level1(c);
      }
      vpass(c, vbuf0);
      __syncthreads();  // V tile complete; the chunk's G oldest raw rows are free
      if (c + 1 < nchunks) stage_rows(y0 + (c + 1) * G + K - 1, y0 + (c + 2) * G + K - 1);
      hpass(c, vbuf0);
    }
  } else {
    constexpr int VBYTES = NM * G * VP;
    constexpr int NB = nbuf_of(VC, ES);
    // NB V tiles in flight; named barriers 2..2+NB-1 = "tile b full",
    // 2+NBUF.. = "tile b free"; barrier 1 = producer-internal
    if constexpr (PERSIST) {
      // Persistent CTA (one per SM): tiles blockIdx.x, + gridDim.x, ...; the V-tile ring and
      // its barriers run on across tile boundaries, so the producers stage and filter the
      // next tile while the consumers drain the previous one (no per-tile fill / drain).
      int total = 0;  // chunks this CTA will run (matches the consumers' "free" arrivals)
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int sg = (t / nstrips) % nseg;
        total += (min((sg + 1) * a.seg_rows, a.ho) - sg * a.seg_rows + G - 1) / G;
      }
      int b = 0, cc = 0;
      if (tid < VC) {  // producers
        for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
          // each warpgroup pair derives the tile's shift itself from the same samples
          // (integer sums: bit-identical in both), so no producer -> consumer hand-off
          if (t != (int)blockIdx.x) tile_of(t);
          if constexpr (TSHIFT) tile_shift(tid, VC, 0, [&] { named_sync(1, VC); });
          if (t != (int)blockIdx.x) {
            stage_rows(y0, y0 + G + K - 1);  // the previous tile's raw rows are no longer read
          }
          for (int c = 0; c < nchunks; ++c, ++cc) {
#if SSK_PROD_SYNC1
            // ONE producer barrier per chunk: chunk c's rows (copies issued a chunk ago) have
            // landed everywhere, and every producer is done with chunk c-1's V pass, so the
            // ring slots of its G oldest rows may be refilled with chunk c+1's new rows now
            cp_async_wait<0>();
            named_sync(1, VC);
            if (c + 1 < nchunks) stage_rows(y0 + (c + 1) * G + K - 1, y0 + (c + 2) * G + K - 1);
#else
            if (c + 1 < nchunks) {
              stage_rows(y0 + (c + 1) * G + K - 1, y0 + (c + 2) * G + K - 1);
              cp_async_wait<1>();
            } else {
              cp_async_wait<0>();
            }
            named_sync(1, VC);
#endif
            if constexpr (VC == 256 && ES == 1) {
              if constexpr (L1) {
                if (a.l1_ref) level1(c);
              }
            }
            if (cc >= NB) named_sync(2 + NB + b, 2 * VC);
            vpass(c, vbuf0 + b * VBYTES);
            named_arrive(2 + b, 2 * VC);
#if !SSK_PROD_SYNC1
            named_sync(1, VC);
#endif
            b = b + 1 == NB ? 0 : b + 1;
          }
        }
      } else {  // consumers: H pass + epilogue, one partial triple per frame and tile
        constexpr int CB = 2 + 2 * NB;  // consumer-internal barrier
        const int cw = (tid - VC) >> 5;
        for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
          if (t != (int)blockIdx.x) tile_of(t);
          if constexpr (TSHIFT) tile_shift(tid - VC, VC, VC / 32, [&] { named_sync(CB, VC); });
          fq = fl = fc = 0ull;
          for (int c = 0; c < nchunks; ++c, ++cc) {
            named_sync(2 + b, 2 * VC);
            hpass(c, vbuf0 + b * VBYTES);
            if (cc + NB < total) named_arrive(2 + NB + b, 2 * VC);
            b = b + 1 == NB ? 0 : b + 1;
          }
          double v[6];
          tile_sums(v);
#pragma unroll
          for (int i = 0; i < 6; ++i) v[i] = warp_sum(v[i]);
          if ((tid & 31) == 0) {
#pragma unroll
            for (int i = 0; i < 6; ++i) s_red[cw * 6 + i] = v[i];
          }
          named_sync(CB, VC);
          const int ct = tid - VC;
          if (ct < 6 && (ct < 3 || has1)) {
            double acc = 0.0;
#pragma unroll
            for (int wi = 0; wi < VC / 32; ++wi) acc += s_red[wi * 6 + ct];
            const int fr = ct < 3 ? f0 : f1;
            const long long part = ((long long)fr * nseg + seg) * nstrips + strip;
            a.partials[part * 3 + (ct % 3)] = acc;
          }
          named_sync(CB, VC);  // s_red is rewritten by the next tile
        }
      }
      return;
    } else if (tid < VC) {  // producers
      int b = 0;
      for (int c = 0; c < nchunks; ++c) {
#if SSK_PROD_SYNC1
        cp_async_wait<0>();
        named_sync(1, VC);  // chunk c's raw rows visible; chunk c-1's V pass done everywhere
        if (c + 1 < nchunks) stage_rows(y0 + (c + 1) * G + K - 1, y0 + (c + 2) * G + K - 1);
#else
        if (c + 1 < nchunks) {
          stage_rows(y0 + (c + 1) * G + K - 1, y0 + (c + 2) * G + K - 1);
          cp_async_wait<1>();
        } else {
          cp_async_wait<0>();
        }
        named_sync(1, VC);                                           // chunk c's raw rows visible
#endif
        if constexpr (VC == 256 && ES == 1) {
          if (a.l1_ref) level1(c);
        }
        if (c >= NB) named_sync(2 + NB + b, 2 * VC);                 // consumers released tile b
        vpass(c, vbuf0 + b * VBYTES);
        named_arrive(2 + b, 2 * VC);                                 // tile b full
#if !SSK_PROD_SYNC1
        named_sync(1, VC);                                           // raw rows of chunk c no longer read
#endif
        b = b + 1 == NB ? 0 : b + 1;
      }
    } else {  // consumers
      int b = 0;
      for (int c = 0; c < nchunks; ++c) {
        named_sync(2 + b, 2 * VC);
        hpass(c, vbuf0 + b * VBYTES);
        if (c + NB < nchunks) named_arrive(2 + NB + b, 2 * VC);
        b = b + 1 == NB ? 0 : b + 1;
      }
    }
  }

  double v[6];
  tile_sums(v);
#pragma unroll
  for (int i = 0; i < 6; ++i) v[i] = warp_sum(v[i]);
  if ((tid & 31) == 0) {
#pragma unroll
    for (int i = 0; i < 6; ++i) s_red[(tid >> 5) * 6 + i] = v[i];
  }
  __syncthreads();
  if (tid < 6 && (tid < 3 || has1)) {
    double t = 0.0;
#pragma unroll
    for (int wi = 0; wi < NT / 32; ++wi) t += s_red[wi * 6 + tid];
    const int fr = tid < 3 ? f0 : f1;
    const long long part = ((long long)fr * nseg + seg) * nstrips + strip;
    a.partials[part * 3 + (tid % 3)] = t;
  }
}

template <int K, typename TIN, int NM>
__global__ void __launch_bounds__(GS_THREADS, GS_MINB) gauss_pair_kernel(const __grid_constant__ GaussArgs a) {
  gauss_body<K, TIN, NM, false, GS_THREADS>(a, blockIdx.x, blockIdx.y, blockIdx.z, gridDim.x, gridDim.y, a.taps);
}

template <int K, typename TIN, int NM, int VC>
__global__ void __launch_bounds__(2 * VC, VC == 128 ? 2 : 1) gauss_ws_kernel(const __grid_constant__ GaussArgs a) {
  gauss_body<K, TIN, NM, true, VC>(a, blockIdx.x, blockIdx.y, blockIdx.z, gridDim.x, gridDim.y, a.taps);
}

// Persistent variant (one CTA per SM walking tiles blockIdx.x, + gridDim.x, ...)
template <int K, typename TIN, int NM, int VC, bool L1>
__global__ void __launch_bounds__(2 * VC, 1)
    gauss_ws_persist_kernel(const __grid_constant__ GaussArgs a, const int nstrips, const int nseg) {
  // (the map branch stays compiled in: measured faster here than the MAPS = false build)
  gauss_body<K, TIN, NM, true, VC, true, true, L1>(a, 0, 0, 0, nstrips, nseg, a.taps);
}

// All pyramid levels of one sample type in one launch: blockIdx.x enumerates the
// (level, segment, strip) tiles, so the small coarse levels share the GPU with
// each other instead of each launching a few dozen CTAs.
template <int K, typename TIN, int NM, bool WS, int VC = GS_THREADS>
__global__ void __launch_bounds__(WS ? 2 * VC : VC, WS ? 2 : (VC == 256 ? 2 : 4))
    gauss_levels_kernel(const __grid_constant__ GaussLevels p) {
  int lv = 0;
#pragma unroll
  for (int i = 1; i < GS_MAX_LEVELS; ++i)
    if (i < p.nlev && (int)blockIdx.x >= p.cta_off[i]) lv = i;
  const int local = blockIdx.x - p.cta_off[lv];
  const int ns = p.nstrips[lv];
  const int ntiles = ns * p.nseg[lv];
  const int pair = local / ntiles, tile = local - pair * ntiles;
  gauss_body<K, TIN, NM, WS, VC, false, false>(p.lv[lv], tile % ns, tile / ns, pair, ns, p.nseg[lv], p.lv[0].taps);
}

template <int K, typename TIN, int NM, int VC = GS_THREADS, bool WS = true>
inline size_t smem_bytes() {
  constexpr int TWI = tw_of(K, VC) + K - 1;
  constexpr int RB = ((TWI * (int)sizeof(TIN) + 15) / 16) * 16;
  constexpr int RR = ring_rows(K, WS, (int)sizeof(TIN));
  return (size_t)RR * 4 * RB + (size_t)NM * G * vp_of(VC);
}

int gauss_persist_level();                    // capi.cu: SSK_GAUSS_PERSIST switch (default 1)
int sm_count();                               // capi.cu: SMs of the current device

template <int K, typename TIN, int NM, int VC>
int launch_ws(const GaussArgs& a, dim3 grid, cudaStream_t st) {
  const size_t smem = smem_bytes<K, TIN, NM, VC>() +
                      (size_t)(nbuf_of(VC, (int)sizeof(TIN)) - 1) * NM * G * vp_of(VC);  // extra V tiles
  if constexpr (VC == 256 && sizeof(TIN) == 1) {
    // wide u8 strips (1 CTA / SM): persistent CTAs keep the V-tile pipeline full across tiles
    const long long ntiles = (long long)grid.x * grid.y * grid.z;
    if (gauss_persist_level() >= 1 && ntiles > 0) {
      // two builds: with the fused level-1 stores (MS-SSIM) and without (score-only launches,
      // smaller code and the strength-reduced staging loop)
      auto fp = a.l1_ref ? gauss_ws_persist_kernel<K, TIN, NM, VC, true> : gauss_ws_persist_kernel<K, TIN, NM, VC, false>;
      if (cudaFuncSetAttribute(fp, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return SSK_E_CUDA;
      int nctas = (int)std::min<long long>(ntiles, (long long)sm_count());
      static const int forced = [] {  // SSK_PERSIST_CTAS: fewer CTAs, more tiles each (stress tests)
        const char* e = std::getenv("SSK_PERSIST_CTAS");
        return e ? std::atoi(e) : 0;
      }();
      if (forced > 0) nctas = (int)std::min<long long>(ntiles, (long long)forced);
      fp<<<nctas, 2 * VC, smem, st>>>(a, (int)grid.x, (int)grid.y);
      note_launch();
      return cudaGetLastError() == cudaSuccess ? SSK_OK : SSK_E_CUDA;
    }
  }
  auto fn = gauss_ws_kernel<K, TIN, NM, VC>;
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return SSK_E_CUDA;
  fn<<<grid, 2 * VC, smem, st>>>(a);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? SSK_OK : SSK_E_CUDA;
}

template <int K, typename TIN>
int launch_levels_one(const GaussLevels& p, dim3 grid, cudaStream_t st);
int gauss_l0_classic();                       // capi.cu: SSK_L0_CLASSIC switch (default 1)
int gauss_narrow_ws();                        // capi.cu: SSK_NARROW_WS switch (default 0)

template <int K, typename TIN, int NM>
int launch_nm(const GaussArgs& a, dim3 grid, cudaStream_t st) {
  // map outputs only from the classic kernel (the planner keeps such launches at 128 columns)
  const bool maps = (a.want & (SSK_MAP_TERMS | SSK_MAP_STATS)) != 0;
  if (maps && a.vcols != GS_THREADS) return SSK_E_ARG;
  if (NM == 4 && a.vcols == 256) {
    if constexpr (sizeof(TIN) <= 2 && K <= 17) {
      // SSK_L0_CLASSIC=1: wide strips on the classic (non-specialised) kernel, 2 CTAs of 256
      // threads per SM, through the multi-level launch with a single level
      if (gauss_l0_classic()) {
        GaussLevels gl{};
        gl.lv[0] = a;
        gl.nlev = 1;
        gl.npairs = (int)grid.z;
        gl.cta_off[0] = 0;
        gl.nstrips[0] = (int)grid.x;
        gl.nseg[0] = (int)grid.y;
        return launch_levels_one<K, TIN>(gl, dim3(grid.x * grid.y * grid.z, 1, 1), st);
      }
    }
    if constexpr (sizeof(TIN) <= 2 && 256 - (K - 1) >= 16) return launch_ws<K, TIN, NM, 256>(a, grid, st);
    return SSK_E_ARG;
  }
  // 128-column strips: the classic kernel (4 CTAs/SM) measures ~5 % faster than the
  // warp-specialised one since the sum / difference epilogue (SSK_NARROW_WS=1 restores it)
  if (NM == 4 && !maps && gauss_ws_enabled() && gauss_narrow_ws()) return launch_ws<K, TIN, NM, GS_THREADS>(a, grid, st);
  auto fn = gauss_pair_kernel<K, TIN, NM>;
  const size_t smem = smem_bytes<K, TIN, NM, GS_THREADS, false>();
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return SSK_E_CUDA;
  fn<<<grid, GS_THREADS, smem, st>>>(a);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? SSK_OK : SSK_E_CUDA;
}

template <int K, typename TIN>
int launch_one(const GaussArgs& a, dim3 grid, cudaStream_t st) {
  // the statistics maps need the five separate moments; everything else runs on four
  return (a.want & SSK_MAP_STATS) ? launch_nm<K, TIN, 5>(a, grid, st) : launch_nm<K, TIN, 4>(a, grid, st);
}

template <int K, typename TIN>
int launch_levels_one(const GaussLevels& p, dim3 grid, cudaStream_t st) {
  // the coarse levels stay on the classic (non-specialised) kernel: measured faster there
  // (small tiles, 3-4 CTAs/SM); SSK_GAUSS_WS=2 forces the warp-specialised variant
  if constexpr (K <= 17) {
    if (p.lv[0].vcols == 256) {  // wide strips (240 outputs), 2 CTAs of 256 threads per SM
      // (a separate build without the fused level-1 stores measured the same: 0.5812 ms)
      auto fw = gauss_levels_kernel<K, TIN, 4, false, 256>;
      const size_t smem = smem_bytes<K, TIN, 4, 256, false>();
      if (cudaFuncSetAttribute(fw, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return SSK_E_CUDA;
      fw<<<grid, 256, smem, st>>>(p);
      note_launch();
      return cudaGetLastError() == cudaSuccess ? SSK_OK : SSK_E_CUDA;
    }
  }
  if (p.lv[0].vcols != GS_THREADS) return SSK_E_ARG;
  const bool ws = gauss_ws_level() >= 2;
  auto fn = ws ? gauss_levels_kernel<K, TIN, 4, true> : gauss_levels_kernel<K, TIN, 4, false>;
  const size_t smem = ws ? smem_bytes<K, TIN, 4>() + (size_t)(GS_NBUF - 1) * 4 * G * vp_of(GS_THREADS)
                        : smem_bytes<K, TIN, 4, GS_THREADS, false>();
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return SSK_E_CUDA;
  fn<<<grid, ws ? 2 * GS_THREADS : GS_THREADS, smem, st>>>(p);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? SSK_OK : SSK_E_CUDA;
}

template <typename TIN>
int launch_levels_dtype(const GaussLevels& p, dim3 grid, int k, cudaStream_t st) {
  switch (k) {
    case 11: return launch_levels_one<11, TIN>(p, grid, st);
#ifndef SSK_K11_ONLY  // (A/B builds: only the 11-tap kernels, a quarter of the compile time)
    case 3: return launch_levels_one<3, TIN>(p, grid, st);
    case 5: return launch_levels_one<5, TIN>(p, grid, st);
    case 7: return launch_levels_one<7, TIN>(p, grid, st);
    case 9: return launch_levels_one<9, TIN>(p, grid, st);
    case 13: return launch_levels_one<13, TIN>(p, grid, st);
    case 15: return launch_levels_one<15, TIN>(p, grid, st);
    case 17: return launch_levels_one<17, TIN>(p, grid, st);
    case 19: return launch_levels_one<19, TIN>(p, grid, st);
    case 21: return launch_levels_one<21, TIN>(p, grid, st);
    case 23: return launch_levels_one<23, TIN>(p, grid, st);
    case 25: return launch_levels_one<25, TIN>(p, grid, st);
    case 27: return launch_levels_one<27, TIN>(p, grid, st);
    case 29: return launch_levels_one<29, TIN>(p, grid, st);
    case 31: return launch_levels_one<31, TIN>(p, grid, st);
#endif
    default: return SSK_E_SHAPE;
  }
}

template <typename TIN>
int launch_dtype(const GaussArgs& a, dim3 grid, int k, cudaStream_t st) {
  switch (k) {
    case 11: return launch_one<11, TIN>(a, grid, st);
#ifndef SSK_K11_ONLY  // (A/B builds: only the 11-tap kernels, a quarter of the compile time)
    case 3: return launch_one<3, TIN>(a, grid, st);
    case 5: return launch_one<5, TIN>(a, grid, st);
    case 7: return launch_one<7, TIN>(a, grid, st);
    case 9: return launch_one<9, TIN>(a, grid, st);
    case 13: return launch_one<13, TIN>(a, grid, st);
    case 15: return launch_one<15, TIN>(a, grid, st);
    case 17: return launch_one<17, TIN>(a, grid, st);
    case 19: return launch_one<19, TIN>(a, grid, st);
    case 21: return launch_one<21, TIN>(a, grid, st);
    case 23: return launch_one<23, TIN>(a, grid, st);
    case 25: return launch_one<25, TIN>(a, grid, st);
    case 27: return launch_one<27, TIN>(a, grid, st);
    case 29: return launch_one<29, TIN>(a, grid, st);
    case 31: return launch_one<31, TIN>(a, grid, st);
#endif
    default: return SSK_E_SHAPE;
  }
}

}  // namespace gk
}  // namespace ssk
