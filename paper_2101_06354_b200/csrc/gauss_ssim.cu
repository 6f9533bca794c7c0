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
// Structure (one CTA = 128 threads = a strip of 128 output columns times a
// segment of output rows, sliding down in chunks of G=8 input rows):
//   stage  : cp.async 16-B copies of the chunk's ref/dist rows (raw u8/u16/
//            f32) into a double-buffered shared-memory stage, zero-filled
//            past the right edge.
//   H-pass : thread (row g, column group j) converts 8+K-1 samples of both
//            frames (exact u8/u16 -> fp32 via PRMT into the 2^23 mantissa),
//            subtracts the symmetric shift L/2 (keeps E[x^2]-E[x]^2 well
//            conditioned in fp32 and preserves exact ref/dist symmetry),
//            forms x, y, x^2, y^2, xy and runs the 11-tap horizontal filter
//            for 8 adjacent outputs from registers; results go to a ring of
//            R = G+K-1 rows per moment in shared memory, so every input row is
//            filtered horizontally exactly once per strip segment.
//   V-pass : thread = output column; gathers G+K-1 ring rows and forms G
//            vertical outputs per moment (5*G accumulators), then the SSIM
//            epilogue, optional map stores and fp32->fp64 partial sums.
//   reduce : warp-shuffle + shared-memory block reduction of (sum q, sum l,
//            sum cs) into one fp64 partial per CTA (deterministic; a second
//            tiny kernel folds the partials per frame in fixed order).
// Every output value is produced by the same operation sequence whatever the
// stride, so strided grids equal dense[::s, ::s] bit-exactly
// (tests/test_stats.py:274-285).
#include "common.cuh"
#include "kernels.h"

namespace ssk {

namespace {

constexpr int G = GS_G;
constexpr int HP = GS_HP;

template <int K>
struct GaussGeom {
  static constexpr int R = G + K - 1;          // ring rows
  static constexpr int NS = 8 + K - 1;         // samples per H item
  static constexpr int TWI = GS_TW + K - 1;    // staged input columns
};

// Load NS consecutive samples starting at column `col` of a staged row and
// return them as shifted fp32 values.
template <int K>
__device__ __forceinline__ void load_samples(const unsigned char* row, int col, int dtype,
                                             float scale, float bias, float (&v)[8 + K - 1]) {
  constexpr int NS = 8 + K - 1;
  if (dtype == SSK_U8) {
    constexpr int NW = (NS + 7) / 8;
    const uint2* p = reinterpret_cast<const uint2*>(row + col);
    uint32_t wds[2 * NW];
#pragma unroll
    for (int i = 0; i < NW; ++i) {
      uint2 t = p[i];
      wds[2 * i] = t.x;
      wds[2 * i + 1] = t.y;
    }
#pragma unroll
    for (int i = 0; i < NS; ++i) v[i] = fmaf(u8_as_biased(wds[i >> 2], i & 3), scale, bias);
  } else if (dtype == SSK_U16) {
    constexpr int NW = (NS + 7) / 8;
    const uint4* p = reinterpret_cast<const uint4*>(row + 2 * col);
    uint32_t wds[4 * NW];
#pragma unroll
    for (int i = 0; i < NW; ++i) {
      uint4 t = p[i];
      wds[4 * i] = t.x;
      wds[4 * i + 1] = t.y;
      wds[4 * i + 2] = t.z;
      wds[4 * i + 3] = t.w;
    }
#pragma unroll
    for (int i = 0; i < NS; ++i) v[i] = fmaf(u16_as_biased(wds[i >> 1], i & 1), scale, bias);
  } else {
    constexpr int NW = (NS + 3) / 4;
    const uint4* p = reinterpret_cast<const uint4*>(row + 4 * col);
    uint32_t wds[4 * NW];
#pragma unroll
    for (int i = 0; i < NW; ++i) {
      uint4 t = p[i];
      wds[4 * i] = t.x;
      wds[4 * i + 1] = t.y;
      wds[4 * i + 2] = t.z;
      wds[4 * i + 3] = t.w;
    }
    if (dtype == SSK_F32) {
#pragma unroll
      for (int i = 0; i < NS; ++i) v[i] = fmaf(__uint_as_float(wds[i]), scale, bias);
    } else {  // SSK_U32: exact below 2^24
#pragma unroll
      for (int i = 0; i < NS; ++i) v[i] = fmaf(__uint2float_rn(wds[i]), scale, bias);
    }
  }
}

// Horizontal K-tap filter of 8 adjacent outputs; taps symmetric (w[i] == w[K-1-i]).
template <int K>
__device__ __forceinline__ void hfilter_store(const float (&t)[8 + K - 1],
                                              const float (&w)[(K + 1) / 2], float* dst) {
  float acc[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) acc[j] = 0.f;
#pragma unroll
  for (int i = 0; i < K; ++i) {
    const float wi = w[i < K - 1 - i ? i : K - 1 - i];
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] = fmaf(wi, t[j + i], acc[j]);
  }
  reinterpret_cast<float4*>(dst)[0] = make_float4(acc[0], acc[1], acc[2], acc[3]);
  reinterpret_cast<float4*>(dst)[1] = make_float4(acc[4], acc[5], acc[6], acc[7]);
}

__device__ __forceinline__ float rcp_approx(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

}  // namespace

template <int K>
__global__ void __launch_bounds__(GS_THREADS, 4) gauss_ssim_kernel(const __grid_constant__ GaussArgs a) {
  using Geo = GaussGeom<K>;
  constexpr int R = Geo::R;
  constexpr int NS = Geo::NS;
  extern __shared__ __align__(16) unsigned char smem[];
  float* ring = reinterpret_cast<float*>(smem);                 // [5][R][HP]
  unsigned char* stage = smem + 5 * R * HP * sizeof(float);     // [2][2][G][in_pitch]
  __shared__ float s_taps[32];
  __shared__ double s_red[(GS_THREADS / 32) * 3];

  const int tid = threadIdx.x;
  const int strip = blockIdx.x, seg = blockIdx.y, frame = blockIdx.z;
  const int c0 = strip * GS_TW;
  const int y0 = seg * a.seg_rows;                  // first output row of this segment
  const int y1 = min(y0 + a.seg_rows, a.ho);        // one past the last output row
  const int in_end = y1 + K - 1;                    // one past the last input row needed
  const int P = a.in_pitch;

  if (tid < 32) s_taps[tid] = a.taps[tid];

  const unsigned char* base_x = a.ref + (long long)frame * a.frame_pitch_b;
  const unsigned char* base_y = a.dist + (long long)frame * a.frame_pitch_b;
  const int esz = a.esize;
  const int nch = (Geo::TWI * esz + 15) >> 4;       // 16-byte chunks per staged row
  const int row_bytes_left = (a.w - c0) * esz;      // valid bytes from c0 to the row end

  auto issue_stage = [&](int chunk, int buf) {
    const int rbase = y0 + chunk * G;
    const int total = 2 * G * nch;
    for (int i = tid; i < total; i += GS_THREADS) {
      const int img = i / (G * nch);
      const int rem = i - img * (G * nch);
      const int g = rem / nch;
      const int q = rem - g * nch;
      const int row = rbase + g;
      if (row >= in_end) continue;
      const int off = q * 16;
      int valid = row_bytes_left - off;
      valid = valid < 0 ? 0 : (valid > 16 ? 16 : valid);
      const unsigned char* rowp = (img ? base_y : base_x) + (long long)row * a.row_pitch_b;
      const unsigned char* src = valid ? rowp + (long long)c0 * esz + off : rowp;
      unsigned char* dst = stage + ((buf * 2 + img) * G + g) * P + off;
      cp_async16(dst, src, valid);
    }
    cp_async_commit();
  };

  const int nchunks = (in_end - y0 + G - 1) / G;
  issue_stage(0, 0);
  __syncthreads();  // s_taps
  float w[(K + 1) / 2];
#pragma unroll
  for (int i = 0; i < (K + 1) / 2; ++i) w[i] = s_taps[i];

  const float scale = a.conv_scale, bias = a.conv_bias, shift = a.shift;
  const float c1 = a.c1, c2 = a.c2;
  const bool full_terms = (a.want & (SSK_WANT_Q | SSK_WANT_L)) != 0;
  const bool want_maps = (a.want & (SSK_MAP_TERMS | SSK_MAP_STATS)) != 0;
  const int s = a.stride;
  const int col = c0 + tid;                         // this thread's output column in the V pass
  const bool col_ok = col < a.wo && (s == 1 || (col % s) == 0);

  double tot_q = 0.0, tot_l = 0.0, tot_cs = 0.0;
  int emitted = y0;                                 // next output row to emit

  // H-pass item of this thread
  const int hg = tid & 7, hj = tid >> 3;

  for (int c = 0; c < nchunks; ++c) {
    if (c + 1 < nchunks) {
      issue_stage(c + 1, (c + 1) & 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();

    // ---------------- H pass ----------------
    {
      const int row = y0 + c * G + hg;
      if (row < in_end) {
        const unsigned char* sx = stage + (((c & 1) * 2 + 0) * G + hg) * P;
        const unsigned char* sy = stage + (((c & 1) * 2 + 1) * G + hg) * P;
        float xs[NS], ys[NS];
        load_samples<K>(sx, 8 * hj, a.dtype, scale, bias, xs);
        load_samples<K>(sy, 8 * hj, a.dtype, scale, bias, ys);
        const int slot = (c * G + hg) % R;
        float* dst = ring + slot * HP + 8 * hj;
        hfilter_store<K>(xs, w, dst);
        hfilter_store<K>(ys, w, dst + R * HP);
        {
          float t[NS];
#pragma unroll
          for (int i = 0; i < NS; ++i) t[i] = xs[i] * xs[i];
          hfilter_store<K>(t, w, dst + 2 * R * HP);
#pragma unroll
          for (int i = 0; i < NS; ++i) t[i] = ys[i] * ys[i];
          hfilter_store<K>(t, w, dst + 3 * R * HP);
#pragma unroll
          for (int i = 0; i < NS; ++i) t[i] = xs[i] * ys[i];
          hfilter_store<K>(t, w, dst + 4 * R * HP);
        }
      }
    }
    __syncthreads();

    // ---------------- V pass + epilogue ----------------
    const int avail = min(y0 + (c + 1) * G - K + 1, y1);  // rows [emitted, avail) are ready
    const int nv = avail - emitted;
    if (nv > 0) {
      float acc[5][G];
#pragma unroll
      for (int m = 0; m < 5; ++m)
#pragma unroll
        for (int r = 0; r < G; ++r) acc[m][r] = 0.f;
      const int sb = (emitted - y0) % R;
#pragma unroll
      for (int u = 0; u < G + K - 1; ++u) {
        int sl = sb + u;
        sl = sl >= R ? sl - R : sl;
        const float* hp = ring + sl * HP + tid;
        float h[5];
#pragma unroll
        for (int m = 0; m < 5; ++m) h[m] = hp[m * R * HP];
#pragma unroll
        for (int r = 0; r < G; ++r) {
          const int i = u - r;
          if (i >= 0 && i < K) {
            const float wi = w[i < K - 1 - i ? i : K - 1 - i];
#pragma unroll
            for (int m = 0; m < 5; ++m) acc[m][r] = fmaf(wi, h[m], acc[m][r]);
          }
        }
      }
      float sq = 0.f, sl_ = 0.f, scs = 0.f;
      if (col_ok) {
#pragma unroll
        for (int r = 0; r < G; ++r) {
          const int orow = emitted + r;
          if (r < nv && (s == 1 || (orow % s) == 0)) {
            const float m1 = acc[0][r], m2 = acc[1][r];
            const float v1 = fmaxf(fmaf(-m1, m1, acc[2][r]), 0.f);
            const float v2 = fmaxf(fmaf(-m2, m2, acc[3][r]), 0.f);
            const float cv = fmaf(-m1, m2, acc[4][r]);
            const float num2 = fmaf(2.f, cv, c2);
            const float den2 = __fadd_rn(__fadd_rn(v1, v2), c2);
            float l = 1.f, cs, q;
            const float mu1 = m1 + shift, mu2 = m2 + shift;
            if (full_terms) {
              const float num1 = fmaf(2.f * mu1, mu2, c1);
              const float den1 = __fadd_rn(__fadd_rn(__fmul_rn(mu1, mu1), __fmul_rn(mu2, mu2)), c1);
              const float inv = rcp_approx(den1 * den2);
              l = num1 * den2 * inv;
              cs = num2 * den1 * inv;
              q = num1 * num2 * inv;
              sq += q;
              sl_ += l;
            } else {
              cs = num2 * rcp_approx(den2);
              q = cs;
            }
            scs += cs;
            if (want_maps) {
              const long long idx = (long long)(orow / s) * a.gw + (col / s);
              float* mp = reinterpret_cast<float*>(a.maps) + (long long)frame * a.map_frame + idx;
              if (a.want & SSK_MAP_TERMS) {
                mp[0] = l;
                mp[a.map_plane] = cs;
                mp[2 * a.map_plane] = q;
              } else {
                mp[0] = mu1;
                mp[a.map_plane] = mu2;
                mp[2 * a.map_plane] = v1;
                mp[3 * a.map_plane] = v2;
                mp[4 * a.map_plane] = cv;
              }
            }
          }
        }
      }
      tot_q += sq;
      tot_l += sl_;
      tot_cs += scs;
      emitted = avail;
    }
  }

  double v[3] = {tot_q, tot_l, tot_cs};
  const long long part = ((long long)frame * gridDim.y + seg) * gridDim.x + strip;
  block_sum_store<3, GS_THREADS / 32>(v, s_red, a.partials + part * 3);
}

// ---------------------------------------------------------------------------

template <int K>
static int launch_k(const GaussArgs& a, dim3 grid, size_t smem, cudaStream_t st) {
  auto fn = gauss_ssim_kernel<K>;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return SSK_E_CUDA;
  fn<<<grid, GS_THREADS, smem, st>>>(a);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? SSK_OK : SSK_E_CUDA;
}

size_t gauss_smem_bytes(int k, int in_pitch) {
  const int R = G + k - 1;
  return (size_t)5 * R * HP * sizeof(float) + (size_t)4 * G * in_pitch;
}

int gauss_in_pitch(int k, int esize) {
  const int twi = GS_TW + k - 1;
  const int ns = 8 + k - 1;
  int vec_bytes;  // bytes an H item reads past its first sample
  if (esize == 1) vec_bytes = ((ns + 7) / 8) * 8;
  else if (esize == 2) vec_bytes = ((ns + 7) / 8) * 16;
  else vec_bytes = ((ns + 3) / 4) * 16;
  const int need = (GS_TW - 8) * esize + vec_bytes;
  int ext = twi * esize;
  ext = ((ext + 15) / 16) * 16;
  if (need > ext) ext = need;
  // pitch == 16 (mod 128) keeps the 8 rows read by a quarter warp on distinct banks
  return ((ext - 16 + 127) / 128) * 128 + 16;
}

int launch_gauss(const GaussArgs& a, dim3 grid, int k, cudaStream_t st) {
  const size_t smem = gauss_smem_bytes(k, a.in_pitch);
  switch (k) {
    case 3: return launch_k<3>(a, grid, smem, st);
    case 5: return launch_k<5>(a, grid, smem, st);
    case 7: return launch_k<7>(a, grid, smem, st);
    case 9: return launch_k<9>(a, grid, smem, st);
    case 11: return launch_k<11>(a, grid, smem, st);
    case 13: return launch_k<13>(a, grid, smem, st);
    case 15: return launch_k<15>(a, grid, smem, st);
    case 17: return launch_k<17>(a, grid, smem, st);
    case 19: return launch_k<19>(a, grid, smem, st);
    case 21: return launch_k<21>(a, grid, smem, st);
    case 23: return launch_k<23>(a, grid, smem, st);
    case 25: return launch_k<25>(a, grid, smem, st);
    case 27: return launch_k<27>(a, grid, smem, st);
    case 29: return launch_k<29>(a, grid, smem, st);
    case 31: return launch_k<31>(a, grid, smem, st);
    default: return SSK_E_SHAPE;
  }
}

}  // namespace ssk
