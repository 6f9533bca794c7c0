// Auxiliary kernels: deterministic partial folding, the 2x2 pyramid step,
// summed-area tables for the IntegralSet API, and the FP32 peak probe.
#include <type_traits>

#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace ssk {

// ---------------------------------------------------------------------------
// Fold per-CTA partials [n][nparts][ncomp] into out[f*out_stride + out_offset + c]
// = (sum_p partials[f][p][comp_offset + c]) / divisor (IEEE division, so a
// mean is rounded exactly like numpy's sum/count); one warp per frame, fixed
// order -> bit-reproducible run to run (the reference's ordered frame results,
// tests/test_cli.py:124-130, rely on determinism).
// ---------------------------------------------------------------------------
// One 256-thread block per frame: thread t folds partials t, t + 256, ... then the eight
// warp sums combine in warp order -- a fixed order that depends on nparts only (a frame's
// mean is the same however frames are batched), with 8x the loads in flight of a single
// warp (per-pair calls with ~16k partials were latency-bound at ~95 us).
__global__ void __launch_bounds__(256) reduce_partials_kernel(const double* __restrict__ partials, int nparts,
                                                              int n, int ncomp, double divisor,
                                                              double* __restrict__ out, int out_stride,
                                                              int out_offset, int comp_offset) {
  __shared__ double s_w[8];
  const int f = blockIdx.x;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const double* p = partials + (long long)f * nparts * 3;
  for (int c = 0; c < ncomp; ++c) {
    double s = 0.0;
    for (int i = threadIdx.x; i < nparts; i += 256) s += p[(long long)i * 3 + comp_offset + c];
    s = warp_sum(s);
    if (lane == 0) s_w[w] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
#pragma unroll
      for (int i = 0; i < 8; ++i) t += s_w[i];
      out[(long long)f * out_stride + out_offset + c] = divisor == 1.0 ? t : __ddiv_rn(t, divisor);
    }
    __syncthreads();
  }
}

int launch_reduce_partials(const double* partials, int nparts, int n, int ncomp, double divisor,
                           double* out, int out_stride, int out_offset, int comp_offset,
                           cudaStream_t st) {
  if (n < 1) return SSK_OK;
  reduce_partials_kernel<<<n, 256, 0, st>>>(partials, nparts, n, ncomp, divisor, out, out_stride, out_offset,
                                             comp_offset);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? SSK_OK : SSK_E_CUDA;
}

// ---------------------------------------------------------------------------
// dyadic_downsample (src/multiscale.py:19-33): 2x2 block over the even-trimmed
// plane.  Integer planes keep the exact sum of the four samples (the caller
// tracks the 4^-s scale); float planes compute ((a00+a01)+a10)+a11 then /4
// exactly like the reference's numpy expression.
// ---------------------------------------------------------------------------
template <typename TS, typename TD>
__global__ void __launch_bounds__(128) downsample_kernel(const unsigned char* __restrict__ src_r,
                                                         const unsigned char* __restrict__ src_d, long long src_rp,
                                                         long long src_fp, int h2, int w2,
                                                         unsigned char* __restrict__ dst_r,
                                                         unsigned char* __restrict__ dst_d, long long dst_rp,
                                                         long long dst_fp) {
  // thread -> 8 adjacent outputs of one row: 16 input samples from each of two rows,
  // read as whole 16-byte vectors (row pitches are 16-byte multiples by contract)
  const int x8 = (blockIdx.x * blockDim.x + threadIdx.x) * 8;
  const int y = blockIdx.y;
  const int f = blockIdx.z >> 1;
  const int img = blockIdx.z & 1;
  if (x8 >= w2) return;
  const TS* s = reinterpret_cast<const TS*>((img ? src_d : src_r)) + f * src_fp;
  TD* d = reinterpret_cast<TD*>((img ? dst_d : dst_r)) + f * dst_fp + (long long)y * dst_rp + x8;
  const TS* r0 = s + (long long)(2 * y) * src_rp + 2 * x8;
  const TS* r1 = r0 + src_rp;
  constexpr int NV = 16 * (int)sizeof(TS) / 16;  // 16-byte vectors per 16 samples
  TS a0[16], a1[16];
  if (x8 + 8 <= w2) {
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      reinterpret_cast<uint4*>(a0)[i] = reinterpret_cast<const uint4*>(r0)[i];
      reinterpret_cast<uint4*>(a1)[i] = reinterpret_cast<const uint4*>(r1)[i];
    }
  } else {
    const int n = 2 * (w2 - x8);
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      a0[i] = i < n ? r0[i] : (TS)0;
      a1[i] = i < n ? r1[i] : (TS)0;
    }
  }
  TD o[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    if constexpr (std::is_floating_point<TS>::value) {
      o[i] = (TD)((((a0[2 * i] + a0[2 * i + 1]) + a1[2 * i]) + a1[2 * i + 1]) / (TS)4);
    } else {
      o[i] = (TD)((uint32_t)a0[2 * i] + a0[2 * i + 1] + a1[2 * i] + a1[2 * i + 1]);
    }
  }
  if (x8 + 8 <= w2 && ((reinterpret_cast<uintptr_t>(d) & 15) == 0)) {
    constexpr int NO = 8 * (int)sizeof(TD) / 16 > 0 ? 8 * (int)sizeof(TD) / 16 : 1;
    if constexpr (8 * sizeof(TD) >= 16) {
#pragma unroll
      for (int i = 0; i < NO; ++i) reinterpret_cast<uint4*>(d)[i] = reinterpret_cast<const uint4*>(o)[i];
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) d[i] = o[i];
    }
  } else {
    const int n = min(8, w2 - x8);
    for (int i = 0; i < n; ++i) d[i] = o[i];
  }
}

template <typename TS, typename TD>
static void ds_launch(const unsigned char* sr, const unsigned char* sd, long long srp, long long sfp,
                      int n, int h2, int w2, unsigned char* dr, unsigned char* dd, long long drp,
                      long long dfp, cudaStream_t st) {
  dim3 block(128);
  dim3 grid((w2 + 8 * 128 - 1) / (8 * 128), h2, 2 * n);
  downsample_kernel<TS, TD><<<grid, block, 0, st>>>(sr, sd, srp, sfp, h2, w2, dr, dd, drp, dfp);
}

int launch_downsample(const unsigned char* src_r, const unsigned char* src_d, int src_dtype,
                      long long src_rp, long long src_fp, int n, int h, int w,
                      unsigned char* dst_r, unsigned char* dst_d, int dst_dtype, long long dst_rp,
                      long long dst_fp, cudaStream_t st) {
  const int h2 = h / 2, w2 = w / 2;
  if (h2 < 1 || w2 < 1) return SSK_E_TOO_SMALL;
  if (2 * n > 65535 || h2 > 65535) return SSK_E_ARG;
#define DS(TS, TD) ds_launch<TS, TD>(src_r, src_d, src_rp, src_fp, n, h2, w2, dst_r, dst_d, dst_rp, dst_fp, st)
  if (src_dtype == SSK_U8 && dst_dtype == SSK_U16) DS(uint8_t, uint16_t);
  else if (src_dtype == SSK_U8 && dst_dtype == SSK_U32) DS(uint8_t, uint32_t);
  else if (src_dtype == SSK_U16 && dst_dtype == SSK_U16) DS(uint16_t, uint16_t);
  else if (src_dtype == SSK_U16 && dst_dtype == SSK_U32) DS(uint16_t, uint32_t);
  else if (src_dtype == SSK_U32 && dst_dtype == SSK_U32) DS(uint32_t, uint32_t);
  else if (src_dtype == SSK_F32 && dst_dtype == SSK_F32) DS(float, float);
  else if (src_dtype == SSK_F64 && dst_dtype == SSK_F64) DS(double, double);
  else return SSK_E_ARG;
#undef DS
  note_launch();
  return cudaGetLastError() == cudaSuccess ? SSK_OK : SSK_E_CUDA;
}

// ---------------------------------------------------------------------------
// Summed-area tables (src/stats.py:66-71): out[f][t][h+1][w+1] with a zero
// first row/column; t = (x, y, x^2, y^2, xy).  The reference takes
// cumsum(axis=0) then cumsum(axis=1), sequentially; the same order is kept
// (column pass then row pass), so float64 tables match bit for bit and
// integer tables are exact int64.
// ---------------------------------------------------------------------------
template <typename TS, typename TA>
__global__ void sat_column_kernel(const unsigned char* __restrict__ ref,
                                  const unsigned char* __restrict__ dist, long long rp, long long fp,
                                  int h, int w, TA* __restrict__ out) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int f = blockIdx.y;
  if (x > w) return;
  const long long plane = (long long)(h + 1) * (w + 1);
  TA* o = out + (long long)f * 5 * plane;
  for (int t = 0; t < 5; ++t) o[t * plane + x] = 0;  // zero first row
  if (x == 0) {
    for (int y = 1; y <= h; ++y)
      for (int t = 0; t < 5; ++t) o[t * plane + (long long)y * (w + 1)] = 0;
    return;
  }
  const TS* a = reinterpret_cast<const TS*>(ref) + f * fp + (x - 1);
  const TS* b = reinterpret_cast<const TS*>(dist) + f * fp + (x - 1);
  TA acc[5] = {0, 0, 0, 0, 0};
  for (int y = 0; y < h; ++y) {
    const TA va = (TA)a[(long long)y * rp], vb = (TA)b[(long long)y * rp];
    acc[0] += va;
    acc[1] += vb;
    acc[2] += va * va;
    acc[3] += vb * vb;
    acc[4] += va * vb;
    for (int t = 0; t < 5; ++t) o[t * plane + (long long)(y + 1) * (w + 1) + x] = acc[t];
  }
}

template <typename TA>
__global__ void sat_row_kernel(int h, int w, TA* __restrict__ out) {
  const int y = blockIdx.x * blockDim.x + threadIdx.x + 1;
  const int t = blockIdx.y;
  const int f = blockIdx.z;
  if (y > h) return;
  const long long plane = (long long)(h + 1) * (w + 1);
  TA* row = out + ((long long)f * 5 + t) * plane + (long long)y * (w + 1);
  TA acc = 0;
  for (int x = 1; x <= w; ++x) {
    acc += row[x];
    row[x] = acc;
  }
}

int launch_integral(const unsigned char* ref, const unsigned char* dist, int dtype, long long rp,
                    long long fp, int n, int h, int w, void* out, cudaStream_t st) {
  dim3 gc((w + 1 + 127) / 128, n), gr((h + 127) / 128, 5, n);
  switch (dtype) {
    case SSK_U8:
      sat_column_kernel<uint8_t, long long><<<gc, 128, 0, st>>>(ref, dist, rp, fp, h, w, (long long*)out);
      sat_row_kernel<long long><<<gr, 128, 0, st>>>(h, w, (long long*)out);
      break;
    case SSK_U16:
      sat_column_kernel<uint16_t, long long><<<gc, 128, 0, st>>>(ref, dist, rp, fp, h, w, (long long*)out);
      sat_row_kernel<long long><<<gr, 128, 0, st>>>(h, w, (long long*)out);
      break;
    case SSK_U32:
      sat_column_kernel<uint32_t, long long><<<gc, 128, 0, st>>>(ref, dist, rp, fp, h, w, (long long*)out);
      sat_row_kernel<long long><<<gr, 128, 0, st>>>(h, w, (long long*)out);
      break;
    case SSK_F32:
      sat_column_kernel<float, double><<<gc, 128, 0, st>>>(ref, dist, rp, fp, h, w, (double*)out);
      sat_row_kernel<double><<<gr, 128, 0, st>>>(h, w, (double*)out);
      break;
    case SSK_F64:
      sat_column_kernel<double, double><<<gc, 128, 0, st>>>(ref, dist, rp, fp, h, w, (double*)out);
      sat_row_kernel<double><<<gr, 128, 0, st>>>(h, w, (double*)out);
      break;
    default:
      return SSK_E_ARG;
  }
  note_launch(2);
  return cudaGetLastError() == cudaSuccess ? SSK_OK : SSK_E_CUDA;
}

// ---------------------------------------------------------------------------
// FP32 FMA probe: 16 independent register-form FFMA chains per thread.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) fp32_probe_kernel(float* out, int iters, float b, float c) {
  float acc[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) acc[i] = threadIdx.x * 1e-6f + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int i = 0; i < 16; ++i) acc[i] = fmaf(acc[i], b, c);
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += acc[i];
  if (s == 1234.5f) out[0] = s;
}

int probe_fp32(double seconds, double* tflops, cudaStream_t st) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  float* d = nullptr;
  if (cudaMalloc(&d, 4) != cudaSuccess) return SSK_E_CUDA;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int blocks = sms * 8, threads = 256, iters = 20000;
  const double flops_per_launch = 2.0 * blocks * threads * (double)iters * 8 * 16;
  fp32_probe_kernel<<<blocks, threads, 0, st>>>(d, iters, 1.0001f, 0.5f);  // warm-up
  note_launch();
  cudaEventRecord(e0, st);
  int launches = 0;
  float ms = 0.f;
  do {
    fp32_probe_kernel<<<blocks, threads, 0, st>>>(d, iters, 1.0001f, 0.5f);
    note_launch();
    ++launches;
    if (launches % 8 == 0) {
      cudaEventRecord(e1, st);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
    }
  } while (ms < seconds * 1e3);
  *tflops = flops_per_launch * launches / (ms * 1e-3) / 1e12;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(d);
  return cudaGetLastError() == cudaSuccess ? SSK_OK : SSK_E_CUDA;
}

}  // namespace ssk

namespace ssk {

// ---------------------------------------------------------------------------
// Whole dyadic pyramid in one pass (src/multiscale.py:19-33 applied level after
// level).  Thread -> one BxB block (B = 2^NL) of the source plane: it reads the
// block once (16-byte vector rows) and emits the block's samples of every level
// 1..NL, each level formed from the previous one exactly as the reference does
// (integer planes: exact sums of 4, scale 4^-l tracked by the caller; float
// planes: ((a00+a01)+a10)+a11)/4 per level).  Level dims nest as floor(h/2^l), so
// every level-l sample lies inside exactly one block.
// ---------------------------------------------------------------------------
template <typename TS, typename TD, int NL>
__global__ void __launch_bounds__(128) pyramid_kernel(const __grid_constant__ PyramidArgs p) {
  constexpr int B = 1 << NL;
  constexpr bool FLT = std::is_floating_point<TS>::value;
  using TA = typename std::conditional<FLT, TS, uint32_t>::type;  // working type
  const int bx = blockIdx.x * blockDim.x + threadIdx.x;
  const int by = blockIdx.y;
  const int f = blockIdx.z >> 1, img = blockIdx.z & 1;
  if (bx * B >= 2 * p.wl[0]) return;  // no level-1 sample in this block
  const TS* src = reinterpret_cast<const TS*>(img ? p.src_d : p.src_r) + (long long)f * p.src_fp;
  const int r0 = by * B, c0 = bx * B;
  // level-1 rows of the block, kept in registers for the coarser levels
  TA lv[B / 2][B / 2];
  const bool full = (r0 + B <= 2 * p.hl[0]) && (c0 + B <= 2 * p.wl[0]);
  constexpr bool VEC = (B * sizeof(TS)) % 16 == 0 && B * sizeof(TS) <= 16;  // one 16-B vector per row
  if (VEC && full) {
    // interior block: issue all B row loads before any arithmetic (memory-level parallelism)
    uint4 rows[B];
#pragma unroll
    for (int r = 0; r < B; ++r) rows[r] = *reinterpret_cast<const uint4*>(src + (long long)(r0 + r) * p.src_rp + c0);
#pragma unroll
    for (int i = 0; i < B / 2; ++i) {
      const TS* a0 = reinterpret_cast<const TS*>(&rows[2 * i]);
      const TS* a1 = reinterpret_cast<const TS*>(&rows[2 * i + 1]);
#pragma unroll
      for (int j = 0; j < B / 2; ++j) {
        if constexpr (FLT) {
          lv[i][j] = (((a0[2 * j] + a0[2 * j + 1]) + a1[2 * j]) + a1[2 * j + 1]) / (TS)4;
        } else {
          lv[i][j] = (TA)a0[2 * j] + a0[2 * j + 1] + a1[2 * j] + a1[2 * j + 1];
        }
      }
    }
  } else {
#pragma unroll
    for (int i = 0; i < B / 2; ++i) {
      TS a0[B], a1[B];
      const TS* s0 = src + (long long)(r0 + 2 * i) * p.src_rp + c0;
      const TS* s1 = s0 + p.src_rp;
      if (full && (B * sizeof(TS)) % 16 == 0) {
#pragma unroll
        for (int v = 0; v < (int)(B * sizeof(TS) / 16); ++v) {
          reinterpret_cast<uint4*>(a0)[v] = reinterpret_cast<const uint4*>(s0)[v];
          reinterpret_cast<uint4*>(a1)[v] = reinterpret_cast<const uint4*>(s1)[v];
        }
      } else {
        const bool rok = r0 + 2 * i < 2 * p.hl[0];
#pragma unroll
        for (int j = 0; j < B; ++j) {
          const bool ok = rok && c0 + j < 2 * p.wl[0];
          a0[j] = ok ? s0[j] : (TS)0;
          a1[j] = ok ? s1[j] : (TS)0;
        }
      }
#pragma unroll
      for (int j = 0; j < B / 2; ++j) {
        if constexpr (FLT) {
          lv[i][j] = (((a0[2 * j] + a0[2 * j + 1]) + a1[2 * j]) + a1[2 * j + 1]) / (TS)4;
        } else {
          lv[i][j] = (TA)a0[2 * j] + a0[2 * j + 1] + a1[2 * j] + a1[2 * j + 1];
        }
      }
    }
  }
  // store level 1, then fold in place to the coarser levels
#pragma unroll
  for (int l = 1; l <= NL; ++l) {
    const int n = B >> l;  // samples per side at level l
    const int rl = by * n, cl = bx * n;
    TD* d = reinterpret_cast<TD*>(img ? p.dst_d[l - 1] : p.dst_r[l - 1]) + (long long)f * p.dst_fp[l - 1];
    if (l > 1) {
#pragma unroll
      for (int i = 0; i < B / 2; ++i)
#pragma unroll
        for (int j = 0; j < B / 2; ++j)
          if (i < n && j < n) {
            if constexpr (FLT) {
              lv[i][j] = (((lv[2 * i][2 * j] + lv[2 * i][2 * j + 1]) + lv[2 * i + 1][2 * j]) + lv[2 * i + 1][2 * j + 1]) / (TS)4;
            } else {
              lv[i][j] = lv[2 * i][2 * j] + lv[2 * i][2 * j + 1] + lv[2 * i + 1][2 * j] + lv[2 * i + 1][2 * j + 1];
            }
          }
    }
    const bool whole = rl + n <= p.hl[l - 1] && cl + n <= p.wl[l - 1];
#pragma unroll
    for (int i = 0; i < B / 2; ++i) {
      if (i < n && rl + i < p.hl[l - 1]) {
        TD* row = d + (long long)(rl + i) * p.dst_rp[l - 1] + cl;
        if (whole) {
          // n samples of this row are contiguous and n*sizeof(TD)-aligned: one vector store
          __align__(16) TD v[B / 2];
#pragma unroll
          for (int j = 0; j < B / 2; ++j) v[j] = (TD)lv[i][j];
          const int bytes = n * (int)sizeof(TD);
          if (bytes >= 16) {
#pragma unroll
            for (int q = 0; q < (B / 2) * (int)sizeof(TD) / 16; ++q)
              if (q * 16 < bytes) reinterpret_cast<uint4*>(row)[q] = reinterpret_cast<const uint4*>(v)[q];
          } else if (bytes == 8) {
            *reinterpret_cast<uint2*>(row) = *reinterpret_cast<const uint2*>(v);
          } else if (bytes == 4) {
            *reinterpret_cast<uint32_t*>(row) = *reinterpret_cast<const uint32_t*>(v);
          } else {
#pragma unroll
            for (int j = 0; j < B / 2; ++j)
              if (j < n) row[j] = v[j];
          }
        } else {
#pragma unroll
          for (int j = 0; j < B / 2; ++j)
            if (j < n && cl + j < p.wl[l - 1]) row[j] = (TD)lv[i][j];
        }
      }
    }
  }
}

template <typename TS, typename TD>
static int pyr_launch(const PyramidArgs& p, int nl, int n, cudaStream_t st) {
  const int B = 1 << nl;
  dim3 block(128);
  dim3 grid(((2 * p.wl[0] + B - 1) / B + 127) / 128, (2 * p.hl[0] + B - 1) / B, 2 * n);
  switch (nl) {
    case 1: pyramid_kernel<TS, TD, 1><<<grid, block, 0, st>>>(p); break;
    case 2: pyramid_kernel<TS, TD, 2><<<grid, block, 0, st>>>(p); break;
    case 3: pyramid_kernel<TS, TD, 3><<<grid, block, 0, st>>>(p); break;
    case 4: pyramid_kernel<TS, TD, 4><<<grid, block, 0, st>>>(p); break;
    default: return SSK_E_ARG;
  }
  note_launch();
  return cudaGetLastError() == cudaSuccess ? SSK_OK : SSK_E_CUDA;
}

int launch_pyramid(const PyramidArgs& p, int src_dtype, int dst_dtype, int nl, int n, cudaStream_t st) {
  if (nl < 1 || nl > GS_MAX_LEVELS || 2 * n > 65535) return SSK_E_ARG;
  if (src_dtype == SSK_U8 && dst_dtype == SSK_U16) return pyr_launch<uint8_t, uint16_t>(p, nl, n, st);
  if (src_dtype == SSK_U8 && dst_dtype == SSK_U32) return pyr_launch<uint8_t, uint32_t>(p, nl, n, st);
  if (src_dtype == SSK_U16 && dst_dtype == SSK_U16) return pyr_launch<uint16_t, uint16_t>(p, nl, n, st);
  if (src_dtype == SSK_U16 && dst_dtype == SSK_U32) return pyr_launch<uint16_t, uint32_t>(p, nl, n, st);
  if (src_dtype == SSK_U32 && dst_dtype == SSK_U32) return pyr_launch<uint32_t, uint32_t>(p, nl, n, st);
  if (src_dtype == SSK_F32 && dst_dtype == SSK_F32) return pyr_launch<float, float>(p, nl, n, st);
  if (src_dtype == SSK_F64 && dst_dtype == SSK_F64) return pyr_launch<double, double>(p, nl, n, st);
  return SSK_E_ARG;
}

// ---------------------------------------------------------------------------
// MS-SSIM finalize: one warp per frame folds every level's partials (fixed
// order), writes mean(cs) below the coarsest level / mean(l*cs) at it, the
// optional level-0 SSIM sums, and the exponent-weighted combination
// (combine_scale_scores, src/multiscale.py:62-74: product of max(s, 0)^e, or
// the normalised sum).
// ---------------------------------------------------------------------------
__global__ void msssim_finalize_kernel(const __grid_constant__ FinalizeArgs a) {
  // one block per frame: warp l folds level l (in parallel, same lane-strided order as a
  // single warp would), warps levels..levels+2 the level-0 SSIM sums; thread 0 combines
  // the per-level terms in level order
  __shared__ double s_term[SSK_MAX_SCALES];
  const int f = blockIdx.x;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (w < a.levels) {
    const int l = w;
    const double* p = a.partials[l] + (long long)f * a.nparts[l] * 3;
    const int comp = (l == a.levels - 1) ? 0 : 2;
    double s = 0.0;
    for (int i = lane; i < a.nparts[l]; i += 32) s += p[(long long)i * 3 + comp];
    s = warp_sum(s);
    if (lane == 0) {
      const double mean = __ddiv_rn(s, a.count[l]);
      a.level_means[(long long)f * a.levels + l] = mean;
      s_term[l] = a.aggregation == 2 ? a.exps[l] * mean : pow(fmax(mean, 0.0), a.exps[l]);
    }
  } else if (a.ssim_sums && w < a.levels + 3) {
    const int c = w - a.levels;
    const double* p = a.partials[0] + (long long)f * a.nparts[0] * 3;
    double t = 0.0;
    for (int i = lane; i < a.nparts[0]; i += 32) t += p[(long long)i * 3 + c];
    t = warp_sum(t);
    if (lane == 0) a.ssim_sums[(long long)f * 3 + c] = __ddiv_rn(t, a.count[0]);
  }
  __syncthreads();
  if (threadIdx.x == 0 && a.scores && a.aggregation != 0) {
    double combined = a.aggregation == 2 ? 0.0 : 1.0;
    for (int l = 0; l < a.levels; ++l) combined = a.aggregation == 2 ? combined + s_term[l] : combined * s_term[l];
    a.scores[f] = combined;
  }
}

int launch_msssim_finalize(const FinalizeArgs& a, cudaStream_t st) {
  if (a.n < 1) return SSK_OK;
  if (a.levels < 1 || a.levels > SSK_MAX_SCALES) return SSK_E_ARG;
  msssim_finalize_kernel<<<a.n, 32 * (a.levels + 3), 0, st>>>(a);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? SSK_OK : SSK_E_CUDA;
}

}  // namespace ssk

// ---------------------------------------------------------------------------
// Elementwise map arithmetic of the public API (off the throughput path, where it is
// fused into K1 / K2): stats_from_sums (src/stats.py:185-202), term_maps_from_stats
// (src/ssim.py:31-46) and the per-frame means.  fp64 with IEEE-rounded intrinsics in the
// reference's operation order (no FMA contraction), so the results are bit-identical to
// numpy's evaluation of the same expressions.
// ---------------------------------------------------------------------------
namespace ssk {
namespace {

__global__ void stats_from_sums_kernel(const double* __restrict__ s1, const double* __restrict__ s2,
                                       const double* __restrict__ q1, const double* __restrict__ q2,
                                       const double* __restrict__ p12, long long count, double area,
                                       double* __restrict__ out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count;
       i += (long long)gridDim.x * blockDim.x) {
    const double mu1 = __ddiv_rn(s1[i], area), mu2 = __ddiv_rn(s2[i], area);
    out[i] = mu1;
    out[count + i] = mu2;
    out[2 * count + i] = fmax(__dsub_rn(__ddiv_rn(q1[i], area), __dmul_rn(mu1, mu1)), 0.0);
    out[3 * count + i] = fmax(__dsub_rn(__ddiv_rn(q2[i], area), __dmul_rn(mu2, mu2)), 0.0);
    out[4 * count + i] = __dsub_rn(__ddiv_rn(p12[i], area), __dmul_rn(mu1, mu2));
  }
}

__global__ void term_maps_kernel(const double* __restrict__ mu1, const double* __restrict__ mu2,
                                 const double* __restrict__ var1, const double* __restrict__ var2,
                                 const double* __restrict__ cov, long long count, double c1, double c2,
                                 double* __restrict__ out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count;
       i += (long long)gridDim.x * blockDim.x) {
    const double m1 = mu1[i], m2 = mu2[i];
    // l = (2.0 * mu1 * mu2 + c1) / (mu1 * mu1 + mu2 * mu2 + c1), numpy's left-to-right order
    const double l = __ddiv_rn(__dadd_rn(__dmul_rn(__dmul_rn(2.0, m1), m2), c1),
                               __dadd_rn(__dadd_rn(__dmul_rn(m1, m1), __dmul_rn(m2, m2)), c1));
    const double cs = __ddiv_rn(__dadd_rn(__dmul_rn(2.0, cov[i]), c2), __dadd_rn(__dadd_rn(var1[i], var2[i]), c2));
    out[i] = l;
    out[count + i] = cs;
    out[2 * count + i] = __dmul_rn(l, cs);
  }
}

__global__ void divide_kernel(const double* __restrict__ x, long long count, double divisor, double* __restrict__ out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count;
       i += (long long)gridDim.x * blockDim.x)
    out[i] = __ddiv_rn(x[i], divisor);
}

dim3 ew_grid(long long count) {
  long long b = (count + 255) / 256;
  return dim3((unsigned)std::max(1LL, std::min(b, 148LL * 16)));
}

}  // namespace

int launch_stats_from_sums(const double* s1, const double* s2, const double* q1, const double* q2,
                           const double* p12, long long count, double area, double* out, cudaStream_t st) {
  if (count < 1) return SSK_OK;
  stats_from_sums_kernel<<<ew_grid(count), 256, 0, st>>>(s1, s2, q1, q2, p12, count, area, out);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? SSK_OK : SSK_E_CUDA;
}

int launch_term_maps(const double* mu1, const double* mu2, const double* var1, const double* var2,
                     const double* cov, long long count, double c1, double c2, double* out, cudaStream_t st) {
  if (count < 1) return SSK_OK;
  term_maps_kernel<<<ew_grid(count), 256, 0, st>>>(mu1, mu2, var1, var2, cov, count, c1, c2, out);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? SSK_OK : SSK_E_CUDA;
}

int launch_divide(const double* x, long long count, double divisor, double* out, cudaStream_t st) {
  if (count < 1) return SSK_OK;
  divide_kernel<<<ew_grid(count), 256, 0, st>>>(x, count, divisor, out);
  note_launch();
  return cudaGetLastError() == cudaSuccess ? SSK_OK : SSK_E_CUDA;
}

}  // namespace ssk
