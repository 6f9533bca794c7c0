/* A host program that uses the engine through the C ABI only (no Python, no torch): the
 * integration a non-Python ssimkit host would write against include/ssimk.h.
 *
 *   ssim_cli <h> <w> <ref.u8> <dist.u8> [sigma levels]
 *
 * Reads two raw 8-bit planes, uploads them with the CUDA runtime, and prints one line
 *   ssim <mean q> <mean l> <mean cs> msssim <score>
 * computed by ssk_ssim (Gaussian window from sigma, library-built taps) and ssk_msssim
 * (product of the standard exponents).  Exit status != 0 on any error (message on stderr).
 */
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "ssimk.h"

#define CHECK_CUDA(x)                                                       \
  do {                                                                      \
    cudaError_t e_ = (x);                                                   \
    if (e_ != cudaSuccess) {                                                \
      fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e_));              \
      return 2;                                                             \
    }                                                                       \
  } while (0)
#define CHECK_SSK(x)                                                        \
  do {                                                                      \
    int r_ = (x);                                                           \
    if (r_ != SSK_OK) {                                                     \
      fprintf(stderr, "%s: %s (%d)\n", #x, ssk_strerror(r_), r_);           \
      return 3;                                                             \
    }                                                                       \
  } while (0)

static unsigned char* read_plane(const char* path, size_t bytes) {
  FILE* f = fopen(path, "rb");
  if (!f) return NULL;
  unsigned char* buf = (unsigned char*)malloc(bytes);
  size_t got = buf ? fread(buf, 1, bytes, f) : 0;
  fclose(f);
  if (got != bytes) {
    free(buf);
    return NULL;
  }
  return buf;
}

int main(int argc, char** argv) {
  if (argc < 5) {
    fprintf(stderr, "usage: %s h w ref.u8 dist.u8 [sigma levels]\n", argv[0]);
    return 1;
  }
  const int h = atoi(argv[1]), w = atoi(argv[2]);
  const double sigma = argc > 5 ? atof(argv[5]) : 1.5;
  const int levels = argc > 6 ? atoi(argv[6]) : 5;
  if (ssk_abi_version() != SSK_ABI_VERSION) {
    fprintf(stderr, "ABI mismatch: library %d, header %d\n", ssk_abi_version(), SSK_ABI_VERSION);
    return 1;
  }
  unsigned char* a = read_plane(argv[3], (size_t)h * w);
  unsigned char* b = read_plane(argv[4], (size_t)h * w);
  if (!a || !b) {
    fprintf(stderr, "cannot read %d x %d planes\n", h, w);
    return 1;
  }
  /* 16-byte aligned row pitch, as the ABI requires */
  const int64_t pitch = ((int64_t)w + 15) / 16 * 16;
  unsigned char *d_ref, *d_dist;
  CHECK_CUDA(cudaMalloc((void**)&d_ref, (size_t)pitch * h));
  CHECK_CUDA(cudaMalloc((void**)&d_dist, (size_t)pitch * h));
  CHECK_CUDA(cudaMemcpy2D(d_ref, pitch, a, w, w, h, cudaMemcpyHostToDevice));
  CHECK_CUDA(cudaMemcpy2D(d_dist, pitch, b, w, w, h, cudaMemcpyHostToDevice));

  ssk_planes p;
  memset(&p, 0, sizeof p);
  p.ref = d_ref;
  p.dist = d_dist;
  p.dtype = SSK_U8;
  p.n = 1;
  p.h = h;
  p.w = w;
  p.bit_depth = 8;
  p.row_pitch = pitch;
  p.frame_pitch = pitch * h;

  ssk_window win;
  memset(&win, 0, sizeof win); /* taps all zero: the library builds them from sigma */
  win.shape = SSK_GAUSS;
  win.k = 2 * (int)(3.0 * sigma + 0.999999999) + 1; /* default_gaussian_size: 2 ceil(3 sigma) + 1 */
  win.stride = 1;
  win.sigma = sigma;
  win.c1 = (0.01 * 255.0) * (0.01 * 255.0);
  win.c2 = (0.03 * 255.0) * (0.03 * 255.0);

  const size_t ws_bytes = ssk_ssim_workspace_bytes(&p, &win);
  const size_t ms_bytes = ssk_msssim_workspace_bytes(&p, &win, levels);
  if (!ws_bytes || !ms_bytes) {
    fprintf(stderr, "workspace query failed (window %d does not fit %d levels of %dx%d?)\n", win.k, levels, w, h);
    return 3;
  }
  void* d_ws;
  double *d_sums, *d_means, *d_score;
  CHECK_CUDA(cudaMalloc(&d_ws, ws_bytes > ms_bytes ? ws_bytes : ms_bytes));
  CHECK_CUDA(cudaMalloc((void**)&d_sums, 4 * sizeof(double)));
  CHECK_CUDA(cudaMalloc((void**)&d_means, 16 * sizeof(double)));
  CHECK_CUDA(cudaMalloc((void**)&d_score, sizeof(double)));

  CHECK_SSK(ssk_ssim(&p, &win, SSK_WANT_Q | SSK_WANT_L | SSK_WANT_CS, d_sums, NULL, d_ws, ws_bytes, NULL));
  static const double exps[5] = {0.0448, 0.2856, 0.3001, 0.2363, 0.1333};
  CHECK_SSK(ssk_msssim(&p, &win, levels, exps, 1 /* product */, d_means, d_score, NULL, d_ws,
                       ws_bytes > ms_bytes ? ws_bytes : ms_bytes, NULL));
  double sums[3], score;
  CHECK_CUDA(cudaMemcpy(sums, d_sums, sizeof sums, cudaMemcpyDeviceToHost));
  CHECK_CUDA(cudaMemcpy(&score, d_score, sizeof score, cudaMemcpyDeviceToHost));
  const double count = (double)(h - win.k + 1) * (double)(w - win.k + 1);
  printf("ssim %.17g %.17g %.17g msssim %.17g\n", sums[0] / count, sums[1] / count, sums[2] / count, score);
  cudaFree(d_ref);
  cudaFree(d_dist);
  cudaFree(d_ws);
  cudaFree(d_sums);
  cudaFree(d_means);
  cudaFree(d_score);
  free(a);
  free(b);
  return 0;
}
