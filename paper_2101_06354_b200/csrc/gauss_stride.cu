// Dispatch of the strided Gaussian score kernel (K1s, gauss_stride.cuh); the kernels are
// instantiated per stride in gauss_stride_s{2..8}.cu so nvcc compiles them in parallel.
// Strides above 8 keep K1 with anchor masking.
#include "common.cuh"
#include "kernels.h"

namespace ssk {
int launch_gauss_stride_s2(const GaussArgs& a, dim3 grid, int k, cudaStream_t st);
int launch_gauss_stride_s3(const GaussArgs& a, dim3 grid, int k, cudaStream_t st);
int launch_gauss_stride_s4(const GaussArgs& a, dim3 grid, int k, cudaStream_t st);
int launch_gauss_stride_s5(const GaussArgs& a, dim3 grid, int k, cudaStream_t st);
int launch_gauss_stride_s6(const GaussArgs& a, dim3 grid, int k, cudaStream_t st);
int launch_gauss_stride_s7(const GaussArgs& a, dim3 grid, int k, cudaStream_t st);
int launch_gauss_stride_s8(const GaussArgs& a, dim3 grid, int k, cudaStream_t st);
int gauss_stride_twa_s2(int k, int es);
int gauss_stride_twa_s3(int k, int es);
int gauss_stride_twa_s4(int k, int es);
int gauss_stride_twa_s5(int k, int es);
int gauss_stride_twa_s6(int k, int es);
int gauss_stride_twa_s7(int k, int es);
int gauss_stride_twa_s8(int k, int es);

int gauss_stride_twa(int k, int s, int es) {
  switch (s) {
    case 2: return gauss_stride_twa_s2(k, es);
    case 3: return gauss_stride_twa_s3(k, es);
    case 4: return gauss_stride_twa_s4(k, es);
    case 5: return gauss_stride_twa_s5(k, es);
    case 6: return gauss_stride_twa_s6(k, es);
    case 7: return gauss_stride_twa_s7(k, es);
    case 8: return gauss_stride_twa_s8(k, es);
    default: return 0;
  }
}

bool gauss_stride_supported(int dtype, int k, int s) {
  return (dtype == SSK_U8 || dtype == SSK_U16) && k >= 3 && k <= 31 && (k & 1) && s >= 2 && s <= 8;
}

int launch_gauss_stride(const GaussArgs& a, dim3 grid, int k, cudaStream_t st) {
  if (!gauss_stride_supported(a.dtype, k, a.stride)) return SSK_E_ARG;
  switch (a.stride) {
    case 2: return launch_gauss_stride_s2(a, grid, k, st);
    case 3: return launch_gauss_stride_s3(a, grid, k, st);
    case 4: return launch_gauss_stride_s4(a, grid, k, st);
    case 5: return launch_gauss_stride_s5(a, grid, k, st);
    case 6: return launch_gauss_stride_s6(a, grid, k, st);
    case 7: return launch_gauss_stride_s7(a, grid, k, st);
    case 8: return launch_gauss_stride_s8(a, grid, k, st);
    default: return SSK_E_ARG;
  }
}
}  // namespace ssk
