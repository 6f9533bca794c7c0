// Dtype dispatch of the fused Gaussian SSIM kernel (K1, gauss_ssim.cuh).
#include "common.cuh"
#include "kernels.h"

namespace ssk {
int launch_gauss(const GaussArgs& a, dim3 grid, int k, cudaStream_t st) {
  switch (a.dtype) {
    case SSK_U8: return launch_gauss_u8(a, grid, k, st);
    case SSK_U16: return launch_gauss_u16(a, grid, k, st);
    case SSK_U32: return launch_gauss_u32(a, grid, k, st);
    case SSK_F32: return launch_gauss_f32(a, grid, k, st);
    default: return SSK_E_ARG;
  }
}
int launch_gauss_levels_u8(const GaussLevels& p, dim3 grid, int k, cudaStream_t st);
int launch_gauss_levels_u16(const GaussLevels& p, dim3 grid, int k, cudaStream_t st);
int launch_gauss_levels_u32(const GaussLevels& p, dim3 grid, int k, cudaStream_t st);
int launch_gauss_levels_f32(const GaussLevels& p, dim3 grid, int k, cudaStream_t st);

int launch_gauss_levels(const GaussLevels& p, dim3 grid, int k, int dtype, cudaStream_t st) {
  switch (dtype) {
    case SSK_U8: return launch_gauss_levels_u8(p, grid, k, st);
    case SSK_U16: return launch_gauss_levels_u16(p, grid, k, st);
    case SSK_U32: return launch_gauss_levels_u32(p, grid, k, st);
    case SSK_F32: return launch_gauss_levels_f32(p, grid, k, st);
    default: return SSK_E_ARG;
  }
}
}  // namespace ssk
