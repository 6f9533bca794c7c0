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
}  // namespace ssk
