// Instantiations of the fused Gaussian SSIM kernel for u8 samples (see gauss_ssim.cuh).
#include "gauss_ssim.cuh"

namespace ssk {
int launch_gauss_u8(const GaussArgs& a, dim3 grid, int k, cudaStream_t st) {
  return gk::launch_dtype<uint8_t>(a, grid, k, st);
}
int launch_gauss_levels_u8(const GaussLevels& p, dim3 grid, int k, cudaStream_t st) {
  return gk::launch_levels_dtype<uint8_t>(p, grid, k, st);
}
}  // namespace ssk
