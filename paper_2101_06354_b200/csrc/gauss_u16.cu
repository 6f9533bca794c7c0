// Instantiations of the fused Gaussian SSIM kernel for u16 samples (see gauss_ssim.cuh).
#include "gauss_ssim.cuh"

namespace ssk {
int launch_gauss_u16(const GaussArgs& a, dim3 grid, int k, cudaStream_t st) {
  return gk::launch_dtype<uint16_t>(a, grid, k, st);
}
int launch_gauss_levels_u16(const GaussLevels& p, dim3 grid, int k, cudaStream_t st) {
  return gk::launch_levels_dtype<uint16_t>(p, grid, k, st);
}
}  // namespace ssk
