// Instantiations of the fused Gaussian SSIM kernel for u32 samples (see gauss_ssim.cuh).
#include "gauss_ssim.cuh"

namespace ssk {
int launch_gauss_u32(const GaussArgs& a, dim3 grid, int k, cudaStream_t st) {
  return gk::launch_dtype<unsigned>(a, grid, k, st);
}
int launch_gauss_levels_u32(const GaussLevels& p, dim3 grid, int k, cudaStream_t st) {
  return gk::launch_levels_dtype<unsigned>(p, grid, k, st);
}
}  // namespace ssk
