// Instantiations of the fused Gaussian SSIM kernel for f32 samples (see gauss_ssim.cuh).
#include "gauss_ssim.cuh"

namespace ssk {
int launch_gauss_f32(const GaussArgs& a, dim3 grid, int k, cudaStream_t st) {
  return gk::launch_dtype<float>(a, grid, k, st);
}
int launch_gauss_levels_f32(const GaussLevels& p, dim3 grid, int k, cudaStream_t st) {
  return gk::launch_levels_dtype<float>(p, grid, k, st);
}
}  // namespace ssk
