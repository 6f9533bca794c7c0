// Instantiations of the strided Gaussian score kernel for stride 7 (see gauss_stride.cuh).
#include "gauss_stride.cuh"

namespace ssk {
int launch_gauss_stride_s7(const GaussArgs& a, dim3 grid, int k, cudaStream_t st) {
  return gk::launch_stride_s<7>(a, grid, k, st);
}
int gauss_stride_twa_s7(int k, int es) {
  switch (k) {
#define C(K) case K: return es == 1 ? gk::sg_twa<K, 7, 1>() : gk::sg_twa<K, 7, 2>();
    C(3) C(5) C(7) C(9) C(11) C(13) C(15) C(17) C(19) C(21) C(23) C(25) C(27) C(29) C(31)
#undef C
    default: return 0;
  }
}
}  // namespace ssk
