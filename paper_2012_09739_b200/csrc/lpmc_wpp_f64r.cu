// Warp-per-path instances for the ArithF64Round bar arithmetic (see wpp_kernel in
// lpmc_level.cuh).  One translation unit per arithmetic, built in parallel.
#include "lpmc_level.cuh"

namespace lpmc_b200 {

cudaError_t launch_wpp_f64r(const LevelArgs& A, bool kahan, void* stream) {
  return dev::launch_level_wpp<dev::ArithF64Round>(A, kahan, static_cast<cudaStream_t>(stream));
}

cudaError_t configure_wpp_f64r() {
  cudaError_t e = math::upload_math_constants();  // this unit's own constant block
  if (e == cudaSuccess) e = dev::configure_wpp<dev::ArithF64Round>();
  return e;
}

}  // namespace lpmc_b200
