// Warp-per-path instances for the ArithF32 bar arithmetic (see wpp_kernel in
// lpmc_level.cuh).  One translation unit per arithmetic, built in parallel.
#include "lpmc_level.cuh"

namespace lpmc_b200 {

cudaError_t launch_wpp_f32(const LevelArgs& A, bool kahan, void* stream) {
  return dev::launch_level_wpp<dev::ArithF32>(A, kahan, static_cast<cudaStream_t>(stream));
}

cudaError_t configure_wpp_f32() {
  cudaError_t e = math::upload_math_constants();  // this unit's own constant block
  if (e == cudaSuccess) e = dev::configure_wpp<dev::ArithF32>();
  return e;
}

}  // namespace lpmc_b200
