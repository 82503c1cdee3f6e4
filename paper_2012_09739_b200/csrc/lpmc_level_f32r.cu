// Level-kernel instances for the ArithF32Round bar arithmetic (see lpmc_level.cuh).
// One translation unit per arithmetic so the build compiles them in parallel.
#include "lpmc_level.cuh"

namespace lpmc_b200 {

cudaError_t launch_level_f32r(const LevelArgs& A, bool kahan, bool dump, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  return dev::launch_level<dev::ArithF32Round>(A, kahan, dump, s);
}

cudaError_t configure_level_f32r() {
  cudaError_t e = math::upload_math_constants();
  if (e == cudaSuccess) e = dev::configure_level<dev::ArithF32Round>();
  return e;
}

}  // namespace lpmc_b200
