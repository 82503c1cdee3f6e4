// Level-kernel instances for the ArithF32 bar arithmetic (see lpmc_level.cuh).
// One translation unit per arithmetic so the build compiles them in parallel.
#include "lpmc_level.cuh"

namespace lpmc_b200 {

cudaError_t launch_level_f32(const LevelArgs& A, bool kahan, bool dump, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  return dev::launch_level<dev::ArithF32>(A, kahan, dump, s);
}

cudaError_t configure_level_f32() {
  cudaError_t e = math::upload_math_constants();
  if (e == cudaSuccess) e = dev::configure_level<dev::ArithF32>();
  return e;
}

}  // namespace lpmc_b200
