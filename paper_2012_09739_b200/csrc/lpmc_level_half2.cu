// Level-kernel instances for the ArithHalf2 bar arithmetic (see lpmc_level.cuh).
// One translation unit per arithmetic so the build compiles them in parallel.
#include "lpmc_level.cuh"

namespace lpmc_b200 {

cudaError_t launch_level_half2(const LevelArgs& A, bool kahan, bool dump, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  return dev::launch_level<dev::ArithHalf2>(A, kahan, dump, s);
}

cudaError_t configure_level_half2() {
  cudaError_t e = math::upload_math_constants();
  if (e == cudaSuccess) e = dev::configure_level<dev::ArithHalf2>();
  return e;
}

}  // namespace lpmc_b200
