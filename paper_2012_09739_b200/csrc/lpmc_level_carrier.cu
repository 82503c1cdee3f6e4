// Level-kernel instances for the ArithCarrier bar arithmetic (see lpmc_level.cuh).
// One translation unit per arithmetic so the build compiles them in parallel.
#include "lpmc_level.cuh"

namespace lpmc_b200 {

cudaError_t launch_level_carrier(const LevelArgs& A, bool kahan, bool dump, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (A.legs == 1) {  // carrier legs only: precision, Kahan and table do not apply
    if (A.exact_z == dev::kZGlibc)
      return dump ? dev::launch_one<dev::ArithCarrier, false, 1, dev::kTabNone, true, dev::kZGlibc>(A, s)
                  : dev::launch_one<dev::ArithCarrier, false, 1, dev::kTabNone, false, dev::kZGlibc>(A, s);
    return dump ? dev::launch_one<dev::ArithCarrier, false, 1, dev::kTabNone, true, dev::kZFast>(A, s)
                : dev::launch_one<dev::ArithCarrier, false, 1, dev::kTabNone, false, dev::kZFast>(A, s);
  }
  return dev::launch_level<dev::ArithCarrier>(A, kahan, dump, s);
}

cudaError_t configure_level_carrier() {
  cudaError_t e = math::upload_math_constants();
  if (e == cudaSuccess) e = dev::configure_level<dev::ArithCarrier>();
  // the hat-only instances (LEGS == 1, launched above)
  if (e == cudaSuccess) e = dev::configure_hat_only<dev::ArithCarrier, false>();
  if (e == cudaSuccess) e = dev::configure_hat_only<dev::ArithCarrier, true>();
  return e;
}

}  // namespace lpmc_b200
