// Level-kernel instances for the ArithHalfScaled bar arithmetic: the
// reference's m = 10 legs on native binary16 with static power-of-two scales
// (lpmc_device.cuh).  Production launches only: no dump, fast exact
// Gaussians, a dyadic-linear table or none; paths that leave the native guard
// are replayed in the fp32-carried emulation inside the same kernel.
#include "lpmc_level.cuh"

namespace lpmc_b200 {

namespace {
template <bool KAHAN, int LEGS>
cudaError_t launch_legs(const LevelArgs& A, cudaStream_t s) {
  if (A.table == nullptr)
    return dev::launch_one<dev::ArithHalfScaled, KAHAN, LEGS, dev::kTabNone, false, dev::kZFast>(A, s);
  return dev::launch_one<dev::ArithHalfScaled, KAHAN, LEGS, dev::kTabDyadicLinear, false,
                         dev::kZFast>(A, s);
}

template <bool KAHAN>
cudaError_t launch_kahan(const LevelArgs& A, cudaStream_t s) {
  if (A.legs == 2) return launch_legs<KAHAN, 2>(A, s);
  if (A.legs == 4) return launch_legs<KAHAN, 4>(A, s);
  return launch_legs<KAHAN, 3>(A, s);
}

template <bool KAHAN, int LEGS, int TAB, bool PW>
cudaError_t configure_inst() {
  constexpr int kBytes = (dev::level_persistent<LEGS, TAB, dev::kZFast>() ? dev::kFastWords * 8 : 0) +
                         (kDyadicRecord * kDyadicRecords + dev::kRunCopyWords) * 8;
  return cudaFuncSetAttribute(
      dev::level_kernel<dev::ArithHalfScaled, KAHAN, LEGS, TAB, false, dev::kZFast, PW>,
      cudaFuncAttributeMaxDynamicSharedMemorySize, kBytes);
}
}  // namespace

cudaError_t launch_level_h16(const LevelArgs& A, bool kahan, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  return kahan ? launch_kahan<true>(A, s) : launch_kahan<false>(A, s);
}

cudaError_t configure_level_h16() {
  cudaError_t e = math::upload_math_constants();
  auto acc = [&](cudaError_t x) {
    if (e == cudaSuccess) e = x;
  };
  acc(configure_inst<false, 2, dev::kTabNone, false>());
  acc(configure_inst<true, 2, dev::kTabNone, false>());
  acc(configure_inst<false, 2, dev::kTabNone, true>());
  acc(configure_inst<true, 2, dev::kTabNone, true>());
  acc(configure_inst<false, 2, dev::kTabDyadicLinear, false>());
  acc(configure_inst<true, 2, dev::kTabDyadicLinear, false>());
  acc(configure_inst<false, 2, dev::kTabDyadicLinear, true>());
  acc(configure_inst<true, 2, dev::kTabDyadicLinear, true>());
  acc(configure_inst<false, 3, dev::kTabNone, false>());
  acc(configure_inst<true, 3, dev::kTabNone, false>());
  acc(configure_inst<false, 3, dev::kTabNone, true>());
  acc(configure_inst<true, 3, dev::kTabNone, true>());
  acc(configure_inst<false, 3, dev::kTabDyadicLinear, false>());
  acc(configure_inst<true, 3, dev::kTabDyadicLinear, false>());
  acc(configure_inst<false, 3, dev::kTabDyadicLinear, true>());
  acc(configure_inst<true, 3, dev::kTabDyadicLinear, true>());
  acc(configure_inst<false, 4, dev::kTabNone, false>());
  acc(configure_inst<true, 4, dev::kTabNone, false>());
  acc(configure_inst<false, 4, dev::kTabNone, true>());
  acc(configure_inst<true, 4, dev::kTabNone, true>());
  acc(configure_inst<false, 4, dev::kTabDyadicLinear, false>());
  acc(configure_inst<true, 4, dev::kTabDyadicLinear, false>());
  acc(configure_inst<false, 4, dev::kTabDyadicLinear, true>());
  acc(configure_inst<true, 4, dev::kTabDyadicLinear, true>());
  return e;
}

}  // namespace lpmc_b200
