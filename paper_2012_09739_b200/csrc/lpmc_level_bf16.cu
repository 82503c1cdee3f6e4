// Level-kernel instances for the ArithBf16 bar arithmetic: the reference's
// m = 7 legs on native bfloat16 (lpmc_device.cuh).  Production launches in
// the fast exact-Gaussian mode; suspect paths are replayed in the
// fp32-carried emulation inside the same kernel.
#include "lpmc_level.cuh"

namespace lpmc_b200 {

namespace {
template <bool KAHAN, int LEGS>
cudaError_t launch_tab(const LevelArgs& A, cudaStream_t s) {
  if (A.table == nullptr)
    return dev::launch_one<dev::ArithBf16, KAHAN, LEGS, dev::kTabNone, false, dev::kZFast>(A, s);
  if (A.dyadic && A.table_simple && A.degree == 1)
    return dev::launch_one<dev::ArithBf16, KAHAN, LEGS, dev::kTabDyadicLinear, false,
                           dev::kZFast>(A, s);
  return dev::launch_one<dev::ArithBf16, KAHAN, LEGS, dev::kTabGeneric, false, dev::kZFast>(A, s);
}

template <bool KAHAN>
cudaError_t launch_kahan(const LevelArgs& A, cudaStream_t s) {
  if (A.legs == 2) return launch_tab<KAHAN, 2>(A, s);
  if (A.legs == 4) return launch_tab<KAHAN, 4>(A, s);
  return launch_tab<KAHAN, 3>(A, s);
}

template <bool KAHAN, int LEGS>
cudaError_t configure_legs() {
  cudaError_t e = dev::configure_tabs<dev::ArithBf16, KAHAN, LEGS, false, dev::kZFast>();
  return e;
}
}  // namespace

cudaError_t launch_level_bf16(const LevelArgs& A, bool kahan, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  return kahan ? launch_kahan<true>(A, s) : launch_kahan<false>(A, s);
}

cudaError_t configure_level_bf16() {
  cudaError_t e = math::upload_math_constants();
  auto acc = [&](cudaError_t x) {
    if (e == cudaSuccess) e = x;
  };
  acc(configure_legs<false, 2>());
  acc(configure_legs<true, 2>());
  acc(configure_legs<false, 3>());
  acc(configure_legs<true, 3>());
  acc(configure_legs<false, 4>());
  acc(configure_legs<true, 4>());
  return e;
}

}  // namespace lpmc_b200
