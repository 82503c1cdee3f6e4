// The per-step rounding-residual probe: step_error_probe
// (proj/include/lpmc/sde.hpp:289-344) on the device.
//
// One path per thread, paths 0, 1, ... of the seed (path_base 0), 2^level
// steps each except the last path, which stops when the sample count is
// reached (sde.hpp:313-336).  Per step, in the target precision, the bar
// arithmetic of the level kernel (same policies, same operation order):
//   a = R(mu) (x) x, b = R(sigma) (x) x, drift = a (x) dt,
//   diff = (b (x) sqrt_dt) (x) z, inner = drift (+) diff, next = x (+) inner
// and in binary64 the residuals eta' = inner - (drift + diff), eta = next -
// (x + inner).  Each thread sums its own residuals in step order; a block
// sums its 256 threads in a fixed tree; the host adds the block sums in
// block order.  The reference adds all samples in one sequential chain, so
// the means agree to the summation-order bound (tests: <= 2 n eps sum|.|).
#include "lpmc_level.cuh"

namespace lpmc_b200 {
namespace dev {

constexpr int kProbeThreads = 256;

template <class Arith, bool APPROX>
__global__ void __launch_bounds__(kProbeThreads)
    step_error_kernel(const __grid_constant__ LevelArgs A, uint64_t last_steps,
                      double* __restrict__ block_sums) {
  using T = typename Arith::T;
  extern __shared__ __align__(16) double s_table[];
  __shared__ __align__(16) double s_math[APPROX ? 2 : kMathWords];
  __shared__ double s_warp[4][kProbeThreads / 32];
  if constexpr (!APPROX) stage_math(s_math);
  TableView tab{};
  if constexpr (APPROX) {
    for (int i = threadIdx.x; i < A.table_words; i += blockDim.x) s_table[i] = A.table[i];
    tab = TableView{s_table, A.table_stride, A.K, A.degree, A.dyadic, A.table_simple, A.tail};
  }
  __syncthreads();

  const uint64_t path = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const bool valid = path < A.n_paths;
  const uint64_t n_steps = 1ull << A.level;
  const uint64_t steps = !valid ? 0 : (path + 1 == A.n_paths ? last_steps : n_steps);

  const Arith ar(A);
  typename Arith::Range range;
  uint64_t kc = path_key(A.seed_key, A.path_base + (valid ? path : 0)) + A.counter0 * kCounterStep;
  const T mu_l = ar.c(A.mu_l, A.h_mu), sg_l = ar.c(A.sigma_l, A.h_sigma);
  const T dt_l = ar.c(A.dtf_l, A.h_dtf), sdt_l = ar.c(A.sdtf_l, A.h_sdtf);
  T x = ar.c(A.x0_l, A.h_x0);
  double se = 0.0, sae = 0.0, sep = 0.0, saep = 0.0;
  uint64_t fk = kNoFail;
  // every lane walks n_steps draws (the warp-collective tail pass of the
  // exact transform wants converged lanes); lanes past their own count
  // neither accumulate nor update
  for (uint64_t n = 0; n < n_steps; ++n) {
    const bool on = n < steps;
    const uint64_t b = next_draw(kc);
    const double u = uniform_of(b);
    double z;
    if constexpr (APPROX) {
      z = approx_inv<true>(tab, u);
    } else if (A.exact_z == kZGlibc) {  // the reference's Z bit for bit
      const double uu[1] = {u};
      double zz[1];
      glibc::inv_cdf_multi<1>(uu, zz, s_math);
      z = zz[0];
    } else {
      const double uu[1] = {u};
      double zz[1];
      math::phi_inv_multi<1>(uu, zz, math::FlatTab{s_math});
      z = zz[0];
    }
    const double zr[1] = {z};
    const T zb = ar.lift(zr);
    const T a = ar.mul(mu_l, x);
    const T bb = ar.mul(sg_l, x);
    const T drift = ar.mul(a, dt_l);
    const T diff = ar.mul(ar.mul(bb, sdt_l), zb);
    const T inner = ar.add(drift, diff);
    const T next = ar.add(x, inner);
    const double dd = ar.get(drift, 0), df = ar.get(diff, 0), di = ar.get(inner, 0);
    const double dx = ar.get(x, 0), dn = ar.get(next, 0);
    const double eta_p = __dsub_rn(di, __dadd_rn(dd, df));
    const double eta = __dsub_rn(dn, __dadd_rn(dx, di));
    if (on) {
      note_fail(fk, b == kTopDraw, n, kStageDraw);
      const uint32_t bad = ar.bad(zb) | ar.bad(a) | ar.bad(bb) | ar.bad(drift) | ar.bad(diff) |
                           ar.bad(inner) | ar.bad(next);
      note_fail(fk, bad != 0u, n, kStageBarFine);
      se = __dadd_rn(se, eta);
      sae = __dadd_rn(sae, fabs(eta));
      sep = __dadd_rn(sep, eta_p);
      saep = __dadd_rn(saep, fabs(eta_p));
      range.track(next);
      x = next;
    }
  }
  if (valid && fk != kNoFail) {
    const uint64_t n = fk >> 3;
    const uint32_t kind = (fk & 7u) == kStageDraw ? kKindU1 : kKindNonFinite;
    atomicMin(A.err_key, err_key_of(path, kind, n, A.err_step_bits));
  }
  if (valid && range.bad()) atomicOr(A.range_flag, 1u);

  // fixed tree: xor butterfly per warp, then over the 8 warp sums
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double v[4] = {se, sae, sep, saep};
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const double s = warp_sum(v[q], 16);
    if (lane == 0) s_warp[q][warp] = s;
  }
  __syncthreads();
  if (warp == 0) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const double g = warp_sum(lane < kProbeThreads / 32 ? s_warp[q][lane] : 0.0, 4);
      if (lane == 0) block_sums[4 * blockIdx.x + q] = g;
    }
  }
}

template <class Arith>
cudaError_t launch_probe(const LevelArgs& A, uint64_t last_steps, double* block_sums,
                         cudaStream_t s) {
  const unsigned blocks =
      static_cast<unsigned>((A.n_paths + kProbeThreads - 1) / kProbeThreads);
  if (A.table != nullptr) {
    const size_t smem = static_cast<size_t>(A.table_words) * sizeof(double);
    cudaError_t e = cudaFuncSetAttribute(step_error_kernel<Arith, true>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    step_error_kernel<Arith, true><<<blocks, kProbeThreads, smem, s>>>(A, last_steps, block_sums);
  } else {
    step_error_kernel<Arith, false><<<blocks, kProbeThreads, 0, s>>>(A, last_steps, block_sums);
  }
  return cudaGetLastError();
}

}  // namespace dev

cudaError_t launch_step_error(const LevelArgs& A, BarArith arith, uint64_t last_steps,
                              double* block_sums, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  switch (arith) {
    case BarArith::kCarrier: return dev::launch_probe<dev::ArithCarrier>(A, last_steps, block_sums, s);
    case BarArith::kF32: return dev::launch_probe<dev::ArithF32>(A, last_steps, block_sums, s);
    case BarArith::kF32Round: return dev::launch_probe<dev::ArithF32Round>(A, last_steps, block_sums, s);
    case BarArith::kF64Round: return dev::launch_probe<dev::ArithF64Round>(A, last_steps, block_sums, s);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t configure_probe() { return math::upload_math_constants(); }

}  // namespace lpmc_b200
