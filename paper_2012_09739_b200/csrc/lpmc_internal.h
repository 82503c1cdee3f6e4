// Internal interface between the host library (lpmc_host.cpp, plain C++) and
// the sm_100a kernels (lpmc_kernels.cu, lpmc_level_*.cu).  Not part of the
// public ABI.
#pragma once

#include <cstdint>

#ifdef __CUDACC__
#include <cuda_runtime.h>
#endif

namespace lpmc_b200 {

// Arithmetic of the low-precision ("bar") legs as the kernels implement it.
enum class BarArith : int {
  kCarrier = 0,   // m >= 52: binary64 ops (the reference's carrier)
  kF32 = 1,       // m == 23: native fp32 __f*_rn (bit-exact inside the guarded range)
  kF32Round = 2,  // m <= 10: fp32 op + RNE to m+1 bits (innocuous double rounding)
  kF64Round = 3,  // any m < 52: binary64 op + integer RNE to m+1 bits (exact emulation)
  kHalf2 = 4      // native IEEE binary16, two paths per thread (__h*2_rn)
};

// Device table layouts (doubles):
//   dyadic (K <= 32): K records {3 - 2^(j+3), 2^(j+3), c0, c1, c2, c3} (kDyadicRecord),
//            then tail records {0, 0, tail, 0, 0, 0} up to kDyadicRecords
//   general: K records {a_j, b_j - a_j, c0, c1} (degree 1) or {.., c2, c3}
//            (degree 3), then the v-thresholds T_1..T_{K-1}, T_tail, then
//            1 / step_w: at most kTableRows * K + 1 doubles
constexpr int kTableRows = 7;
constexpr int kDyadicRecord = 6;
// dyadic tables carry records j = 0..52 (K interval records, then tail
// records): j = floor(-log2 v) - 1 for every v = 1 - u' in [2^-53, 1/2]
constexpr int kDyadicRecords = 53;

#ifdef __CUDACC__
#define LPMC_KEY_HD __host__ __device__
#else
#define LPMC_KEY_HD
#endif

struct LevelArgs {
  uint64_t seed_key;   // mix64(seed + 0x9e37...) (uniform.hpp:23), hoisted per launch
  uint64_t path_base;  // global path index of local path 0
  uint64_t n_paths;    // paths of the whole run (local indices 0..n_paths-1)
  uint64_t batch0;     // first batch (256 paths) this launch covers
  uint64_t n_batches;  // batches in this launch
  int32_t level;
  int32_t legs;        // 1 hat, 2 bar, 3 both
  // carrier legs (sde.hpp:219-221)
  double mu, sigma, x0, dtf, sdtf, dtc;
  // bar-leg constants already rounded into the low precision (sde.hpp:222-224, :232)
  double mu_l, sigma_l, x0_l, dtf_l, sdtf_l, dtc_l;
  // IEEE binary16 bit patterns of the same constants (kHalf2 only)
  uint16_t h_mu, h_sigma, h_x0, h_dtf, h_sdtf, h_dtc;
  int32_t mantissa_bits;
  // approximation table (nullptr = exact inverse CDF for the bar legs)
  const double* table;
  int32_t K, degree, dyadic;
  int32_t table_stride;  // general layout: record width (4 or 6 doubles)
  int32_t table_words;   // doubles to stage into shared memory
  int32_t table_simple;  // every c0 != 0 and c2 = c3 = +0: no signed-zero fix-up
  double tail;
  // payoff on terminal values (extension)
  int32_t payoff;
  double strike;
  // outputs
  double* batch_acc;             // tree mode: n_batches x 3 x 5
  double* path_diff;             // sequential mode: slice paths x 2 (d_hat, d_bar)
  double* path_out;              // dump: n x 4
  double* z_out;                 // dump: n x 2^level
  unsigned long long* err_key;   // atomicMin: err_key_of(local path, kind, step, err_step_bits)
  unsigned int* range_flag;      // native bar legs left the guarded exponent range
  // exact Gaussians: LPMC_EXACT_Z_FAST / _GLIBC (last: the fields above keep
  // the offsets the kernels' 128-bit uniform constant loads were tuned for)
  int32_t exact_z;
  // packed-fp32 operands (-0, -0) and (-1, -1) as f32x2 bit patterns, passed
  // as parameters so that the kernels cannot see them as constants: ptxas
  // folds an f32x2 multiply and add with known constant operands into one
  // fused FFMA2, which would change the rounding (dev::ffma2).
  uint64_t f2_neg0 = 0x8000000080000000ull;
  uint64_t f2_neg1 = 0xbf800000bf800000ull;
  // bits of the step field of the failure key (err_step_bits_for(level))
  int32_t err_step_bits = 22;
  // first counter of every path's stream (lpmc_options::counter)
  uint64_t counter0 = 0;
  // native fp32 bar legs with power-of-two dt, 2dt, sqrt(dt) (host-proved):
  // the products mu dt, mu 2dt, sigma sqrt(dt), exact
  int32_t bar_pow2 = 0;
  double mu_dtf_l = 0.0, mu_dtc_l = 0.0, sg_sdt_l = 0.0;
  // the same products for the carrier legs (bar_pow2 also proves the
  // carrier's dt, 2dt, sqrt(dt) powers of two; step_hat_pw)
  double hat_mu_dtf = 0.0, hat_mu_dtc = 0.0, hat_sg_sdt = 0.0;
  // m = 10 legs on native binary16 with static scales (dev::ArithHalfScaled;
  // host-proved, hs_native = 1): binary16 bit patterns of the mantissas of
  // mu_l, sigma_l, sqrt_dt_l, of P1, P1c, P2, and 2^kz
  int32_t hs_native = 0;
  uint16_t hs_mu = 0, hs_sigma = 0, hs_sdt = 0, hs_p1 = 0, hs_p1c = 0, hs_p2 = 0;
  uint16_t hs_q1 = 0, hs_q2 = 0;  // Q1 Q2 = 1 / P2 (the Kahan compensation's scale)
  double hs_zscale = 1.0;
};

// Failure key: the path in the high bits (atomicMin finds the lowest failing
// path, the reference's serial order), then the failure kind (2 bits), then
// the step.  The step field has max(22, level) bits, so every step of a
// path fits; the host rejects runs whose path indices would not fit the rest
// (n_paths >= 2^(62 - bits): n_paths 2^level >= 2^62 fine steps).
constexpr int err_step_bits_for(int level) { return level > 22 ? level : 22; }
inline LPMC_KEY_HD unsigned long long err_key_of(uint64_t path, uint32_t kind, uint64_t step,
                                                 int bits) {
  return (path << (bits + 2)) | (static_cast<uint64_t>(kind) << bits) | step;
}

// Production launches of the m = 10 emulation that run on native binary16
// (dev::ArithHalfScaled): the host proved the scales (hs_native), no
// dump, fast exact Gaussians, a dyadic-linear table or none.  Everything
// else, and every path that leaves the native guard, runs the fp32-carried
// emulation.
inline bool use_native_half(const LevelArgs& A, bool kahan, bool dump) {
  (void)kahan;  // with or without Kahan compensation
  return A.hs_native != 0 && !dump && A.exact_z == 0 && A.legs != 1 &&
         (A.table == nullptr || (A.dyadic != 0 && A.table_simple != 0 && A.degree == 1));
}

// Production launches of the m = 7 emulation that run on native bfloat16
// (dev::ArithBf16): fast exact Gaussians, no dump.  bfloat16 has fp32's
// exponent range, so the native fp32 range guard is the whole condition.
inline bool use_native_bf16(const LevelArgs& A, bool dump) {
  return A.mantissa_bits == 7 && !dump && A.exact_z == 0 && A.legs != 1;
}

struct LaunchResult {
  int cuda_error;  // cudaError_t
  int kernels;     // kernels enqueued
};

// Enqueue the path kernel for one launch slice; dump selects the instance
// that writes path_out / z_out.
LaunchResult launch_paths(const LevelArgs& args, BarArith arith, bool kahan, bool dump,
                          void* stream);
// Chunk tree over batch accumulators: chunks [0, n_chunks) of batches
// [0, n_batches) in `batch_acc` -> chunk_acc (n_chunks x 3 x 5).
LaunchResult launch_chunk_reduce(const double* batch_acc, uint64_t n_batches, uint64_t n_chunks,
                                 double* chunk_acc, void* stream);
// Reference-order batch accumulation of per-path (d_hat, d_bar).
LaunchResult launch_sequential_batches(const double* path_diff, uint64_t n_paths,
                                       double* batch_acc, void* stream);
// Exact / approximate inverse CDF of host-given uniforms (parity hooks).
// op 0 exact, 1 approximate (table), 2 libdevice reference formula, 3 erfc core.
LaunchResult launch_inv_cdf(const double* u, uint64_t n, const double* table, int K, int degree,
                            int dyadic, int stride, int simple, double tail, int op, double* out,
                            void* stream);
// run_density_report's histogram (experiments.hpp:276-285); key = the path
// key of (seed, path 0); table == nullptr: exact transform.
LaunchResult launch_density(uint64_t key, uint64_t n, const double* table, int table_words,
                            int K, int degree, int dyadic, int stride, int simple, double tail,
                            double z_max, double width, int n_bins, int exact_z,
                            unsigned long long* bins, unsigned long long* top_index,
                            void* stream);
// The warp-per-path schedule (wpp_kernel, lpmc_level.cuh) for one launch
// slice: per-path (d_hat, d_bar) into args.path_diff (slice-relative).
// Not for the IEEE half2 arithmetic (two paths per thread).
LaunchResult launch_paths_wpp(const LevelArgs& args, BarArith arith, bool kahan, void* stream);
// The fused kernel's batch tree over per-path differences: batch b of
// path_diff (n_paths slice paths) -> batch_acc + 15 b.
LaunchResult launch_path_batches(const double* path_diff, uint64_t n_paths, double* batch_acc,
                                 void* stream);
// Upload constants and set kernel attributes on the current device.
int configure_kernels();
// Lane-op rates on the current device: fp64 FMA, fp32 FMA, half2 HFMA2
// (per half lane), 64-bit integer multiply-add.  Returns cudaError_t.
int measure_pipe_peaks(double* out4);

#ifdef __CUDACC__
// per-arithmetic translation units (lpmc_level_*.cu)
cudaError_t launch_level_carrier(const LevelArgs& A, bool kahan, bool dump, void* stream);
cudaError_t launch_level_f32(const LevelArgs& A, bool kahan, bool dump, void* stream);
cudaError_t launch_level_f32r(const LevelArgs& A, bool kahan, bool dump, void* stream);
cudaError_t launch_level_f64r(const LevelArgs& A, bool kahan, bool dump, void* stream);
cudaError_t launch_level_half2(const LevelArgs& A, bool kahan, bool dump, void* stream);
cudaError_t launch_level_h16(const LevelArgs& A, bool kahan, void* stream);
cudaError_t launch_level_bf16(const LevelArgs& A, bool kahan, void* stream);  // dev::ArithBf16  // dev::ArithHalfScaled
cudaError_t configure_level_carrier();
cudaError_t configure_level_f32();
cudaError_t configure_level_f32r();
cudaError_t configure_level_f64r();
cudaError_t configure_level_half2();
cudaError_t configure_level_h16();
cudaError_t configure_level_bf16();
cudaError_t configure_probe();
// warp-per-path instances (lpmc_wpp_*.cu; NP == 1 arithmetics)
cudaError_t launch_wpp_carrier(const LevelArgs& A, bool kahan, void* stream);
cudaError_t launch_wpp_f32(const LevelArgs& A, bool kahan, void* stream);
cudaError_t launch_wpp_f32r(const LevelArgs& A, bool kahan, void* stream);
cudaError_t launch_wpp_f64r(const LevelArgs& A, bool kahan, void* stream);
cudaError_t configure_wpp_carrier();
cudaError_t configure_wpp_f32();
cudaError_t configure_wpp_f32r();
cudaError_t configure_wpp_f64r();
#endif
// step_error_probe (lpmc_probe.cu): block_sums = 4 per 256-path block
cudaError_t launch_step_error(const LevelArgs& A, BarArith arith, uint64_t last_steps,
                              double* block_sums, void* stream);

}  // namespace lpmc_b200
