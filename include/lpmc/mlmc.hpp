// Drop-in for the reference's lpmc/mlmc.hpp (proj/include/lpmc/mlmc.hpp):
// CostModel, LevelStats, CoupledMoments, run_coupled_paths,
// estimate_level_stats (:20-149) and the estimator layer above them --
// allocate_samples, predicted_times, per_level_speedup, run_nested_estimator
// (:151-285).  Every entry point keeps the reference signature; the sampling
// runs on the sm_100a kernels behind lpmc_run_coupled_paths /
// lpmc_estimate_level_stats / lpmc_run_nested_estimator, the allocation
// arithmetic in the library's host code (bitwise the reference's).  `threads` only
// scheduled the CPU reference and never changed its result (mlmc.hpp:4-5);
// it is accepted and ignored.
//
// Extension: an optional trailing DeviceOptions selects legs, payoff,
// reduction order, device and stream.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <vector>

#include "../lpmc_b200.h"
#include "error.hpp"
#include "invcdf_approx.hpp"
#include "sde.hpp"
#include "softfloat.hpp"
#include "stats.hpp"

namespace lpmc {

struct CostModel {
  double cycles_exact_rng = 3.5;
  double cycles_approx_rng_single = 0.5;
  double cycles_approx_rng_half = 0.25;
  double kahan_overhead_factor = 1.4;
  double per_step_arithmetic = 0.0;

  double approx_rng_cycles(const PrecisionSpec& spec) const {
    return spec.mantissa_bits <= 10 ? cycles_approx_rng_half : cycles_approx_rng_single;
  }
  lpmc_cost_model c_abi() const {
    return lpmc_cost_model{cycles_exact_rng, cycles_approx_rng_single, cycles_approx_rng_half,
                           kahan_overhead_factor, per_step_arithmetic};
  }
};

struct LevelStats {
  int level = 0;
  double mean_hat = 0.0, v_hat = 0.0, v_hat_stderr = 0.0;
  double mean_bar = 0.0, v_bar = 0.0, v_bar_stderr = 0.0;
  double mean_four = 0.0, V_bar = 0.0, V_bar_stderr = 0.0;
  double c_hat = 0.0, c_bar = 0.0, C_bar = 0.0;
  std::uint64_t m_hat = 0, m_bar = 0, M_bar = 0;
};

struct CoupledMoments {
  MomentAccumulator d_hat;
  MomentAccumulator d_bar;
  MomentAccumulator d_four;

  void merge(const CoupledMoments& other) {
    d_hat.merge(other.d_hat);
    d_bar.merge(other.d_bar);
    d_four.merge(other.d_four);
  }
};

// Extension knobs (defaults reproduce the reference).
struct DeviceOptions {
  unsigned legs = LPMC_LEGS_ALL;
  int payoff = LPMC_PAYOFF_TERMINAL;
  double strike = 1.0;
  int reduce = LPMC_REDUCE_TREE;
  int device = -1;
  void* stream = nullptr;
  int exact_z = LPMC_EXACT_Z_FAST;  // LPMC_EXACT_Z_GLIBC: the reference's Z bit for bit
  std::vector<int32_t> devices;      // > 1 entries: shard every run over these devices
  int schedule = LPMC_SCHEDULE_AUTO;  // kernel schedule (results identical)

  lpmc_options c_abi() const {
    return lpmc_options{legs,    payoff,         strike,
                        reduce,  device,         stream,
                        exact_z, devices.empty() ? nullptr : devices.data(),
                        static_cast<int32_t>(devices.size()), schedule};
  }
};

namespace detail {
inline lpmc_gbm gbm_of(const SdeModel& model) {
  if (!model.gbm)
    throw std::invalid_argument("the device sampler supports GBM models built by make_gbm");
  return lpmc_gbm{model.gbm->mu, model.gbm->sigma, model.x0, model.horizon};
}
}  // namespace detail

inline CoupledMoments run_coupled_paths(const SdeModel& model, int level,
                                        const PrecisionSpec& spec_low,
                                        const InvCdfApprox* approx, bool kahan,
                                        std::uint64_t n_paths, std::uint64_t seed,
                                        std::uint64_t path_base, int threads = 1,
                                        const DeviceOptions& options = {}) {
  (void)threads;
  const lpmc_gbm g = detail::gbm_of(model);
  const lpmc_precision p = spec_low.c_abi();
  const lpmc_options o = options.c_abi();
  lpmc_invcdf_table t{};
  if (approx != nullptr) t = approx->c_abi();
  lpmc_moments acc[3];
  lpmc_error err{};
  detail::throw_status(lpmc_run_coupled_paths(&g, level, &p, approx ? &t : nullptr, kahan ? 1 : 0,
                                              n_paths, seed, path_base, &o, acc, &err),
                       err);
  CoupledMoments m;
  m.d_hat = MomentAccumulator(acc[0]);
  m.d_bar = MomentAccumulator(acc[1]);
  m.d_four = MomentAccumulator(acc[2]);
  return m;
}

// Extension (diagnostic, no device needed): the arithmetic a production
// launch of run_coupled_paths uses for the low-precision legs -- low byte 0
// carrier, 1 native fp32, 2 fp32-carried rounding, 3 binary64 rounding, 4 IEEE
// half2; LPMC_ARITH_POW2_FOLDED / LPMC_ARITH_NATIVE_BINARY16 flags
// (lpmc_bar_arithmetic, include/lpmc_b200.h).  The choice never changes a
// result.
inline int bar_arithmetic(const SdeModel& model, int level, const PrecisionSpec& spec_low,
                          const InvCdfApprox* approx, bool kahan,
                          const DeviceOptions& options = {}) {
  const lpmc_gbm g = detail::gbm_of(model);
  const lpmc_precision p = spec_low.c_abi();
  const lpmc_options o = options.c_abi();
  lpmc_invcdf_table t{};
  if (approx != nullptr) t = approx->c_abi();
  std::int32_t out = 0;
  lpmc_error err{};
  detail::throw_status(
      lpmc_bar_arithmetic(&g, level, &p, approx ? &t : nullptr, kahan ? 1 : 0, &o, &out, &err), err);
  return out;
}

namespace detail {
inline LevelStats stats_from_c(const lpmc_level_stats& s) {
  LevelStats r;
  r.level = s.level;
  r.mean_hat = s.mean_hat;
  r.v_hat = s.v_hat;
  r.v_hat_stderr = s.v_hat_stderr;
  r.mean_bar = s.mean_bar;
  r.v_bar = s.v_bar;
  r.v_bar_stderr = s.v_bar_stderr;
  r.mean_four = s.mean_four;
  r.V_bar = s.V_bar;
  r.V_bar_stderr = s.V_bar_stderr;
  r.c_hat = s.c_hat;
  r.c_bar = s.c_bar;
  r.C_bar = s.C_bar;
  r.m_hat = s.m_hat;
  r.m_bar = s.m_bar;
  r.M_bar = s.M_bar;
  return r;
}

inline lpmc_level_stats stats_to_c(const LevelStats& s) {
  return lpmc_level_stats{s.level,  s.mean_hat, s.v_hat,  s.v_hat_stderr, s.mean_bar, s.v_bar,
                          s.v_bar_stderr, s.mean_four, s.V_bar, s.V_bar_stderr, s.c_hat,
                          s.c_bar, s.C_bar, s.m_hat, s.m_bar, s.M_bar};
}

inline std::vector<lpmc_level_stats> stats_to_c(const std::vector<LevelStats>& v) {
  std::vector<lpmc_level_stats> out;
  out.reserve(v.size());
  for (const auto& s : v) out.push_back(stats_to_c(s));
  return out;
}
}  // namespace detail

inline LevelStats estimate_level_stats(const SdeModel& model, int level,
                                       const PrecisionSpec& spec_low,
                                       const InvCdfApprox* approx, bool kahan,
                                       std::uint64_t n_paths, std::uint64_t seed,
                                       const CostModel& cost = {}, int threads = 1,
                                       std::uint64_t path_base = 0,
                                       const DeviceOptions& options = {}) {
  (void)threads;
  const lpmc_gbm g = detail::gbm_of(model);
  const lpmc_precision p = spec_low.c_abi();
  const lpmc_options o = options.c_abi();
  const lpmc_cost_model c = cost.c_abi();
  lpmc_invcdf_table t{};
  if (approx != nullptr) t = approx->c_abi();
  lpmc_level_stats s{};
  lpmc_error err{};
  detail::throw_status(lpmc_estimate_level_stats(&g, level, &p, approx ? &t : nullptr,
                                                 kahan ? 1 : 0, n_paths, seed, &c, path_base, &o,
                                                 &s, &err),
                       err);
  return detail::stats_from_c(s);
}

// ---------------------------------------------------------------------------
// Estimator layer (mlmc.hpp:151-285).

enum class AllocationKind { standard, nested };

struct Allocation {
  std::vector<std::uint64_t> primary;
  std::vector<std::uint64_t> secondary;
  bool degenerate = false;
};

inline Allocation allocate_samples(const std::vector<LevelStats>& stats, double eps,
                                   AllocationKind kind) {
  const std::vector<lpmc_level_stats> c = detail::stats_to_c(stats);
  Allocation a;
  a.primary.assign(stats.size(), 0);
  std::vector<std::uint64_t> sec(stats.size(), 0);
  std::int32_t degenerate = 0;
  lpmc_error err{};
  const bool nested = kind == AllocationKind::nested;
  detail::throw_status(
      lpmc_allocate_samples(c.data(), c.size(), eps,
                            nested ? LPMC_ALLOCATION_NESTED : LPMC_ALLOCATION_STANDARD,
                            a.primary.data(), sec.data(), &degenerate, &err),
      err);
  if (nested) a.secondary = sec;
  a.degenerate = degenerate != 0;
  return a;
}

struct PredictedTimes {
  double t_hat = 0.0;
  double t_bar = 0.0;
};

inline PredictedTimes predicted_times(const std::vector<LevelStats>& stats, double eps) {
  const std::vector<lpmc_level_stats> c = detail::stats_to_c(stats);
  PredictedTimes t;
  lpmc_error err{};
  detail::throw_status(lpmc_predicted_times(c.data(), c.size(), eps, &t.t_hat, &t.t_bar, &err),
                       err);
  return t;
}

struct SpeedupResult {
  double value = 0.0;
  bool cost_ratio_only = false;
};

inline SpeedupResult per_level_speedup(const LevelStats& s) {
  const lpmc_level_stats c = detail::stats_to_c(s);
  SpeedupResult r;
  std::int32_t flag = 0;
  lpmc_error err{};
  detail::throw_status(lpmc_per_level_speedup(&c, &r.value, &flag, &err), err);
  r.cost_ratio_only = flag != 0;
  return r;
}

struct EstimatorResult {
  double value = 0.0;
  std::vector<double> level_contributions;
  std::vector<LevelStats> pilot_stats;
  Allocation allocation;
  PredictedTimes times;
  double eps = 0.0;
};

// The pilot pass and the main pass each run all their levels concurrently
// on the device (lpmc_run_nested_estimator); results as the reference's
// serial loops.
inline EstimatorResult run_nested_estimator(const SdeModel& model, int max_level,
                                            const PrecisionSpec& spec_low,
                                            const InvCdfApprox* approx, bool kahan, double eps,
                                            std::uint64_t seed, const CostModel& cost = {},
                                            int threads = 1, std::uint64_t pilot_paths = 1000,
                                            const DeviceOptions& options = {}) {
  (void)threads;
  if (max_level < 0) throw std::invalid_argument("max level must be >= 0");
  const lpmc_gbm g = detail::gbm_of(model);
  const lpmc_precision p = spec_low.c_abi();
  const lpmc_options o = options.c_abi();
  const lpmc_cost_model c = cost.c_abi();
  lpmc_invcdf_table t{};
  if (approx != nullptr) t = approx->c_abi();
  const std::size_t L = static_cast<std::size_t>(max_level) + 1;
  EstimatorResult r;
  r.level_contributions.assign(L, 0.0);
  std::vector<lpmc_level_stats> pilot(L);
  r.allocation.primary.assign(L, 0);
  r.allocation.secondary.assign(L, 0);
  lpmc_estimator_result out{};
  out.level_contributions = r.level_contributions.data();
  out.pilot_stats = pilot.data();
  out.primary = r.allocation.primary.data();
  out.secondary = r.allocation.secondary.data();
  lpmc_error err{};
  detail::throw_status(lpmc_run_nested_estimator(&g, max_level, &p, approx ? &t : nullptr,
                                                 kahan ? 1 : 0, eps, seed, &c, pilot_paths, &o,
                                                 &out, &err),
                       err);
  r.value = out.value;
  r.eps = out.eps;
  r.times = PredictedTimes{out.t_hat, out.t_bar};
  r.allocation.degenerate = out.degenerate != 0;
  for (const auto& s : pilot) r.pilot_stats.push_back(detail::stats_from_c(s));
  return r;
}

}  // namespace lpmc
