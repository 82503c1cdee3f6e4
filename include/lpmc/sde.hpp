// Drop-in for the reference's lpmc/sde.hpp (proj/include/lpmc/sde.hpp):
// the model types (SdeModel / make_gbm, :24-44), the Euler-Maruyama scheme
// layer (LevelSpec, KahanState, em_step*, detail::kahan_accumulate,
// detail::check_state, :46-125), the per-path simulators (simulate_path,
// simulate_two_way, simulate_coupled, :126-284) and step_error_probe
// (:286-344).
//
// * The scheme functions take the caller's SdeModel and evaluate it on the
//   host op by op in the given precision, exactly as the reference defines
//   them (fp_* round through liblpmc_b200, bitwise the reference's).
// * The path simulators run on the device: one lpmc_simulate_paths call for
//   the stream's (seed, path, counter), the same kernels as the level
//   sampler (coupled legs; the fine legs = simulate_two_way; simulate_path
//   is that kernel's low-precision fine leg) in the bit-exact glibc mode of
//   the exact Gaussians, so the results are the reference's bitwise.  The
//   reference's SdeModel is a
//   pair of type-erased std::functions, which a GPU kernel cannot call, so
//   make_gbm also records its GBM parameters in `gbm`; the device paths
//   reject any other model with std::invalid_argument.  There is no CPU
//   fallback.
#pragma once

#include <cmath>
#include <cstdint>
#include <functional>
#include <optional>
#include <stdexcept>
#include <string>

#include "gaussian.hpp"
#include "invcdf_approx.hpp"
#include "softfloat.hpp"
#include "uniform.hpp"

namespace lpmc {

struct GbmParams {
  double mu;
  double sigma;
};

struct SdeModel {
  // evaluated op by op in the supplied precision; t is carrier precision
  std::function<double(double t, double x, const PrecisionSpec&)> drift;
  std::function<double(double t, double x, const PrecisionSpec&)> diffusion;
  double x0 = 1.0;
  double horizon = 1.0;
  std::optional<GbmParams> gbm;  // set by make_gbm; required by the device paths
};

inline SdeModel make_gbm(double mu = 0.05, double sigma = 0.2, double x0 = 1.0,
                         double horizon = 1.0) {
  SdeModel m;
  m.drift = [mu](double, double x, const PrecisionSpec& s) {
    return fp_mul(round_to_precision(mu, s), x, s);
  };
  m.diffusion = [sigma](double, double x, const PrecisionSpec& s) {
    return fp_mul(round_to_precision(sigma, s), x, s);
  };
  m.x0 = x0;
  m.horizon = horizon;
  m.gbm = GbmParams{mu, sigma};
  return m;
}

struct LevelSpec {
  int level;  // l >= 0
  double horizon = 1.0;
  std::uint64_t step_count() const { return std::uint64_t{1} << level; }
  double step() const { return std::ldexp(horizon, -level); }
};

struct KahanState {
  double sum = 0.0;
  double comp = 0.0;
};

// X (+) ((a (x) dt) (+) ((b (x) sqrt_dt) (x) z))  (sde.hpp:60-68)
inline double em_step(double x, double t, double dt, double sqrt_dt, double z,
                      const SdeModel& model, const PrecisionSpec& spec) {
  const double a = model.drift(t, x, spec);
  const double b = model.diffusion(t, x, spec);
  const double drift_term = fp_mul(a, dt, spec);
  const double diffusion_term = fp_mul(fp_mul(b, sqrt_dt, spec), z, spec);
  return fp_add(x, fp_add(drift_term, diffusion_term, spec), spec);
}

// the coarse form with a precomputed Wiener increment (sde.hpp:70-80)
inline double em_step_dw(double x, double t, double dt, double dw, const SdeModel& model,
                         const PrecisionSpec& spec) {
  const double a = model.drift(t, x, spec);
  const double b = model.diffusion(t, x, spec);
  const double drift_term = fp_mul(a, dt, spec);
  const double diffusion_term = fp_mul(b, dw, spec);
  return fp_add(x, fp_add(drift_term, diffusion_term, spec), spec);
}

namespace detail {

// Kahan compensation of the outer accumulation only (sde.hpp:84-92)
inline double kahan_accumulate(KahanState& k, double increment, const PrecisionSpec& spec) {
  const double y = fp_sub(increment, k.comp, spec);
  const double updated = fp_add(k.sum, y, spec);
  k.comp = fp_sub(fp_sub(updated, k.sum, spec), y, spec);
  k.sum = updated;
  return updated;
}

inline void check_state(double x, std::uint64_t step_index) {  // sde.hpp:120-124
  if (!std::isfinite(x))
    throw std::runtime_error("non-finite state at step " + std::to_string(step_index));
}

}  // namespace detail

inline double em_step_kahan(double x, KahanState& kahan, double t, double dt, double sqrt_dt,
                            double z, const SdeModel& model, const PrecisionSpec& spec) {
  const double a = model.drift(t, x, spec);
  const double b = model.diffusion(t, x, spec);
  const double drift_term = fp_mul(a, dt, spec);
  const double diffusion_term = fp_mul(fp_mul(b, sqrt_dt, spec), z, spec);
  return detail::kahan_accumulate(kahan, fp_add(drift_term, diffusion_term, spec), spec);
}

inline double em_step_kahan_dw(double x, KahanState& kahan, double t, double dt, double dw,
                               const SdeModel& model, const PrecisionSpec& spec) {
  const double a = model.drift(t, x, spec);
  const double b = model.diffusion(t, x, spec);
  const double drift_term = fp_mul(a, dt, spec);
  const double diffusion_term = fp_mul(b, dw, spec);
  return detail::kahan_accumulate(kahan, fp_add(drift_term, diffusion_term, spec), spec);
}

struct PathResult {
  double terminal = 0.0;
  std::uint64_t rng_draws = 0;
  std::uint64_t steps = 0;
};

struct TwoWayResult {
  double x_hat = 0.0;  // carrier precision, exact inverse CDF
  double x_bar = 0.0;  // target precision, approximate variables
  std::uint64_t rng_draws = 0;
};

struct CoupledResult {
  double x_hat_fine = 0.0;
  double x_hat_coarse = 0.0;
  double x_bar_fine = 0.0;
  double x_bar_coarse = 0.0;
  std::uint64_t rng_draws = 0;
  std::uint64_t steps = 0;
};

namespace detail {

// One path of the device sampler: terminal values {x_hat_f, x_hat_c,
// x_bar_f, x_bar_c} of the stream's path (lpmc_simulate_paths, n = 1).
inline void device_path(const SdeModel& model, int level, double horizon,
                        const PrecisionSpec& spec, const InvCdfApprox* approx, bool kahan,
                        const UniformStream& stream, std::uint32_t legs, double out4[4]) {
  if (!model.gbm)
    throw std::invalid_argument("the device sampler supports GBM models built by make_gbm");
  const lpmc_gbm g{model.gbm->mu, model.gbm->sigma, model.x0, horizon};
  const lpmc_precision p = spec.c_abi();
  lpmc_invcdf_table t{};
  if (approx != nullptr) t = approx->c_abi();
  lpmc_options o;
  lpmc_default_options(&o);
  o.legs = legs;
  o.counter = stream.counter();
  // per-path calls are parity-sized: the reference's own exact Gaussians
  // (glibc mode), so every leg equals the reference's bit for bit
  o.exact_z = LPMC_EXACT_Z_GLIBC;
  lpmc_error err{};
  throw_status(lpmc_simulate_paths(&g, level, &p, approx ? &t : nullptr, kahan ? 1 : 0, 1,
                                   stream.seed(), stream.path_index(), &o, out4, nullptr, &err),
               err);
}

}  // namespace detail

// sde.hpp:129-155: one path in `spec` (Gaussians rounded into spec) -- the
// device's low-precision fine leg with spec as the bar precision
inline PathResult simulate_path(const SdeModel& model, const LevelSpec& level,
                                const PrecisionSpec& spec, const InvCdfApprox* approx, bool kahan,
                                UniformStream stream) {
  if (level.level < 0) throw std::invalid_argument("level must be >= 0");
  double out[4];
  detail::device_path(model, level.level, level.horizon, spec, approx, kahan, stream,
                      LPMC_LEGS_FINE, out);
  return {out[2], level.step_count(), level.step_count()};
}

// sde.hpp:157-196
inline TwoWayResult simulate_two_way(const SdeModel& model, const LevelSpec& level,
                                     const PrecisionSpec& spec_low, const InvCdfApprox* approx,
                                     bool kahan, UniformStream stream) {
  if (level.level < 0) throw std::invalid_argument("level must be >= 0");
  double out[4];
  detail::device_path(model, level.level, level.horizon, spec_low, approx, kahan, stream,
                      LPMC_LEGS_FINE, out);
  return {out[0], out[2], level.step_count()};
}

// sde.hpp:198-284: the four coupled terminal values of one path pair
inline CoupledResult simulate_coupled(const SdeModel& model, int level,
                                      const PrecisionSpec& spec_low, const InvCdfApprox* approx,
                                      bool kahan, UniformStream stream) {
  if (level < 0) throw std::invalid_argument("level must be >= 0");
  double out[4];
  detail::device_path(model, level, model.horizon, spec_low, approx, kahan, stream,
                      LPMC_LEGS_ALL, out);
  const std::uint64_t n_fine = std::uint64_t{1} << level;
  return {out[0], out[1], out[2], out[3], n_fine, level == 0 ? n_fine : n_fine + n_fine / 2};
}

// sde.hpp:286-295
struct StepErrorStats {
  double mean_eta = 0.0;
  double mean_abs_eta = 0.0;
  double mean_eta_prime = 0.0;
  double mean_abs_eta_prime = 0.0;
  std::uint64_t samples = 0;
};

// step_error_probe (sde.hpp:297-344) on the device.  The level's horizon is
// the model's (the reference builds LevelSpec{l, horizon} from the same
// config, experiments.hpp:315).
inline StepErrorStats step_error_probe(const SdeModel& model, const LevelSpec& level,
                                       const PrecisionSpec& spec, const InvCdfApprox* approx,
                                       std::uint64_t n_samples, std::uint64_t seed) {
  if (!model.gbm)
    throw std::invalid_argument("the device sampler supports GBM models built by make_gbm");
  const lpmc_gbm g{model.gbm->mu, model.gbm->sigma, model.x0, level.horizon};
  const lpmc_precision p = spec.c_abi();
  lpmc_invcdf_table t{};
  if (approx != nullptr) t = approx->c_abi();
  lpmc_step_error_stats out{};
  lpmc_error err{};
  detail::throw_status(lpmc_step_error_probe(&g, level.level, &p, approx ? &t : nullptr,
                                             n_samples, seed, nullptr, &out, &err),
                       err);
  return StepErrorStats{out.mean_eta, out.mean_abs_eta, out.mean_eta_prime,
                        out.mean_abs_eta_prime, out.samples};
}

}  // namespace lpmc
