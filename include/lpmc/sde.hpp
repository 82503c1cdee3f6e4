// Drop-in for the model types of the reference's lpmc/sde.hpp
// (SdeModel / make_gbm, proj/include/lpmc/sde.hpp:24-44).
//
// The reference's SdeModel is a pair of type-erased std::function objects,
// which a GPU kernel cannot call.  make_gbm therefore also records its GBM
// parameters in `gbm`; the device sampler reads those and rejects any model
// without them with std::invalid_argument (there is no CPU fallback).  The
// per-path CPU routines of sde.hpp (simulate_coupled & co.) are the oracle's
// business (oracle/), not this library's; step_error_probe (:289-344) runs on
// the device (lpmc_step_error_probe).
#pragma once

#include <cstdint>
#include <functional>
#include <optional>

#include "invcdf_approx.hpp"
#include "softfloat.hpp"

namespace lpmc {

struct GbmParams {
  double mu;
  double sigma;
};

struct SdeModel {
  std::function<double(double t, double x, const PrecisionSpec&)> drift;
  std::function<double(double t, double x, const PrecisionSpec&)> diffusion;
  double x0 = 1.0;
  double horizon = 1.0;
  std::optional<GbmParams> gbm;  // set by make_gbm; required by the device sampler
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
  int level;
  double horizon = 1.0;
  unsigned long long step_count() const { return 1ull << level; }
  double step() const { return std::ldexp(horizon, -level); }
};

// sde.hpp:289-295
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
