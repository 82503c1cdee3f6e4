// Drop-in for the model types of the reference's lpmc/sde.hpp
// (SdeModel / make_gbm, proj/include/lpmc/sde.hpp:24-44).
//
// The reference's SdeModel is a pair of type-erased std::function objects,
// which a GPU kernel cannot call.  make_gbm therefore also records its GBM
// parameters in `gbm`; the device sampler reads those and rejects any model
// without them with std::invalid_argument (there is no CPU fallback).  The
// per-path CPU routines of sde.hpp (simulate_coupled & co.) are the oracle's
// business (oracle/), not this library's.
#pragma once

#include <functional>
#include <optional>

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

}  // namespace lpmc
