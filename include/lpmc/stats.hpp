// Drop-in for the reference's lpmc/stats.hpp (MomentAccumulator,
// proj/include/lpmc/stats.hpp:13-90).  add/merge run in liblpmc_b200
// (lpmc_moments_add / lpmc_moments_merge), bitwise the reference's formulas.
#pragma once

#include <cmath>
#include <cstdint>

#include "../lpmc_b200.h"

namespace lpmc {

class MomentAccumulator {
 public:
  MomentAccumulator() = default;
  explicit MomentAccumulator(const lpmc_moments& raw) : s_(raw) {}

  void add(double x) { lpmc_moments_add(&s_, x); }
  void merge(const MomentAccumulator& other) { lpmc_moments_merge(&s_, &other.s_); }

  std::uint64_t count() const { return s_.n; }
  double mean() const { return s_.n ? s_.mean : 0.0; }
  double variance() const { return s_.n < 2 ? 0.0 : s_.m2 / static_cast<double>(s_.n - 1); }
  double fourth_central_moment() const { return s_.n ? s_.m4 / static_cast<double>(s_.n) : 0.0; }
  double variance_stderr() const {
    if (s_.n < 2) return 0.0;
    const double v = variance();
    const double spread = fourth_central_moment() - v * v;
    return std::sqrt((spread < 0.0 ? 0.0 : spread) / static_cast<double>(s_.n));
  }
  double mean_stderr() const {
    return s_.n < 2 ? 0.0 : std::sqrt(variance() / static_cast<double>(s_.n));
  }

  const lpmc_moments& raw() const { return s_; }

 private:
  lpmc_moments s_{0, 0.0, 0.0, 0.0, 0.0};
};

}  // namespace lpmc
