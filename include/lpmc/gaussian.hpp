// Drop-in for the reference's lpmc/gaussian.hpp (normal CDF / PDF and the
// exact inverse CDF, proj/include/lpmc/gaussian.hpp:14-65), evaluated by
// liblpmc_b200 on the host with the reference's expression trees (Acklam +
// one Newton step on glibc's erfc/exp; bitwise the reference's on the same
// libm).  The device sampler's exact Gaussians are the LPMC_EXACT_Z_* modes
// (include/lpmc_b200.h).
#pragma once

#include "error.hpp"

namespace lpmc {

inline double normal_cdf(double x) { return lpmc_normal_cdf(x); }
inline double normal_pdf(double x) { return lpmc_normal_pdf(x); }

namespace detail {
// Acklam's rational for u in (0, 1/2] polished by one Newton step (gaussian.hpp:26-55)
inline double inv_cdf_lower(double u) { return lpmc_inv_cdf_lower(u); }
}  // namespace detail

// gaussian.hpp:59-65: domain_error outside (0, 1), exactly 0 at 1/2,
// bit-exact reflection of the upper half
inline double exact_inv_cdf(double u) {
  double z = 0.0;
  lpmc_error err{};
  detail::throw_status(lpmc_exact_inv_cdf(u, &z, &err), err);
  return z;
}

}  // namespace lpmc
