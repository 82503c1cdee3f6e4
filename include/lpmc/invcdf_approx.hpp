// Drop-in for the reference's lpmc/invcdf_approx.hpp (InvCdfApprox,
// proj/include/lpmc/invcdf_approx.hpp:28-145).  The table is built by
// liblpmc_b200 (lpmc_invcdf_build, same operation order, bitwise the
// reference's table); evaluation on the host goes through lpmc_invcdf_eval,
// and the sampler ships the table to the device per call.
// Extensions: Kind::constant ("constant:K", degree-0 projection, BASELINE
// config 3) and coefficients() (the reference keeps them private).
#pragma once

#include <array>
#include <stdexcept>
#include <string>
#include <vector>

#include "error.hpp"
#include "gaussian.hpp"
#include "quadrature.hpp"

namespace lpmc {

class InvCdfApprox {
 public:
  enum class Kind { linear, cubic, constant };

  Kind kind() const { return kind_; }
  int interval_count() const { return static_cast<int>(breakpoints_.size()); }
  int degree() const { return kind_ == Kind::cubic ? 3 : (kind_ == Kind::linear ? 1 : 0); }
  const std::vector<double>& breakpoints() const { return breakpoints_; }
  double truncation_point() const { return breakpoints_.back(); }
  double max_value() const { return tail_value_; }
  const std::vector<std::array<double, 4>>& coefficients() const { return coeff_; }

  double operator()(double u) const {
    const lpmc_invcdf_table t = c_abi();
    double z = 0.0;
    lpmc_error err{};
    detail::throw_status(lpmc_invcdf_eval(&t, u, &z, &err), err);
    return z;
  }

  static InvCdfApprox build(Kind kind, int interval_count) {
    if (interval_count < 2 || (interval_count & (interval_count - 1)) != 0)
      throw std::invalid_argument("interval count must be a power of two >= 2");
    InvCdfApprox a;
    a.kind_ = kind;
    a.breakpoints_.assign(interval_count, 0.0);
    a.coeff_.assign(interval_count, {0.0, 0.0, 0.0, 0.0});
    lpmc_error err{};
    detail::throw_status(
        lpmc_invcdf_build(static_cast<int32_t>(kind_id(kind)), interval_count, a.breakpoints_.data(),
                          a.coeff_.front().data(), &a.w_max_, &a.step_w_, &a.tail_value_, &err),
        err);
    return a;
  }

  // linear:K | cubic:K | constant:K
  static InvCdfApprox parse(const std::string& name) {
    const auto colon = name.find(':');
    if (colon == std::string::npos) throw std::invalid_argument("bad approximation name: " + name);
    const std::string kind_name = name.substr(0, colon);
    int k = 0;
    try {
      k = std::stoi(name.substr(colon + 1));
    } catch (const std::exception&) {
      throw std::invalid_argument("bad approximation name: " + name);
    }
    if (kind_name == "linear") return build(Kind::linear, k);
    if (kind_name == "cubic") return build(Kind::cubic, k);
    if (kind_name == "constant") return build(Kind::constant, k);
    throw std::invalid_argument("bad approximation name: " + name);
  }

  // C-ABI view (valid while *this lives).
  lpmc_invcdf_table c_abi() const {
    return lpmc_invcdf_table{kind_id(kind_), interval_count(), w_max_, step_w_, tail_value_,
                             breakpoints_.data(), coeff_.front().data()};
  }

 private:
  InvCdfApprox() = default;

  static int32_t kind_id(Kind k) {
    return k == Kind::linear ? LPMC_APPROX_LINEAR
                             : (k == Kind::cubic ? LPMC_APPROX_CUBIC : LPMC_APPROX_CONSTANT);
  }

  Kind kind_ = Kind::linear;
  double w_max_ = 0.0;
  double step_w_ = 0.0;
  double tail_value_ = 0.0;
  std::vector<double> breakpoints_;
  std::vector<std::array<double, 4>> coeff_;
};

// E[Z^p], p = 1..p_max, by the reference's per-interval quadrature over both
// halves plus the clamped tails (invcdf_approx.hpp:147-185)
inline std::vector<double> moment_diagnostics(const InvCdfApprox& approx, int p_max) {
  if (p_max < 1 || p_max > 8) throw std::invalid_argument("moment order must be in [1, 8]");
  std::vector<double> out(p_max, 0.0);
  const lpmc_invcdf_table t = approx.c_abi();
  lpmc_error err{};
  detail::throw_status(lpmc_moment_diagnostics(&t, p_max, out.data(), &err), err);
  return out;
}

}  // namespace lpmc
