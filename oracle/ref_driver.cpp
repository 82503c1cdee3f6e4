// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// C-ABI driver around the UNMODIFIED reference headers (proj/include/lpmc under
// /root/reference). `oracle/Makefile` compiles it the way the reference CLI is
// built (proj/CMakeLists.txt:12,24: -O2 -DNDEBUG, gnu++20) plus
// -ffp-contract=off into oracle/_ref/liblpmc_ref.so.  Only the
// tests, the golden-vector generator, smoke() and bench.py's reference /
// cpu_baseline legs load it.
//
// The reference keeps the approximation coefficients and the accumulator
// fields private (invcdf_approx.hpp:92-98, stats.hpp:84-89); this driver opens
// them with an access macro so fixtures can record them bit-for-bit.  No
// reference source is copied: everything below only calls into the headers.

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <optional>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#define private public
#include "lpmc/experiments.hpp"
#include "lpmc/gaussian.hpp"
#include "lpmc/invcdf_approx.hpp"
#include "lpmc/mlmc.hpp"
#include "lpmc/sde.hpp"
#include "lpmc/softfloat.hpp"
#include "lpmc/stats.hpp"
#include "lpmc/uniform.hpp"
#undef private

namespace {

enum : int { kOk = 0, kInvalidArgument = 1, kDomainError = 2, kRuntimeError = 3, kOther = 4 };

std::mutex g_mu;
std::map<std::string, std::unique_ptr<lpmc::InvCdfApprox>> g_tables;

// nullptr for "exact"; throws invalid_argument for unknown names.
const lpmc::InvCdfApprox* table_for(const char* name) {
  if (name == nullptr || std::strcmp(name, "exact") == 0) return nullptr;
  std::lock_guard<std::mutex> lock(g_mu);
  auto it = g_tables.find(name);
  if (it != g_tables.end()) return it->second.get();
  auto t = std::make_unique<lpmc::InvCdfApprox>(lpmc::InvCdfApprox::parse(name));
  const lpmc::InvCdfApprox* raw = t.get();
  g_tables.emplace(name, std::move(t));
  return raw;
}

void put_msg(char* msg, int len, const char* what) {
  if (msg == nullptr || len <= 0) return;
  std::snprintf(msg, static_cast<size_t>(len), "%s", what);
}

template <typename F>
int guarded(char* msg, int len, F&& f) {
  try {
    f();
    put_msg(msg, len, "");
    return kOk;
  } catch (const std::invalid_argument& e) {
    put_msg(msg, len, e.what());
    return kInvalidArgument;
  } catch (const std::domain_error& e) {
    put_msg(msg, len, e.what());
    return kDomainError;
  } catch (const std::runtime_error& e) {
    put_msg(msg, len, e.what());
    return kRuntimeError;
  } catch (const std::exception& e) {
    put_msg(msg, len, e.what());
    return kOther;
  }
}

void dump_acc(const lpmc::MomentAccumulator& a, double* out5) {
  out5[0] = static_cast<double>(a.n_);
  out5[1] = a.mean_;
  out5[2] = a.m2_;
  out5[3] = a.m3_;
  out5[4] = a.m4_;
}

}  // namespace

extern "C" {

int ref_abi_version() { return 1; }

uint64_t ref_stream_word(uint64_t seed, uint64_t path, uint64_t ctr) {
  return lpmc::detail::stream_word(seed, path, ctr);
}

// Fills out[0..count) with UniformStream(seed, path, ctr0).next() draws.
void ref_uniforms(uint64_t seed, uint64_t path, uint64_t ctr0, uint64_t count, double* out) {
  lpmc::UniformStream s(seed, path, ctr0);
  for (uint64_t i = 0; i < count; ++i) out[i] = s.next();
}

int ref_exact_inv_cdf(double u, double* z, char* msg, int len) {
  return guarded(msg, len, [&] { *z = lpmc::exact_inv_cdf(u); });
}

void ref_exact_inv_cdf_many(const double* u, uint64_t n, double* z) {
  for (uint64_t i = 0; i < n; ++i) {
    try {
      z[i] = lpmc::exact_inv_cdf(u[i]);
    } catch (...) {
      z[i] = std::nan("");
    }
  }
}

int ref_round(double x, int m, double* out, char* msg, int len) {
  return guarded(msg, len, [&] { *out = lpmc::round_to_precision(x, lpmc::PrecisionSpec{m}); });
}

void ref_round_many(const double* x, uint64_t n, int m, double* out) {
  for (uint64_t i = 0; i < n; ++i) out[i] = lpmc::round_to_precision(x[i], lpmc::PrecisionSpec{m});
}

// Table layout: K, degree, w_max, step_w, tail, breakpoints[K], coeff[4K].
int ref_table(const char* name, int* k, int* degree, double* w_max, double* step_w,
              double* tail, double* breakpoints, double* coeff, int cap, char* msg, int len) {
  return guarded(msg, len, [&] {
    const lpmc::InvCdfApprox* t = table_for(name);
    if (t == nullptr) throw std::invalid_argument("exact has no table");
    *k = t->interval_count();
    *degree = t->degree();
    *w_max = t->w_max_;
    *step_w = t->step_w_;
    *tail = t->tail_value_;
    if (cap < t->interval_count()) throw std::invalid_argument("table capacity too small");
    for (int j = 0; j < t->interval_count(); ++j) {
      breakpoints[j] = t->breakpoints_[j];
      for (int c = 0; c < 4; ++c) coeff[4 * j + c] = t->coeff_[j][c];
    }
  });
}

void ref_approx_many(const char* name, const double* u, uint64_t n, double* z) {
  const lpmc::InvCdfApprox* t = table_for(name);
  for (uint64_t i = 0; i < n; ++i) {
    try {
      z[i] = (*t)(u[i]);
    } catch (...) {
      z[i] = std::nan("");
    }
  }
}

// Four terminal values of simulate_coupled (sde.hpp:211) for each of n
// consecutive paths path_base.. ; out is n x 4 (hat_f, hat_c, bar_f, bar_c).
int ref_simulate_coupled(double mu, double sigma, double x0, double horizon, int level,
                         int mantissa_bits, const char* approx, int kahan, uint64_t seed,
                         uint64_t path_base, uint64_t n, double* out, char* msg, int len) {
  return guarded(msg, len, [&] {
    const lpmc::SdeModel model = lpmc::make_gbm(mu, sigma, x0, horizon);
    const lpmc::InvCdfApprox* t = table_for(approx);
    const lpmc::PrecisionSpec spec{mantissa_bits};
    for (uint64_t i = 0; i < n; ++i) {
      lpmc::CoupledResult r = lpmc::simulate_coupled(model, level, spec, t, kahan != 0,
                                                     lpmc::UniformStream(seed, path_base + i));
      out[4 * i + 0] = r.x_hat_fine;
      out[4 * i + 1] = r.x_hat_coarse;
      out[4 * i + 2] = r.x_bar_fine;
      out[4 * i + 3] = r.x_bar_coarse;
    }
  });
}

// run_coupled_paths (mlmc.hpp:67): out15 = 3 x {n, mean, m2, m3, m4} for
// d_hat, d_bar, d_four, raw accumulator state.
int ref_run_coupled_paths(double mu, double sigma, double x0, double horizon, int level,
                          int mantissa_bits, const char* approx, int kahan, uint64_t n_paths,
                          uint64_t seed, uint64_t path_base, int threads, double* out15,
                          char* msg, int len) {
  return guarded(msg, len, [&] {
    const lpmc::SdeModel model = lpmc::make_gbm(mu, sigma, x0, horizon);
    const lpmc::InvCdfApprox* t = table_for(approx);
    lpmc::CoupledMoments m =
        lpmc::run_coupled_paths(model, level, lpmc::PrecisionSpec{mantissa_bits}, t,
                                kahan != 0, n_paths, seed, path_base, threads);
    dump_acc(m.d_hat, out15);
    dump_acc(m.d_bar, out15 + 5);
    dump_acc(m.d_four, out15 + 10);
  });
}

// estimate_level_stats (mlmc.hpp:113) with the default CostModel except
// per_step_arithmetic; out18 = LevelStats fields in declaration order
// (mean_hat, v_hat, v_hat_stderr, mean_bar, v_bar, v_bar_stderr, mean_four,
// V_bar, V_bar_stderr, c_hat, c_bar, C_bar, m_hat, m_bar, M_bar, level).
int ref_estimate_level_stats(double mu, double sigma, double x0, double horizon, int level,
                             int mantissa_bits, const char* approx, int kahan, uint64_t n_paths,
                             uint64_t seed, double per_step_arithmetic, int threads,
                             uint64_t path_base, double* out16, char* msg, int len) {
  return guarded(msg, len, [&] {
    const lpmc::SdeModel model = lpmc::make_gbm(mu, sigma, x0, horizon);
    const lpmc::InvCdfApprox* t = table_for(approx);
    lpmc::CostModel cost;
    cost.per_step_arithmetic = per_step_arithmetic;
    lpmc::LevelStats s =
        lpmc::estimate_level_stats(model, level, lpmc::PrecisionSpec{mantissa_bits}, t,
                                   kahan != 0, n_paths, seed, cost, threads, path_base);
    const double v[16] = {s.mean_hat, s.v_hat, s.v_hat_stderr, s.mean_bar, s.v_bar,
                          s.v_bar_stderr, s.mean_four, s.V_bar, s.V_bar_stderr, s.c_hat,
                          s.c_bar, s.C_bar, static_cast<double>(s.m_hat),
                          static_cast<double>(s.m_bar), static_cast<double>(s.M_bar),
                          static_cast<double>(s.level)};
    std::memcpy(out16, v, sizeof v);
  });
}

// Sequential MomentAccumulator::add over x[0..n) -> {n, mean, m2, m3, m4}.
void ref_moments_add(const double* x, uint64_t n, double* out5) {
  lpmc::MomentAccumulator a;
  for (uint64_t i = 0; i < n; ++i) a.add(x[i]);
  dump_acc(a, out5);
}

// MomentAccumulator::merge of two raw states.
void ref_moments_merge(const double* a5, const double* b5, double* out5) {
  lpmc::MomentAccumulator a, b;
  a.n_ = static_cast<uint64_t>(a5[0]);
  a.mean_ = a5[1];
  a.m2_ = a5[2];
  a.m3_ = a5[3];
  a.m4_ = a5[4];
  b.n_ = static_cast<uint64_t>(b5[0]);
  b.mean_ = b5[1];
  b.m2_ = b5[2];
  b.m3_ = b5[3];
  b.m4_ = b5[4];
  a.merge(b);
  dump_acc(a, out5);
}

// LevelStats <-> 16 doubles, the ref_estimate_level_stats order.
static lpmc::LevelStats stats_from16(const double* v) {
  lpmc::LevelStats s;
  s.mean_hat = v[0];
  s.v_hat = v[1];
  s.v_hat_stderr = v[2];
  s.mean_bar = v[3];
  s.v_bar = v[4];
  s.v_bar_stderr = v[5];
  s.mean_four = v[6];
  s.V_bar = v[7];
  s.V_bar_stderr = v[8];
  s.c_hat = v[9];
  s.c_bar = v[10];
  s.C_bar = v[11];
  s.m_hat = static_cast<uint64_t>(v[12]);
  s.m_bar = static_cast<uint64_t>(v[13]);
  s.M_bar = static_cast<uint64_t>(v[14]);
  s.level = static_cast<int>(v[15]);
  return s;
}

static void stats_to16(const lpmc::LevelStats& s, double* out) {
  const double v[16] = {s.mean_hat, s.v_hat, s.v_hat_stderr, s.mean_bar, s.v_bar,
                        s.v_bar_stderr, s.mean_four, s.V_bar, s.V_bar_stderr, s.c_hat,
                        s.c_bar, s.C_bar, static_cast<double>(s.m_hat),
                        static_cast<double>(s.m_bar), static_cast<double>(s.M_bar),
                        static_cast<double>(s.level)};
  std::memcpy(out, v, sizeof v);
}

// allocate_samples (mlmc.hpp:165): stats16 = n x 16 doubles; kind 0/1.
int ref_allocate_samples(const double* stats16, uint64_t n, double eps, int kind,
                         uint64_t* primary, uint64_t* secondary, int* degenerate, char* msg,
                         int len) {
  return guarded(msg, len, [&] {
    std::vector<lpmc::LevelStats> st;
    for (uint64_t i = 0; i < n; ++i) st.push_back(stats_from16(stats16 + 16 * i));
    lpmc::Allocation a = lpmc::allocate_samples(
        st, eps, kind ? lpmc::AllocationKind::nested : lpmc::AllocationKind::standard);
    for (size_t i = 0; i < a.primary.size(); ++i) primary[i] = a.primary[i];
    for (size_t i = 0; i < a.secondary.size(); ++i) secondary[i] = a.secondary[i];
    *degenerate = a.degenerate ? 1 : 0;
  });
}

int ref_predicted_times(const double* stats16, uint64_t n, double eps, double* out2, char* msg,
                        int len) {
  return guarded(msg, len, [&] {
    std::vector<lpmc::LevelStats> st;
    for (uint64_t i = 0; i < n; ++i) st.push_back(stats_from16(stats16 + 16 * i));
    lpmc::PredictedTimes t = lpmc::predicted_times(st, eps);
    out2[0] = t.t_hat;
    out2[1] = t.t_bar;
  });
}

int ref_per_level_speedup(const double* stats16, double* value, int* cost_ratio_only, char* msg,
                          int len) {
  return guarded(msg, len, [&] {
    lpmc::SpeedupResult r = lpmc::per_level_speedup(stats_from16(stats16));
    *value = r.value;
    *cost_ratio_only = r.cost_ratio_only ? 1 : 0;
  });
}

// run_nested_estimator (mlmc.hpp:244): out = {value, t_hat, t_bar, degenerate};
// contributions[L+1], pilot16[(L+1) x 16], primary[L+1], secondary[L+1].
int ref_run_nested_estimator(double mu, double sigma, double x0, double horizon, int max_level,
                             int mantissa_bits, const char* approx, int kahan, double eps,
                             uint64_t seed, uint64_t pilot_paths, int threads, double* out4,
                             double* contributions, double* pilot16, uint64_t* primary,
                             uint64_t* secondary, char* msg, int len) {
  return guarded(msg, len, [&] {
    const lpmc::SdeModel model = lpmc::make_gbm(mu, sigma, x0, horizon);
    const lpmc::InvCdfApprox* t = table_for(approx);
    lpmc::EstimatorResult r = lpmc::run_nested_estimator(
        model, max_level, lpmc::PrecisionSpec{mantissa_bits}, t, kahan != 0, eps, seed,
        lpmc::CostModel{}, threads, pilot_paths);
    out4[0] = r.value;
    out4[1] = r.times.t_hat;
    out4[2] = r.times.t_bar;
    out4[3] = r.allocation.degenerate ? 1.0 : 0.0;
    for (size_t l = 0; l < r.level_contributions.size(); ++l) {
      contributions[l] = r.level_contributions[l];
      stats_to16(r.pilot_stats[l], pilot16 + 16 * l);
      primary[l] = r.allocation.primary[l];
      secondary[l] = r.allocation.secondary[l];
    }
  });
}

// simulate_two_way (sde.hpp:168) for n consecutive paths: out n x 2 (x_hat, x_bar).
int ref_simulate_two_way(double mu, double sigma, double x0, double horizon, int level,
                         int mantissa_bits, const char* approx, int kahan, uint64_t seed,
                         uint64_t path_base, uint64_t n, double* out, char* msg, int len) {
  return guarded(msg, len, [&] {
    const lpmc::SdeModel model = lpmc::make_gbm(mu, sigma, x0, horizon);
    const lpmc::InvCdfApprox* t = table_for(approx);
    const lpmc::LevelSpec ls{level, horizon};
    for (uint64_t i = 0; i < n; ++i) {
      lpmc::TwoWayResult r = lpmc::simulate_two_way(model, ls, lpmc::PrecisionSpec{mantissa_bits},
                                                    t, kahan != 0,
                                                    lpmc::UniformStream(seed, path_base + i));
      out[2 * i] = r.x_hat;
      out[2 * i + 1] = r.x_bar;
    }
  });
}

// run_two_way_experiment (experiments.hpp:119) for one precision name and a
// level range, paths per level broadcast; out = rows x {n_steps, variance,
// stderr, paths}.
int ref_two_way_experiment(double mu, double sigma, double x0, double horizon,
                           const char* precision, const char* approx, int kahan, int level_min,
                           int level_max, uint64_t paths, uint64_t seed, int threads,
                           double* out4, char* msg, int len) {
  return guarded(msg, len, [&] {
    lpmc::ExperimentConfig c;
    c.mu = mu;
    c.sigma = sigma;
    c.x0 = x0;
    c.horizon = horizon;
    c.precisions = {precision};
    c.approx = approx;
    c.kahan = kahan != 0;
    c.level_min = level_min;
    c.level_max = level_max;
    if (paths) c.paths = {paths};
    c.seed = seed;
    c.threads = threads;
    std::vector<lpmc::TwoWayRow> rows = lpmc::run_two_way_experiment(c);
    for (size_t i = 0; i < rows.size(); ++i) {
      out4[4 * i] = static_cast<double>(rows[i].n_steps);
      out4[4 * i + 1] = rows[i].variance;
      out4[4 * i + 2] = rows[i].stderr_variance;
      out4[4 * i + 3] = static_cast<double>(rows[i].paths);
    }
  });
}

// step_error_probe (sde.hpp:297): out5 = {mean_eta, mean_abs_eta,
// mean_eta_prime, mean_abs_eta_prime, samples}.
int ref_step_error_probe(double mu, double sigma, double x0, double horizon, int level,
                         int mantissa_bits, const char* approx, uint64_t n_samples, uint64_t seed,
                         double* out5, char* msg, int len) {
  return guarded(msg, len, [&] {
    const lpmc::SdeModel model = lpmc::make_gbm(mu, sigma, x0, horizon);
    const lpmc::InvCdfApprox* t = table_for(approx);
    lpmc::StepErrorStats r = lpmc::step_error_probe(model, lpmc::LevelSpec{level, horizon},
                                                    lpmc::PrecisionSpec{mantissa_bits}, t,
                                                    n_samples, seed);
    out5[0] = r.mean_eta;
    out5[1] = r.mean_abs_eta;
    out5[2] = r.mean_eta_prime;
    out5[3] = r.mean_abs_eta_prime;
    out5[4] = static_cast<double>(r.samples);
  });
}

// run_density_report (experiments.hpp:258): rows as {series (0 curve, 1 hist),
// x, y} triples; returns the row count in *n_rows (cap rows max).
int ref_density_report(const char* approx, uint64_t seed, int curve_points, uint64_t hist_samples,
                       double bin_width, double* out3, int cap, int* n_rows, char* msg,
                       int len) {
  return guarded(msg, len, [&] {
    lpmc::ExperimentConfig c;
    c.approx = approx;
    c.seed = seed;
    c.level_min = 0;
    c.level_max = 0;
    std::vector<lpmc::DensityRow> rows =
        lpmc::run_density_report(c, curve_points, hist_samples, bin_width);
    if (static_cast<int>(rows.size()) > cap) throw std::runtime_error("density rows exceed cap");
    for (size_t i = 0; i < rows.size(); ++i) {
      out3[3 * i] = rows[i].series == "curve" ? 0.0 : 1.0;
      out3[3 * i + 1] = rows[i].x;
      out3[3 * i + 2] = rows[i].y;
    }
    *n_rows = static_cast<int>(rows.size());
  });
}

int ref_hardware_threads() { return static_cast<int>(std::thread::hardware_concurrency()); }

}  // extern "C"
