// Drop-in check: code written against the reference's C++ API
// (proj/include/lpmc: mlmc.hpp / invcdf_approx.hpp / softfloat.hpp / sde.hpp)
// compiles unchanged against include/lpmc and runs on liblpmc_b200.
// Shaped after the reference's own unit tests (tests/test_mlmc.cpp:72-95,
// 191-202; tests/test_randvar.cpp:106-139; tests/test_softfloat.cpp:55-64).
//
//   api_smoke --host-only   host numerics only (no GPU)
//   api_smoke               + device sampling (needs a B200)
#include <cmath>
#include <cstdio>
#include <cstring>
#include <stdexcept>

#include "lpmc/experiments.hpp"
#include "lpmc/mlmc.hpp"

using namespace lpmc;

static int g_fail = 0;
#define CHECK(c)                                              \
  do {                                                        \
    if (!(c)) {                                               \
      std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #c); \
      ++g_fail;                                               \
    }                                                         \
  } while (0)

template <typename E, typename F>
static bool throws(F&& f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

int main(int argc, char** argv) {
  const bool host_only = argc > 1 && std::strcmp(argv[1], "--host-only") == 0;

  // softfloat ties (test_softfloat.cpp:55-64)
  PrecisionSpec half{10};
  CHECK(round_to_precision(1.0 + 0x1p-11, half) == 1.0);
  CHECK(round_to_precision(1.0 + 3 * 0x1p-11, half) == 1.0 + 0x1p-9);
  CHECK(PrecisionSpec::parse("fp22").mantissa_bits == 16);
  CHECK(throws<std::invalid_argument>([] { PrecisionSpec::parse("fp8"); }));

  // approximation validation and evaluation (test_randvar.cpp:106-139)
  CHECK(throws<std::invalid_argument>([] { InvCdfApprox::build(InvCdfApprox::Kind::linear, 3); }));
  CHECK(InvCdfApprox::parse("linear:8").interval_count() == 8);
  CHECK(InvCdfApprox::parse("cubic:64").degree() == 3);
  auto approx8 = InvCdfApprox::build(InvCdfApprox::Kind::linear, 8);
  CHECK(approx8(0.5) == 0.0);
  CHECK(throws<std::domain_error>([&] { approx8(1.0); }));
  CHECK(approx8(0.3) == -approx8(0.7));

  // moments (stats.hpp)
  MomentAccumulator acc;
  for (int i = 0; i < 100; ++i) acc.add(0.01 * i);
  CHECK(acc.count() == 100);
  CHECK(std::fabs(acc.mean() - 0.495) < 1e-14);

  // allocation / predicted times / speedup closed forms (test_mlmc.cpp:97-189)
  {
    LevelStats a, b;
    a.level = 0;
    a.v_hat = 4.0;
    a.c_hat = 1.0;
    b.level = 1;
    b.v_hat = 1.0;
    b.c_hat = 4.0;
    auto alloc = allocate_samples({a, b}, 0.1, AllocationKind::standard);
    CHECK(alloc.primary.size() == 2 && !alloc.degenerate);
    CHECK(alloc.primary[0] == 1600 && alloc.primary[1] == 400);
    CHECK(allocate_samples({a}, 0.1, AllocationKind::standard).primary[0] == 800);
    CHECK(throws<std::invalid_argument>([] { allocate_samples({}, 0.1, AllocationKind::standard); }));
    CHECK(throws<std::invalid_argument>([&] { allocate_samples({a}, 0.0, AllocationKind::standard); }));
    LevelStats n;
    n.v_bar = 1.0;
    n.c_bar = 1.0;
    n.V_bar = 0.25;
    n.C_bar = 4.0;
    auto nested = allocate_samples({n}, 0.1, AllocationKind::nested);
    CHECK(nested.primary[0] == 400 && nested.secondary[0] == 100);
    auto d = allocate_samples({LevelStats{}}, 0.1, AllocationKind::nested);
    CHECK(d.degenerate && d.primary[0] == 1 && d.secondary[0] == 1);
    LevelStats t = n;
    t.v_hat = 4.0;
    t.c_hat = 1.0;
    auto pt = predicted_times({t}, 0.1);
    CHECK(std::fabs(pt.t_hat - 800.0) < 1e-9 && std::fabs(pt.t_bar - 800.0) < 1e-9);
    CHECK(std::fabs(predicted_times({t, t}, 0.1).t_hat - 4.0 * pt.t_hat) < 1e-9);
    LevelStats sp;
    sp.v_hat = 1.0;
    sp.c_hat = 8.0;
    sp.v_bar = 1.0;
    sp.c_bar = 2.0;
    sp.V_bar = 0.0;
    sp.C_bar = 10.0;
    CHECK(std::fabs(per_level_speedup(sp).value - 4.0) < 1e-12 && !per_level_speedup(sp).cost_ratio_only);
    sp.V_bar = 0.2;
    const double ratio = (1.0 * 2.0) / (1.0 * 8.0), mix = 1.0 + std::sqrt(0.2 * 10.0 / 2.0);
    CHECK(std::fabs(per_level_speedup(sp).value - 1.0 / (ratio * mix * mix)) < 1e-12);
    sp.v_bar = 0.0;
    CHECK(per_level_speedup(sp).cost_ratio_only && std::fabs(per_level_speedup(sp).value - 4.0) < 1e-12);
    sp.v_hat = 0.0;
    CHECK(throws<std::invalid_argument>([&] { per_level_speedup(sp); }));
    CHECK(ExperimentConfig{}.paths_for_level(11) == 2500);
  }

  {  // extension: which arithmetic the low-precision legs run on (host decision)
    const SdeModel gbm = make_gbm(0.05, 0.2, 1.0, 1.0);
    const InvCdfApprox lin = InvCdfApprox::build(InvCdfApprox::Kind::linear, 16);
    const int h = bar_arithmetic(gbm, 12, PrecisionSpec::fp16(), &lin, false);
    CHECK((h & 0xff) == 2 && (h & LPMC_ARITH_NATIVE_BINARY16) && (h & LPMC_ARITH_POW2_FOLDED));
    const int k = bar_arithmetic(gbm, 11, PrecisionSpec::fp16(), &lin, true);
    CHECK((k & LPMC_ARITH_NATIVE_BINARY16) && !(k & LPMC_ARITH_POW2_FOLDED));
    const int f = bar_arithmetic(gbm, 12, PrecisionSpec::fp32(), &lin, false);
    CHECK((f & 0xff) == 1 && !(f & LPMC_ARITH_NATIVE_BINARY16) && (f & LPMC_ARITH_POW2_FOLDED));
    CHECK((bar_arithmetic(gbm, 6, PrecisionSpec::carrier(), nullptr, false) & 0xff) == 0);
  }

  if (host_only) {
    std::printf(g_fail ? "host-only FAILED\n" : "host-only ok\n");
    return g_fail ? 1 : 0;
  }

  // estimate_level_stats: costs and the degenerate model (test_mlmc.cpp:72-95)
  SdeModel det = make_gbm(0.05, 0.0);
  CostModel cost;
  cost.per_step_arithmetic = 0.25;
  auto s = estimate_level_stats(det, 3, PrecisionSpec::carrier(), nullptr, false, 64, 1, cost);
  CHECK(s.v_hat == 0.0 && s.v_bar == 0.0 && s.V_bar == 0.0);
  CHECK(std::fabs(s.c_hat - (8 * 3.5 + 12 * 0.25)) < 1e-12);
  CHECK(std::fabs(s.c_bar - (8 * 0.5 + 12 * 0.25)) < 1e-12);
  CHECK(s.m_hat == 64);
  CHECK(throws<std::invalid_argument>(
      [&] { estimate_level_stats(det, 0, PrecisionSpec::fp16(), nullptr, false, 1, 1, cost); }));

  // thread-count independent moments (test_mlmc.cpp:191-202)
  SdeModel gbm = make_gbm();
  auto approx = InvCdfApprox::parse("linear:64");
  auto one = run_coupled_paths(gbm, 4, PrecisionSpec::fp16(), &approx, false, 1000, 5, 0, 1);
  auto three = run_coupled_paths(gbm, 4, PrecisionSpec::fp16(), &approx, false, 1000, 5, 0, 3);
  CHECK(one.d_bar.mean() == three.d_bar.mean());
  CHECK(one.d_bar.variance() == three.d_bar.variance());
  CHECK(one.d_four.variance() == three.d_four.variance());
  CHECK(one.d_hat.count() == 1000);

  // carrier + exact: four-way correction vanishes (test_mlmc.cpp:225-230)
  auto c = run_coupled_paths(gbm, 3, PrecisionSpec::carrier(), nullptr, false, 4096, 3, 0);
  CHECK(c.d_four.variance() == 0.0);

  // bit-exact mode: the reference's C1 checkpoint (tests/golden: seed 1,
  // level 6, fp64, exact Gaussians, 2^20 paths) in the reference's order
  {
    DeviceOptions o;
    o.exact_z = LPMC_EXACT_Z_GLIBC;
    o.reduce = LPMC_REDUCE_SEQUENTIAL;
    auto m = run_coupled_paths(gbm, 6, PrecisionSpec::carrier(), nullptr, false, 1u << 20, 1, 0, 1, o);
    CHECK(m.d_hat.mean() == 0x1.6bc234c2c6020p-16);
    CHECK(m.d_hat.variance() == 0x1.e0629aa8f5008p+3 / 1048575.0);
    o.devices = {0, 0};  // sharded over two sub-ranges of the process's devices: same bits
    auto m2 = run_coupled_paths(gbm, 6, PrecisionSpec::carrier(), nullptr, false, 1u << 20, 1, 0, 1, o);
    CHECK(m2.d_hat.mean() == m.d_hat.mean() && m2.d_four.variance() == m.d_four.variance());
  }

  // non-finite operand -> std::domain_error (test_sde.cpp:168-173 shape)
  SdeModel blow = make_gbm(1e30, 0.0, 1e300);
  CHECK(throws<std::domain_error>(
      [&] { run_coupled_paths(blow, 4, PrecisionSpec::carrier(), nullptr, false, 8, 1, 0); }));

  // nested estimator (test_mlmc.cpp:204-236)
  {
    SdeModel det0 = make_gbm(0.05, 0.0);
    auto r = run_nested_estimator(det0, 4, PrecisionSpec::carrier(), nullptr, false, 0.01, 1);
    CHECK(r.allocation.degenerate);
    const double expected = std::pow(1.0 + 0.05 * 0x1p-4, 16.0);
    CHECK(std::fabs(r.value - expected) <= 1e-12 * expected);
    CHECK(r.level_contributions.size() == 5 && r.pilot_stats.size() == 5);
    auto rc = run_nested_estimator(gbm, 2, PrecisionSpec::carrier(), nullptr, false, 0.05, 3);
    for (const auto& st : rc.pilot_stats) CHECK(st.V_bar == 0.0);
    auto a1024 = InvCdfApprox::parse("linear:1024");
    auto g = run_nested_estimator(gbm, 6, PrecisionSpec::fp32(), &a1024, false, 0.01, 11);
    CHECK(std::fabs(g.value - std::exp(0.05)) < 0.04);
    CHECK(g.times.t_hat > 0.0 && g.times.t_bar > 0.0);
  }

  // two-way / four-way experiments (experiments.hpp)
  {
    ExperimentConfig cfg;
    cfg.precisions = {"fp16", "fp32"};
    cfg.approx = "linear:16";
    cfg.level_min = 0;
    cfg.level_max = 3;
    cfg.paths = {2000};
    auto rows = run_two_way_experiment(cfg);
    CHECK(rows.size() == 8 && rows[3].n_steps == 8 && rows[4].precision == "fp32");
    CHECK(rows[0].variance > rows[4].variance);  // fp16 rounding dominates fp32's
    auto four = run_four_way_experiment(cfg);
    CHECK(four.rows.size() == 24 && four.high_stats.size() == 4);
    auto report = run_speedup_report(four.high_stats, four.low_stats, four.low_kahan_stats);
    CHECK(report.size() == 12);
  }

  // step-error probe (sde.hpp:297-344) and its report
  {
    auto lin = InvCdfApprox::parse("linear:16");
    auto st = step_error_probe(gbm, LevelSpec{3, 1.0}, PrecisionSpec::fp16(), &lin, 20000, 1);
    CHECK(st.samples == 20000 && st.mean_abs_eta > 0.0 && st.mean_abs_eta_prime > 0.0);
    ExperimentConfig cfg;
    cfg.approx = "linear:16";
    cfg.level_max = 2;
    CHECK(run_step_error_report(cfg, 10000).size() == 3);
    CHECK(throws<std::invalid_argument>([&] { run_step_error_report(cfg, 9999); }));
  }

  // density report (experiments.hpp:258-295)
  {
    ExperimentConfig cfg;
    cfg.approx = "linear:16";
    auto rows = run_density_report(cfg, 64, 20000, 0.1);
    CHECK(rows.size() == 63 + 88 && rows[0].series == "curve" && rows.back().series == "hist");
    double mass = 0.0;
    for (const auto& r : rows)
      if (r.series == "hist") mass += r.y * 0.1;
    CHECK(std::fabs(mass - 1.0) < 1e-12);
  }

  // non-GBM models are rejected (no CPU fallback)
  SdeModel custom = gbm;
  custom.gbm.reset();
  CHECK(throws<std::invalid_argument>(
      [&] { run_coupled_paths(custom, 2, PrecisionSpec::fp32(), nullptr, false, 8, 1, 0); }));

  std::printf(g_fail ? "device FAILED\n" : "device ok\n");
  return g_fail ? 1 : 0;
}
