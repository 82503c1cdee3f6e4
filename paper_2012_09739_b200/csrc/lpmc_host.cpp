// Host side of the C-ABI (include/lpmc_b200.h): argument checking with the
// reference's error contract, host numerics that must be bitwise the
// reference's (table build, rounding of the per-level constants, moment
// merges), device contexts, plans, and the index-order fold.
//
// Compiled with -O2 -ffp-contract=off (never contract: every double op here
// mirrors a reference op 1:1).  No CPU sampling fallback
// exists: if the device path fails, the call fails.

#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdlib>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/lpmc_b200.h"
#include "lpmc_internal.h"
#include "lpmc_glibc.cuh"
#include "lpmc_math.cuh"

namespace lpmc_b200 {
namespace {

constexpr uint64_t kBatch = LPMC_BATCH_PATHS;
constexpr uint64_t kChunkBatches = LPMC_CHUNK_BATCHES;
constexpr uint64_t kChunkPaths = LPMC_CHUNK_PATHS;
constexpr uint64_t kSliceChunks = 64;     // paths per launch slice = 2^24
constexpr uint64_t kSeqSliceChunks = 16;  // sequential mode keeps per-path diffs
constexpr int kMaxK = 1024;

thread_local uint64_t t_launches = 0;

// ------------------------------------------------------------ errors -------
lpmc_status fail(lpmc_error* err, lpmc_status st, const std::string& msg, int kind = 0,
                 uint64_t path = 0, uint64_t step = 0) {
  if (err != nullptr) {
    err->status = st;
    err->kind = kind;
    err->path_index = path;
    err->step = step;
    std::snprintf(err->message, sizeof(err->message), "%s", msg.c_str());
  }
  return st;
}

lpmc_status ok(lpmc_error* err) {
  if (err != nullptr) {
    err->status = LPMC_OK;
    err->kind = 0;
    err->path_index = 0;
    err->step = 0;
    err->message[0] = '\0';
  }
  return LPMC_OK;
}

lpmc_status cuda_fail(lpmc_error* err, cudaError_t e, const char* where) {
  return fail(err, LPMC_CUDA_ERROR, std::string(where) + ": " + cudaGetErrorString(e));
}

// --------------------------------------------------- host numerics ---------
// round_to_precision (softfloat.hpp:69-80): RNE to m+1 significant bits,
// unbounded exponent.  Returns false for a non-finite operand.
bool round_prec(double x, int m, double* out) {
  if (!std::isfinite(x)) return false;
  if (x == 0.0 || m >= 52) {
    *out = x;
    return true;
  }
  int e = 0;
  const double frac = std::frexp(x, &e);
  const int p = m + 1;
  *out = std::ldexp(std::nearbyint(std::ldexp(frac, p)), e - p);
  return true;
}

// double -> IEEE binary16 bits, one round-to-nearest-even (== __double2half).
uint16_t half_bits(double x) {
  const uint16_t sign = std::signbit(x) ? 0x8000 : 0;
  const double ax = std::fabs(x);
  if (std::isnan(x)) return 0x7e00;
  if (ax == 0.0) return sign;
  if (ax < 0x1p-14) {  // subnormal range: units of 2^-24
    const double q = std::nearbyint(ax * 0x1p24);
    return static_cast<uint16_t>(sign | static_cast<uint16_t>(q));  // q == 1024 -> min normal
  }
  int e = 0;
  const double f = std::frexp(ax, &e);  // ax = f 2^e, f in [1/2, 1)
  double r = std::nearbyint(f * 2048.0);
  if (r == 2048.0) {
    r = 1024.0;
    e += 1;
  }
  const int ef = e - 1 + 15;
  if (ef >= 31 || std::isinf(x)) return static_cast<uint16_t>(sign | 0x7c00);
  return static_cast<uint16_t>(sign | (ef << 10) | (static_cast<int>(r) - 1024));
}

double half_value(uint16_t h) {  // binary16 pattern -> double (finite patterns)
  const int e = (h >> 10) & 0x1f;
  const int f = h & 0x3ff;
  const double mag = e == 0 ? std::ldexp(static_cast<double>(f), -24)
                            : std::ldexp(static_cast<double>(f + 1024), e - 25);
  return (h & 0x8000) ? -mag : mag;
}

// v as a binary16 pattern if it is exactly representable (finite), else false
bool exact_half(double v, uint16_t* out) {
  if (!std::isfinite(v)) return false;
  const uint16_t h = half_bits(v);
  if ((h & 0x7c00) == 0x7c00 || half_value(h) != v) return false;
  *out = h;
  return true;
}

// gauss_legendre (quadrature.hpp:17-41): Newton on the Legendre recurrence.
void gauss_legendre_rule(int n, std::vector<double>& x_out, std::vector<double>& w_out) {
  x_out.assign(n, 0.0);
  w_out.assign(n, 0.0);
  for (int i = 0; i < n; ++i) {
    double x = std::cos(M_PI * (i + 0.75) / (n + 0.5));
    double deriv = 0.0;
    for (int iter = 0; iter < 100; ++iter) {
      double p_prev = 1.0;
      double p_cur = x;
      for (int k = 2; k <= n; ++k) {
        const double p_next = ((2.0 * k - 1.0) * x * p_cur - (k - 1.0) * p_prev) / k;
        p_prev = p_cur;
        p_cur = p_next;
      }
      deriv = n * (x * p_cur - p_prev) / (x * x - 1.0);
      const double dx = p_cur / deriv;
      x -= dx;
      if (std::fabs(dx) < 1e-15) break;
    }
    x_out[i] = x;
    w_out[i] = 2.0 / ((1.0 - x * x) * deriv * deriv);
  }
}

// Host exact inverse CDF, used only to build tables (invcdf_approx.hpp:128);
// same Acklam + Newton expression trees as gaussian.hpp:26-65.
double host_phi_inv_lower(double u) {
  double x;
  if (u < 0.02425) {
    const double q = std::sqrt(-2.0 * std::log(u));
    const double num = ((((-7.784894002430293e-03 * q + -3.223964580411365e-01) * q +
                          -2.400758277161838e+00) * q + -2.549732539343734e+00) * q +
                        4.374664141464968e+00) * q + 2.938163982698783e+00;
    const double den = (((7.784695709041462e-03 * q + 3.224671290700398e-01) * q +
                         2.445134137142996e+00) * q + 3.754408661907416e+00) * q + 1.0;
    x = num / den;
  } else {
    const double q = u - 0.5;
    const double r = q * q;
    const double num = ((((-3.969683028665376e+01 * r + 2.209460984245205e+02) * r +
                          -2.759285104469687e+02) * r + 1.383577518672690e+02) * r +
                        -3.066479806614716e+01) * r + 2.506628277459239e+00;
    const double den = ((((-5.447609879822406e+01 * r + 1.615858368580409e+02) * r +
                          -1.556989798598866e+02) * r + 6.680131188771972e+01) * r +
                        -1.328068155288572e+01) * r + 1.0;
    x = num * q / den;
  }
  const double resid = 0.5 * std::erfc(-x * 0.7071067811865475244) - u;
  const double dens = 0.3989422804014326779 * std::exp(-0.5 * x * x);
  return x - resid / dens;
}

double host_phi_inv(double u) {
  if (u == 0.5) return 0.0;
  return u > 0.5 ? -host_phi_inv_lower(1.0 - u) : host_phi_inv_lower(u);
}

bool valid_interval_count(int k) { return k >= 2 && (k & (k - 1)) == 0; }

// The reference's interval index J(v) for v = 1 - u' (invcdf_approx.hpp:75-79),
// K meaning "tail".
int reference_index(double v, int K, double w_max, double step_w) {
  const double w = -std::log2(v);
  if (w >= w_max) return K;
  int j = static_cast<int>((w - 1.0) / step_w);
  if (j < 0) j = 0;
  if (j >= K) j = K - 1;
  return j;
}

// v-thresholds T_k = max{v on the 2^-53 grid in (0, 1/2] : J(v) >= k}, k=1..K
// (T_K = tail).  J is non-increasing in v, so a bisection over the grid
// integer g (v = g 2^-53) reproduces the reference on every reachable v.
std::vector<double> index_thresholds(int K, double w_max, double step_w) {
  static std::mutex mu;
  static std::map<std::tuple<int, double, double>, std::vector<double>> cache;
  std::lock_guard<std::mutex> lock(mu);
  auto key = std::make_tuple(K, w_max, step_w);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  std::vector<double> thr(K, 0.0);
  const uint64_t g_max = 1ull << 52;  // v = 1/2
  for (int k = 1; k <= K; ++k) {
    auto pred = [&](uint64_t g) { return reference_index(std::ldexp(double(g), -53), K, w_max, step_w) >= k; };
    if (!pred(1)) {
      thr[k - 1] = 0.0;
      continue;
    }
    uint64_t lo = 1, hi = g_max;  // pred(lo) true
    if (pred(hi)) {
      lo = hi;
    } else {
      while (hi - lo > 1) {
        const uint64_t mid = lo + (hi - lo) / 2;
        if (pred(mid)) lo = mid; else hi = mid;
      }
    }
    thr[k - 1] = std::ldexp(double(lo), -53);
  }
  cache.emplace(key, thr);
  return thr;
}

struct HostTable {
  int K = 0, degree = 1, dyadic = 0, stride = 0, simple = 0;
  double tail = 0.0;
  std::vector<double> rows;  // device layout (lpmc_internal.h)
};

lpmc_status prepare_table(const lpmc_invcdf_table* t, HostTable* out, lpmc_error* err) {
  if (t->kind < 0 || t->kind > 2)
    return fail(err, LPMC_INVALID_ARGUMENT, "bad approximation kind");
  if (!valid_interval_count(t->interval_count))
    return fail(err, LPMC_INVALID_ARGUMENT, "interval count must be a power of two >= 2");
  if (t->interval_count > kMaxK)
    return fail(err, LPMC_INVALID_ARGUMENT, "device tables support interval counts up to 1024");
  if (t->breakpoints == nullptr || t->coeff == nullptr)
    return fail(err, LPMC_INVALID_ARGUMENT, "table has no coefficients");
  const int K = t->interval_count;
  out->K = K;
  out->degree = t->kind == LPMC_APPROX_CUBIC ? 3 : 1;
  out->tail = t->tail_value;
  bool dyadic = K <= 32 && t->step_w == 1.0 && t->w_max == static_cast<double>(K + 1);
  for (int j = 0; dyadic && j < K; ++j) dyadic = t->breakpoints[j] == 1.0 - std::ldexp(1.0, -(j + 2));
  out->dyadic = dyadic ? 1 : 0;
  out->stride = K;
  // signed-zero fix-up provably unnecessary (see dev::approx_inv)
  bool simple = t->kind != LPMC_APPROX_CUBIC;
  for (int j = 0; simple && j < K; ++j) {
    const double* c = t->coeff + 4 * j;
    simple = c[0] != 0.0 && c[2] == 0.0 && !std::signbit(c[2]) && c[3] == 0.0 &&
             !std::signbit(c[3]);
  }
  out->simple = simple ? 1 : 0;
  auto left = [&](int j) { return j == 0 ? 0.5 : t->breakpoints[j - 1]; };
  if (dyadic) {  // records {3 - 2^(j+3), 2^(j+3), c0, c1, c2, c3} (dev::approx_inv)
    // K interval records, then tail records {0, 0, tail, 0, 0, 0} up to
    // j = 52 (v = 1 - u' >= 2^-53): the straight-line dyadic-linear
    // evaluation indexes j = floor(-log2 v) - 1 without a clamp or a tail
    // select, and a tail record gives tail + 0 * 0 = tail exactly.
    out->rows.assign(static_cast<size_t>(kDyadicRecord) * kDyadicRecords, 0.0);
    for (int j = 0; j < kDyadicRecords; ++j) {
      double* r = out->rows.data() + kDyadicRecord * j;
      if (j < K) {
        r[0] = 3.0 - std::ldexp(1.0, j + 3);
        r[1] = std::ldexp(1.0, j + 3);
        for (int c = 0; c < 4; ++c) r[2 + c] = t->coeff[4 * j + c];
      } else {
        r[2] = t->tail_value;
      }
    }
  } else {  // records {a, b - a, c0, c1 (, c2, c3)}, thresholds, 1 / step_w
    const int W = out->degree == 3 ? 6 : 4;
    out->stride = W;
    const size_t th = static_cast<size_t>(W) * K;
    out->rows.assign(th + K + 1, 0.0);
    for (int j = 0; j < K; ++j) {
      double* r = out->rows.data() + static_cast<size_t>(W) * j;
      r[0] = left(j);
      r[1] = t->breakpoints[j] - left(j);
      for (int c = 0; c < W - 2; ++c) r[2 + c] = t->coeff[4 * j + c];
    }
    const std::vector<double> thr = index_thresholds(K, t->w_max, t->step_w);
    std::copy(thr.begin(), thr.end(), out->rows.begin() + th);
    out->rows[th + K] = t->step_w > 0.0 ? 1.0 / t->step_w : 0.0;
  }
  return LPMC_OK;
}

// --------------------------------------------------------- moments ---------
struct Moments {
  uint64_t n = 0;
  double mean = 0.0, m2 = 0.0, m3 = 0.0, m4 = 0.0;
};

// MomentAccumulator::merge (stats.hpp:29-54); identical expression trees so
// the fold is bitwise the reference's.
void merge_into(Moments& a, const Moments& b) {
  if (b.n == 0) return;
  if (a.n == 0) {
    a = b;
    return;
  }
  const double na = static_cast<double>(a.n);
  const double nb = static_cast<double>(b.n);
  const double n = na + nb;
  const double d = b.mean - a.mean;
  const double d2 = d * d;
  const double m2 = a.m2 + b.m2 + d2 * na * nb / n;
  const double m3 = a.m3 + b.m3 + d2 * d * na * nb * (na - nb) / (n * n) +
                    3.0 * d * (na * b.m2 - nb * a.m2) / n;
  const double m4 = a.m4 + b.m4 + d2 * d2 * na * nb * (na * na - na * nb + nb * nb) / (n * n * n) +
                    6.0 * d2 * (na * na * b.m2 + nb * nb * a.m2) / (n * n) +
                    4.0 * d * (na * b.m3 - nb * a.m3) / n;
  a.mean += d * nb / n;
  a.m2 = m2;
  a.m3 = m3;
  a.m4 = m4;
  a.n += b.n;
}

Moments from_device(const double* p) {
  Moments m;
  m.n = static_cast<uint64_t>(p[0]);
  m.mean = p[1];
  m.m2 = p[2];
  m.m3 = p[3];
  m.m4 = p[4];
  return m;
}

lpmc_moments to_abi(const Moments& m) { return lpmc_moments{m.n, m.mean, m.m2, m.m3, m.m4}; }
Moments from_abi(const lpmc_moments& m) {
  Moments r;
  r.n = m.n;
  r.mean = m.mean;
  r.m2 = m.m2;
  r.m3 = m.m3;
  r.m4 = m.m4;
  return r;
}

// ------------------------------------------------------------ RNG keys ----
// detail::mix64 (uniform.hpp:13-19) on the host
uint64_t host_mix64(uint64_t z) {
  z ^= z >> 33;
  z *= 0xff51afd7ed558ccdull;
  z ^= z >> 33;
  z *= 0xc4ceb9fe1a85ec53ull;
  z ^= z >> 33;
  return z;
}

// mix64(seed + golden ratio) (uniform.hpp:23): the per-seed half of every
// path key, hoisted out of the kernels
uint64_t seed_key_of(uint64_t seed) { return host_mix64(seed + 0x9e3779b97f4a7c15ull); }

// ------------------------------------------------------- run spec ----------
struct RunSpec {
  LevelArgs args{};
  BarArith arith = BarArith::kCarrier;
  bool kahan = false;
  int reduce = LPMC_REDUCE_TREE;
  uint64_t n_paths = 0;
  uint64_t chunk_begin = 0, chunk_end = 0;  // chunk range this run covers
  HostTable table;
  bool has_table = false;
  int device = -1;
  std::vector<int> devices;  // > 1 entries: shard over these devices (run_multi_device)
  bool ieee = false;
  int schedule = LPMC_SCHEDULE_AUTO;
};

// Warp-per-path when asked, or (AUTO) when the fused grid of this run would
// leave most of the GPU idle at a level long enough for latency to rule:
// measured crossover (tools/gpu_schedule_sweep.sh) about
// 7e3-1e4 paths at levels 8-10; below 6144 paths (24 fused CTAs on 148 SMs)
// the warp-per-path schedule is 1.6-4.7x faster from level 10 up.
constexpr uint64_t kWppMaxAutoPaths = 6144;
constexpr int kWppMinAutoLevel = 5;
bool use_wpp(const RunSpec& s) {
  if (s.arith == BarArith::kHalf2 || s.args.level < 1) return false;
  if (s.schedule == LPMC_SCHEDULE_WARP_PER_PATH) return true;
  if (s.schedule == LPMC_SCHEDULE_FUSED) return false;
  return s.args.level >= kWppMinAutoLevel && s.n_paths <= kWppMaxAutoPaths;
}

bool in_native_range(double c, double lo, double hi) {
  const double a = std::fabs(c);
  return a == 0.0 || (a >= lo && a <= hi);
}

lpmc_status build_spec(const lpmc_gbm* model, int32_t level, const lpmc_precision* prec,
                       const lpmc_invcdf_table* table, int32_t kahan, uint64_t n_paths,
                       uint64_t seed, uint64_t path_base, const lpmc_options* opts,
                       RunSpec* spec, lpmc_error* err) {
  if (model == nullptr || prec == nullptr)
    return fail(err, LPMC_INVALID_ARGUMENT, "null model or precision");
  if (level < 0) return fail(err, LPMC_INVALID_ARGUMENT, "level must be >= 0");  // sde.hpp:215
  if (level > 40) return fail(err, LPMC_INVALID_ARGUMENT, "level must be <= 40");
  const int m = prec->mantissa_bits;
  if (m < 1) return fail(err, LPMC_INVALID_ARGUMENT, "mantissa_bits must be >= 1");
  lpmc_options o;
  lpmc_default_options(&o);
  if (opts != nullptr) o = *opts;
  if (o.legs == 0) o.legs = LPMC_LEGS_ALL;
  if (o.legs > 4) return fail(err, LPMC_INVALID_ARGUMENT, "bad legs mask");
  if (o.payoff != LPMC_PAYOFF_TERMINAL && o.payoff != LPMC_PAYOFF_CALL)
    return fail(err, LPMC_INVALID_ARGUMENT, "bad payoff");
  if (o.reduce != LPMC_REDUCE_TREE && o.reduce != LPMC_REDUCE_SEQUENTIAL)
    return fail(err, LPMC_INVALID_ARGUMENT, "bad reduction mode");
  if (prec->ieee_half && m != 10)
    return fail(err, LPMC_INVALID_ARGUMENT, "ieee_half requires mantissa_bits == 10");
  if (o.exact_z != LPMC_EXACT_Z_FAST && o.exact_z != LPMC_EXACT_Z_GLIBC)
    return fail(err, LPMC_INVALID_ARGUMENT, "bad exact_z mode");
  if (o.n_devices < 0 || (o.n_devices > 0 && o.devices == nullptr) || o.n_devices > 1024)
    return fail(err, LPMC_INVALID_ARGUMENT, "bad device list");
  if (o.schedule < LPMC_SCHEDULE_AUTO || o.schedule > LPMC_SCHEDULE_WARP_PER_PATH)
    return fail(err, LPMC_INVALID_ARGUMENT, "bad schedule");

  RunSpec& s = *spec;
  s = RunSpec{};
  s.n_paths = n_paths;
  s.kahan = kahan != 0;
  s.reduce = o.reduce;
  s.device = o.device;
  s.schedule = o.schedule;
  if (o.n_devices > 1) s.devices.assign(o.devices, o.devices + o.n_devices);
  s.ieee = prec->ieee_half != 0;
  if (table != nullptr) {
    const lpmc_status st = prepare_table(table, &s.table, err);
    if (st != LPMC_OK) return st;
    s.has_table = true;
  }
  LevelArgs& A = s.args;
  A.seed_key = seed_key_of(seed);  // hoisted out of every path
  A.path_base = path_base;
  A.n_paths = n_paths;
  A.level = level;
  A.legs = static_cast<int32_t>(o.legs);
  A.exact_z = o.exact_z;
  A.counter0 = o.counter;
  A.err_step_bits = err_step_bits_for(level);
  if (n_paths > (1ull << (62 - A.err_step_bits)))  // failure key layout (lpmc_internal.h)
    return fail(err, LPMC_INVALID_ARGUMENT,
                "n_paths too large for the failure record: at most 2^(62 - max(22, level))");
  // per-level constants (sde.hpp:217-224)
  const double dtf = std::ldexp(model->horizon, -level);
  const double sdtf = std::sqrt(dtf);
  const double dtc = 2.0 * dtf;
  A.mu = model->mu;
  A.sigma = model->sigma;
  A.x0 = model->x0;
  A.dtf = dtf;
  A.sdtf = sdtf;
  A.dtc = dtc;
  const double consts[6] = {model->mu, model->sigma, model->x0, dtf, sdtf, dtc};
  double low[6];
  for (int i = 0; i < 6; ++i) {
    if (!std::isfinite(consts[i]))
      return fail(err, LPMC_DOMAIN_ERROR, "non-finite operand", LPMC_FAIL_NONFINITE, path_base, 0);
    if (s.ieee) {
      low[i] = 0.0;
    } else if (!round_prec(consts[i], m, &low[i])) {
      return fail(err, LPMC_DOMAIN_ERROR, "non-finite operand", LPMC_FAIL_NONFINITE, path_base, 0);
    }
  }
  A.mu_l = low[0];
  A.sigma_l = low[1];
  A.x0_l = low[2];
  A.dtf_l = low[3];
  A.sdtf_l = low[4];
  A.dtc_l = low[5];
  A.h_mu = half_bits(consts[0]);
  A.h_sigma = half_bits(consts[1]);
  A.h_x0 = half_bits(consts[2]);
  A.h_dtf = half_bits(consts[3]);
  A.h_sdtf = half_bits(consts[4]);
  A.h_dtc = half_bits(consts[5]);
  A.mantissa_bits = m;
  A.payoff = o.payoff;
  A.strike = o.strike;
  if (s.has_table) {
    A.K = s.table.K;
    A.degree = s.table.degree;
    A.dyadic = s.table.dyadic;
    A.table_stride = s.table.stride;
    A.table_words = static_cast<int32_t>(s.table.rows.size());
    A.table_simple = s.table.simple;
    A.tail = s.table.tail;
  }
  // bar arithmetic; native fp32 paths only inside the guarded range
  const bool native_ok = in_native_range(low[0], 0x1p-20, 0x1p20) &&
                         in_native_range(low[1], 0x1p-20, 0x1p20) &&
                         in_native_range(low[2], 0x1p-20, 0x1p20) &&
                         in_native_range(low[3], 0x1p-40, 0x1p20) &&
                         in_native_range(low[4], 0x1p-20, 0x1p20) &&
                         in_native_range(low[5], 0x1p-40, 0x1p20);
  if (o.legs == LPMC_LEGS_HAT) {
    s.arith = BarArith::kCarrier;  // carrier legs only: the bar arithmetic is never run
  } else if (s.ieee) {
    s.arith = BarArith::kHalf2;
  } else if (m >= 52) {
    s.arith = BarArith::kCarrier;
  } else if (m == 23 && native_ok) {
    s.arith = BarArith::kF32;
  } else if (m <= 10 && native_ok) {
    s.arith = BarArith::kF32Round;
  } else {
    s.arith = BarArith::kF64Round;
  }
  // Power-of-two steps (T = 1 and an even level: dt, 2dt and sqrt(dt) are
  // powers of two): the native fp32 bar legs may fold them into the model
  // constants, R(R(mu x) dt) = R(x (mu dt)) etc., bitwise within the native
  // range guard (every intermediate stays normal; lpmc_level.cuh, step_bar_pw).
  auto pow2 = [](double v) {
    int e = 0;
    return v > 0.0 && std::frexp(v, &e) == 0.5;
  };
  // The carrier legs fold the same way (step_hat_pw): the carrier's own dt,
  // 2dt, sqrt(dt) must be powers of two as well, and mu, sigma and the folded
  // products far inside the binary64 range (RangeF64's argument).
  auto mid_range = [](double v) {
    const double a = std::fabs(v);
    return v == 0.0 || (a >= 0x1p-200 && a <= 0x1p200);
  };
  const bool hat_ok = pow2(A.dtf) && pow2(A.sdtf) && pow2(A.dtc) && mid_range(A.mu) &&
                      mid_range(A.sigma) && std::fabs(A.mu * A.dtc) <= 0x1p10 &&
                      std::fabs(A.sigma * A.sdtf) <= 0x1p10 && mid_range(A.mu * A.dtf) &&
                      mid_range(A.sigma * A.sdtf);
  // (binary64 bar legs -- the carrier arithmetic -- fold under the same proof)
  const bool carrier_ok = s.arith == BarArith::kCarrier && mid_range(low[0]) &&
                          mid_range(low[1]) && mid_range(low[2]) && low[2] != 0.0 &&
                          mid_range(low[0] * low[3]) && mid_range(low[1] * low[4]);
  if ((s.arith == BarArith::kF32 || s.arith == BarArith::kF32Round || carrier_ok) &&
      pow2(low[3]) && pow2(low[4]) && pow2(low[5]) && hat_ok) {
    A.bar_pow2 = 1;
    A.mu_dtf_l = low[0] * low[3];  // exact: a power-of-two scaling
    A.mu_dtc_l = low[0] * low[5];
    A.sg_sdt_l = low[1] * low[4];
    A.hat_mu_dtf = A.mu * A.dtf;
    A.hat_mu_dtc = A.mu * A.dtc;
    A.hat_sg_sdt = A.sigma * A.sdtf;
  }
  // A/B and stress checks (tools/stress_native.py): the unfolded kernels
  if (A.bar_pow2 != 0 && std::getenv("LPMC_NO_POW2") != nullptr) A.bar_pow2 = 0;
  // m = 10 on native binary16 with static power-of-two scales
  // (dev::ArithHalfScaled): dt and 2dt powers of two, every mantissa and
  // scale factor an exact binary16 number, P1 = 4 by the choice of kz, the
  // scaled Gaussians far from binary16's overflow, x0 inside the guard.
  if (s.arith == BarArith::kF32Round && m == 10 && pow2(low[3]) && low[5] == 2.0 * low[3] &&
      low[0] != 0.0 && low[1] != 0.0 && low[4] > 0.0) {
    int e_mu = 0, e_sg = 0, e_sdt = 0, e_dt = 0;
    const double mu_m = 2.0 * std::frexp(low[0], &e_mu);  // mantissa in [1, 2), sign kept
    const double sg_m = 2.0 * std::frexp(low[1], &e_sg);
    const double sdt_m = 2.0 * std::frexp(low[4], &e_sdt);
    std::frexp(low[3], &e_dt);
    e_mu -= 1, e_sg -= 1, e_sdt -= 1, e_dt -= 1;
    const int kz = 2 - e_mu - e_dt + e_sg + e_sdt;  // P1 = 2^(e_mu + e_dt - e_d) = 4
    const int e_d = e_sg + e_sdt - kz;
    double zmax = 8.5;  // exact Gaussians of draws u >= 2^-54
    if (s.has_table) {
      zmax = std::fabs(s.table.tail);
      const size_t rec = s.table.dyadic ? kDyadicRecord : static_cast<size_t>(s.table.stride);
      const size_t nrec = s.table.dyadic ? kDyadicRecords : static_cast<size_t>(s.table.K);
      for (size_t j = 0; j < nrec; ++j) {
        const double* r = s.table.rows.data() + rec * j;
        zmax = std::max(zmax, std::fabs(r[2]) + std::fabs(r[3]));
      }
    }
    // 1 / P2 = 2^-e_d as two binary16 powers of two (the Kahan compensation)
    const int q1e = -e_d > 12 ? 12 : -e_d;
    const int q2e = -e_d - q1e;
    uint16_t hx0 = 0;
    const bool ok = exact_half(std::ldexp(1.0, q1e), &A.hs_q1) &&
                    exact_half(std::ldexp(1.0, q2e), &A.hs_q2) && q1e >= -10 && q2e >= 0 &&
                    kz >= 0 && kz <= 13 && std::ldexp(zmax, kz) <= 30000.0 && e_d >= -24 &&
                    e_d <= 14 && exact_half(mu_m, &A.hs_mu) && exact_half(sg_m, &A.hs_sigma) &&
                    exact_half(sdt_m, &A.hs_sdt) && exact_half(std::ldexp(1.0, e_d), &A.hs_p2) &&
                    exact_half(low[2], &hx0) && hx0 == A.h_x0 && std::fabs(low[2]) >= 0x1p-4 &&
                    std::fabs(low[2]) < 0x1p14;
    if (ok) {
      A.hs_native = 1;
      A.hs_p1 = 0x4400;   // 4
      A.hs_p1c = 0x4800;  // 8 (2 dt)
      A.hs_zscale = std::ldexp(1.0, kz);
    }
  }
  const uint64_t n_chunks = (n_paths + kChunkPaths - 1) / kChunkPaths;
  s.chunk_begin = 0;
  s.chunk_end = n_chunks;
  return LPMC_OK;
}

// --------------------------------------------------- device state ----------
template <typename T>
struct DevBuf {
  T* ptr = nullptr;
  size_t cap = 0;
  cudaError_t ensure(size_t n) {
    if (n <= cap) return cudaSuccess;
    if (ptr != nullptr) cudaFree(ptr);
    ptr = nullptr;
    cap = 0;
    const size_t want = std::max(n, static_cast<size_t>(16));
    cudaError_t e = cudaMalloc(reinterpret_cast<void**>(&ptr), want * sizeof(T));
    if (e == cudaSuccess) cap = want;
    return e;
  }
  void release() {
    if (ptr != nullptr) cudaFree(ptr);
    ptr = nullptr;
    cap = 0;
  }
};

struct Buffers {
  DevBuf<double> table, batch_acc, chunk_acc, path_diff, seq_acc, io_in, io_out;
  DevBuf<unsigned long long> err_key, counts;
  DevBuf<unsigned int> range_flag;
  std::vector<double> host_parts;
  void release() {
    io_in.release();
    io_out.release();
    counts.release();
    table.release();
    batch_acc.release();
    chunk_acc.release();
    path_diff.release();
    seq_acc.release();
    err_key.release();
    range_flag.release();
  }
};

// Streams and buffer sets for concurrent runs (lpmc_run_coupled_many), plus
// a pinned staging area for their asynchronous read-backs.
constexpr int kPoolStreams = 16;
struct StreamPool {
  cudaStream_t streams[kPoolStreams] = {};
  Buffers bufs[kPoolStreams];
  cudaEvent_t start = nullptr;
  double* pinned = nullptr;
  size_t pinned_cap = 0;  // doubles
};

struct DeviceCtx {
  std::mutex mu;
  cudaStream_t stream = nullptr;
  Buffers scratch;
  StreamPool pool;
  bool configured = false;
};

std::mutex g_ctx_mu;
std::map<int, std::unique_ptr<DeviceCtx>> g_ctx;

struct DeviceGuard {
  int prev = -1;
  bool changed = false;
  cudaError_t set(int dev) {
    cudaError_t e = cudaGetDevice(&prev);
    if (e != cudaSuccess) return e;
    if (dev >= 0 && dev != prev) {
      e = cudaSetDevice(dev);
      changed = e == cudaSuccess;
    }
    return e;
  }
  ~DeviceGuard() {
    if (changed) cudaSetDevice(prev);
  }
};

lpmc_status get_ctx(int device, DeviceCtx** out, int* resolved, lpmc_error* err) {
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0)
    return fail(err, LPMC_NO_DEVICE, "no CUDA device available (the sampler has no CPU fallback)");
  int dev = device;
  if (dev < 0) {
    e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(err, e, "cudaGetDevice");
  }
  if (dev >= count) return fail(err, LPMC_INVALID_ARGUMENT, "device ordinal out of range");
  std::lock_guard<std::mutex> lock(g_ctx_mu);
  auto& slot = g_ctx[dev];
  if (!slot) {
    cudaDeviceProp prop{};
    e = cudaGetDeviceProperties(&prop, dev);
    if (e != cudaSuccess) return cuda_fail(err, e, "cudaGetDeviceProperties");
    if (prop.major != 10)
      return fail(err, LPMC_NO_DEVICE, "device is not sm_100 (B200); kernels are built for sm_100a only");
    auto ctx = std::make_unique<DeviceCtx>();
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(dev);
    e = cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = static_cast<cudaError_t>(configure_kernels());
    cudaSetDevice(prev);
    if (e != cudaSuccess) return cuda_fail(err, e, "device setup");
    ctx->configured = true;
    slot = std::move(ctx);
  }
  *out = slot.get();
  *resolved = dev;
  return LPMC_OK;
}

// -------------------------------------------------------- enqueue ----------
struct Enqueued {
  uint64_t n_chunks = 0;        // chunk partials produced (tree)
  uint64_t n_batches_seq = 0;   // batch accumulators produced (sequential)
  int kernels = 0;
};

// Grow B to what enqueue_run(s) needs (no-op when already large enough).
// Runs sharing a buffer set on one stream reserve up front, so no buffer is
// reallocated under an in-flight kernel.
cudaError_t reserve(const RunSpec& s, Buffers& B) {
  cudaError_t e;
  if ((e = B.err_key.ensure(1)) != cudaSuccess) return e;
  if ((e = B.range_flag.ensure(1)) != cudaSuccess) return e;
  if (s.has_table && (e = B.table.ensure(s.table.rows.size())) != cudaSuccess) return e;
  const uint64_t chunks = s.chunk_end - s.chunk_begin;
  if (chunks == 0) return cudaSuccess;
  if (s.reduce == LPMC_REDUCE_SEQUENTIAL) {
    const uint64_t n_batches_total = (s.n_paths + kBatch - 1) / kBatch;
    const uint64_t b0 = s.chunk_begin * kChunkBatches;
    const uint64_t b1 = std::min(s.chunk_end * kChunkBatches, n_batches_total);
    if ((e = B.seq_acc.ensure(15 * (b1 - b0))) != cudaSuccess) return e;
    return B.path_diff.ensure(2 * std::min(b1 - b0, kSeqSliceChunks * kChunkBatches) * kBatch);
  }
  if ((e = B.chunk_acc.ensure(15 * chunks)) != cudaSuccess) return e;
  if (use_wpp(s) &&
      (e = B.path_diff.ensure(2 * std::min(chunks, kSliceChunks) * kChunkBatches * kBatch)) !=
          cudaSuccess)
    return e;
  return B.batch_acc.ensure(15 * std::min(chunks, kSliceChunks) * kChunkBatches);
}

// Accumulators a run produces (chunk partials, or batch accumulators in the
// sequential mode).
uint64_t acc_count_of(const RunSpec& s) {
  if (s.reduce != LPMC_REDUCE_SEQUENTIAL) return s.chunk_end - s.chunk_begin;
  const uint64_t n_batches_total = (s.n_paths + kBatch - 1) / kBatch;
  return std::min(s.chunk_end * kChunkBatches, n_batches_total) - s.chunk_begin * kChunkBatches;
}

// NVTX ranges (header-only NVTX3: no-ops unless a tool such as nsys or ncu
// injects itself): one per level enqueue, one per host fold.
struct NvtxRange {
  explicit NvtxRange(const char* msg) { nvtxRangePushA(msg); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

cudaError_t enqueue_run(const RunSpec& s, Buffers& B, cudaStream_t st, Enqueued* q) {
  char label[96];
  std::snprintf(label, sizeof label, "lpmc level %d m=%d%s legs=%d chunks [%llu,%llu)",
                s.args.level, s.args.mantissa_bits, s.kahan ? " kahan" : "", s.args.legs,
                static_cast<unsigned long long>(s.chunk_begin),
                static_cast<unsigned long long>(s.chunk_end));
  const NvtxRange range(label);
  cudaError_t e;
  *q = Enqueued{};
  if ((e = reserve(s, B)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(B.err_key.ptr, 0xff, sizeof(unsigned long long), st)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(B.range_flag.ptr, 0, sizeof(unsigned int), st)) != cudaSuccess) return e;
  LevelArgs A = s.args;
  A.err_key = B.err_key.ptr;
  A.range_flag = B.range_flag.ptr;
  A.table = nullptr;
  if (s.has_table) {
    if ((e = cudaMemcpyAsync(B.table.ptr, s.table.rows.data(), s.table.rows.size() * sizeof(double),
                             cudaMemcpyHostToDevice, st)) != cudaSuccess)
      return e;
    A.table = B.table.ptr;
  }
  const uint64_t n_batches_total = (s.n_paths + kBatch - 1) / kBatch;
  const uint64_t chunks = s.chunk_end - s.chunk_begin;
  if (chunks == 0) return cudaSuccess;
  const bool seq = s.reduce == LPMC_REDUCE_SEQUENTIAL;
  const bool wpp = use_wpp(s);
  const uint64_t slice_chunks = seq ? kSeqSliceChunks : kSliceChunks;
  if (seq) {
    q->n_batches_seq = acc_count_of(s);
  } else {
    q->n_chunks = chunks;
  }
  for (uint64_t c0 = s.chunk_begin; c0 < s.chunk_end; c0 += slice_chunks) {
    const uint64_t c1 = std::min(c0 + slice_chunks, s.chunk_end);
    const uint64_t b0 = c0 * kChunkBatches;
    const uint64_t b1 = std::min(c1 * kChunkBatches, n_batches_total);
    LevelArgs S = A;
    S.batch0 = b0;
    S.n_batches = b1 - b0;
    S.batch_acc = seq ? nullptr : B.batch_acc.ptr;
    S.path_diff = seq ? B.path_diff.ptr : nullptr;
    S.path_out = nullptr;
    S.z_out = nullptr;
    LaunchResult r;
    if (wpp) {  // per-path differences, then the fused kernel's batch tree over them
      S.batch_acc = nullptr;
      S.path_diff = B.path_diff.ptr;
      r = launch_paths_wpp(S, s.arith, s.kahan, st);
      q->kernels += r.kernels;
      if (r.cuda_error != 0) return static_cast<cudaError_t>(r.cuda_error);
      if (!seq) {
        const uint64_t paths_slice = std::min(b1 * kBatch, s.n_paths) - b0 * kBatch;
        r = launch_path_batches(B.path_diff.ptr, paths_slice, B.batch_acc.ptr, st);
      }
    } else {
      r = launch_paths(S, s.arith, s.kahan, false, st);
    }
    q->kernels += r.kernels;
    if (r.cuda_error != 0) return static_cast<cudaError_t>(r.cuda_error);
    if (seq) {
      const uint64_t paths_slice = std::min(b1 * kBatch, s.n_paths) - b0 * kBatch;
      r = launch_sequential_batches(B.path_diff.ptr, paths_slice,
                                    B.seq_acc.ptr + 15 * (b0 - s.chunk_begin * kChunkBatches), st);
    } else {
      r = launch_chunk_reduce(B.batch_acc.ptr, b1 - b0, c1 - c0,
                              B.chunk_acc.ptr + 15 * (c0 - s.chunk_begin), st);
    }
    q->kernels += r.kernels;
    if (r.cuda_error != 0) return static_cast<cudaError_t>(r.cuda_error);
  }
  t_launches += static_cast<uint64_t>(q->kernels);
  return cudaSuccess;
}

// Map the device failure word to the reference's exception (first failing
// path in path order, as the serial reference would throw).
lpmc_status failure_from_key(const RunSpec& s, unsigned long long key, lpmc_error* err) {
  const int bits = s.args.err_step_bits;
  const uint64_t local = key >> (bits + 2);
  const int kind = static_cast<int>((key >> bits) & 3u);
  const uint64_t step = key & ((1ull << bits) - 1);
  const uint64_t path = s.args.path_base + local;
  if (kind == LPMC_FAIL_UNIFORM_IS_ONE)
    return fail(err, LPMC_DOMAIN_ERROR, "exact_inv_cdf requires u in (0, 1)", kind, path, step);
  if (kind == LPMC_FAIL_NONFINITE_STATE)
    return fail(err, LPMC_RUNTIME_ERROR, "non-finite state at step " + std::to_string(step), kind,
                path, step);
  return fail(err, LPMC_DOMAIN_ERROR, "non-finite operand", LPMC_FAIL_NONFINITE, path, step);
}

uint64_t acc_count(const Enqueued& q) { return q.n_batches_seq ? q.n_batches_seq : q.n_chunks; }

// Device -> host copies of an enqueued run's failure word, range flag and
// partials into caller memory (pinned for an asynchronous copy).
cudaError_t enqueue_readback(const Enqueued& q, const Buffers& B, cudaStream_t st,
                             unsigned long long* key, unsigned int* range, double* parts) {
  cudaError_t e = cudaMemcpyAsync(key, B.err_key.ptr, sizeof *key, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(range, B.range_flag.ptr, sizeof *range, cudaMemcpyDeviceToHost, st);
  const uint64_t n_acc = acc_count(q);
  const double* src = q.n_batches_seq ? B.seq_acc.ptr : B.chunk_acc.ptr;
  if (e == cudaSuccess && n_acc > 0)
    e = cudaMemcpyAsync(parts, src, 15 * n_acc * sizeof(double), cudaMemcpyDeviceToHost, st);
  return e;
}

// Failure flags and partials of a finished run.  *rerun set when native
// legs left their range (the caller re-runs with the exact emulation).
lpmc_status interpret_run(const RunSpec& s, uint64_t n_acc, unsigned long long key,
                          unsigned int range, const double* host, std::vector<Moments>* parts,
                          bool* rerun, lpmc_error* err) {
  *rerun = false;
  if (range != 0 && (s.arith == BarArith::kF32 || s.arith == BarArith::kF32Round)) {
    *rerun = true;
    return LPMC_OK;
  }
  if (key != ~0ull) return failure_from_key(s, key, err);
  parts->resize(3 * n_acc);
  for (uint64_t i = 0; i < 3 * n_acc; ++i) (*parts)[i] = from_device(host + 5 * i);
  return LPMC_OK;
}

// Wait, check failure flags, copy partials back.
lpmc_status collect_run(const RunSpec& s, Buffers& B, cudaStream_t st, const Enqueued& q,
                        std::vector<Moments>* parts, bool* rerun, lpmc_error* err) {
  unsigned long long key = ~0ull;
  unsigned int range = 0;
  B.host_parts.resize(15 * acc_count(q));
  cudaError_t e = enqueue_readback(q, B, st, &key, &range, B.host_parts.data());
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_fail(err, e, "level sampler");
  return interpret_run(s, acc_count(q), key, range, B.host_parts.data(), parts, rerun, err);
}

void mask_legs(const RunSpec& s, std::vector<Moments>& parts) {
  const int legs = s.args.legs;
  for (size_t i = 0; i < parts.size(); ++i) {
    const int f = static_cast<int>(i % 3);
    const bool keep = legs == LPMC_LEGS_FINE ||
                      (f == 0 ? (legs & 1) : (f == 1 ? (legs & 2) : ((legs & 3) == 3)));
    if (!keep) parts[i] = Moments{};
  }
}

// ------------------------------------------------ several devices -------
// Runs sharded over the devices of one process: run i's chunk range splits
// into one contiguous sub-range per listed device (device of sub-range k =
// list[(k + i) mod n], so one-chunk runs rotate over the devices); each
// device's sub-runs go round-robin to its stream pool with that slot's
// buffers; read-backs land in one portable pinned staging area; the host
// waits once, then interprets runs in list order and sub-runs in chunk
// order -- the first failure is the serial one, and the concatenated
// partials are exactly one device's (chunk partials do not depend on where
// they are computed).  A sub-run whose native legs left their range is
// re-run alone in the exact emulation (bitwise what a full re-run gives).
struct MultiStage {
  std::mutex mu;
  double* ptr = nullptr;
  size_t cap = 0;  // doubles
};
MultiStage g_multi_stage;

lpmc_status run_multi_device(std::vector<RunSpec>& specs, const std::vector<int>& devs,
                             std::vector<std::vector<Moments>>* out, lpmc_error* err) {
  out->assign(specs.size(), {});
  const size_t nd = devs.size();
  // contexts of the distinct devices, locked in ascending order
  std::map<int, DeviceCtx*> ctxs;
  for (int d : devs) {
    if (ctxs.count(d)) continue;
    DeviceCtx* ctx = nullptr;
    int resolved = -1;
    const lpmc_status stt = get_ctx(d, &ctx, &resolved, err);
    if (stt != LPMC_OK) return stt;
    ctxs[resolved] = ctx;
  }
  std::lock_guard<std::mutex> stage_lock(g_multi_stage.mu);
  std::vector<std::unique_lock<std::mutex>> locks;
  for (auto& kv : ctxs) locks.emplace_back(kv.second->mu);
  DeviceGuard guard;  // restores the caller's current device on return
  cudaError_t e = guard.set(-1);
  if (e != cudaSuccess) return cuda_fail(err, e, "cudaGetDevice");
  guard.changed = true;

  struct Sub {
    size_t run;
    int dev, slot;
    RunSpec spec;
    Enqueued q;
    size_t off;
  };
  std::vector<Sub> subs;
  std::map<int, int> next_slot;
  for (size_t i = 0; i < specs.size(); ++i) {
    const RunSpec& s = specs[i];
    if (s.n_paths == 0) continue;  // mlmc.hpp:75: nothing simulated
    const uint64_t b = s.chunk_begin, n = s.chunk_end - s.chunk_begin;
    for (size_t k = 0; k < nd; ++k) {
      const uint64_t c0 = b + n * k / nd, c1 = b + n * (k + 1) / nd;
      if (c0 == c1) continue;
      int dev = devs[(k + i) % nd];
      if (dev < 0 && cudaGetDevice(&dev) != cudaSuccess) dev = 0;
      Sub u{i, dev, next_slot[dev]++ % kPoolStreams, s, Enqueued{}, 0};
      u.spec.chunk_begin = c0;
      u.spec.chunk_end = c1;
      u.spec.devices.clear();
      subs.push_back(std::move(u));
    }
  }
  size_t total = 0;
  for (Sub& u : subs) {
    u.off = total;
    total += 2 + 15 * acc_count_of(u.spec);
  }
  if (total > g_multi_stage.cap) {
    if (g_multi_stage.ptr != nullptr) cudaFreeHost(g_multi_stage.ptr);
    g_multi_stage.ptr = nullptr;
    g_multi_stage.cap = 0;
    e = cudaHostAlloc(reinterpret_cast<void**>(&g_multi_stage.ptr), total * sizeof(double),
                      cudaHostAllocPortable);
    if (e != cudaSuccess) return cuda_fail(err, e, "pinned staging");
    g_multi_stage.cap = total;
  }
  // streams and buffers (each slot reserved for its largest sub-run first)
  for (Sub& u : subs) {
    StreamPool& P = ctxs.at(u.dev)->pool;
    if ((e = cudaSetDevice(u.dev)) != cudaSuccess) break;
    if (P.streams[u.slot] == nullptr &&
        (e = cudaStreamCreateWithFlags(&P.streams[u.slot], cudaStreamNonBlocking)) != cudaSuccess)
      break;
    if ((e = reserve(u.spec, P.bufs[u.slot])) != cudaSuccess) break;
  }
  for (size_t j = 0; j < subs.size() && e == cudaSuccess; ++j) {
    Sub& u = subs[j];
    StreamPool& P = ctxs.at(u.dev)->pool;
    double* stage = g_multi_stage.ptr + u.off;
    if ((e = cudaSetDevice(u.dev)) != cudaSuccess) break;
    e = enqueue_run(u.spec, P.bufs[u.slot], P.streams[u.slot], &u.q);
    if (e == cudaSuccess)
      e = enqueue_readback(u.q, P.bufs[u.slot], P.streams[u.slot],
                           reinterpret_cast<unsigned long long*>(stage),
                           reinterpret_cast<unsigned int*>(stage + 1), stage + 2);
  }
  for (auto& kv : ctxs) {
    if (cudaSetDevice(kv.first) != cudaSuccess) continue;
    for (int k = 0; k < kPoolStreams; ++k)
      if (kv.second->pool.streams[k] != nullptr) {
        const cudaError_t s2 = cudaStreamSynchronize(kv.second->pool.streams[k]);
        if (e == cudaSuccess) e = s2;
      }
  }
  if (e != cudaSuccess) return cuda_fail(err, e, "level sampler");
  for (Sub& u : subs) {
    const double* stage = g_multi_stage.ptr + u.off;
    unsigned long long key;
    unsigned int range;
    std::memcpy(&key, stage, sizeof key);
    std::memcpy(&range, stage + 1, sizeof range);
    std::vector<Moments> parts;
    bool rerun = false;
    lpmc_status stt = interpret_run(u.spec, acc_count(u.q), key, range, stage + 2, &parts, &rerun,
                                    err);
    if (stt != LPMC_OK) return stt;
    if (rerun) {
      StreamPool& P = ctxs.at(u.dev)->pool;
      if ((e = cudaSetDevice(u.dev)) != cudaSuccess) return cuda_fail(err, e, "cudaSetDevice");
      u.spec.arith = BarArith::kF64Round;
      Enqueued q2;
      e = enqueue_run(u.spec, P.bufs[u.slot], P.streams[u.slot], &q2);
      if (e != cudaSuccess) return cuda_fail(err, e, "fallback launch");
      stt = collect_run(u.spec, P.bufs[u.slot], P.streams[u.slot], q2, &parts, &rerun, err);
      if (stt != LPMC_OK) return stt;
    }
    auto& dst = (*out)[u.run];
    dst.insert(dst.end(), parts.begin(), parts.end());
  }
  for (size_t i = 0; i < specs.size(); ++i) mask_legs(specs[i], (*out)[i]);
  return ok(err);
}

// Full synchronous run on one device: enqueue, collect, fallback re-run.
lpmc_status run_sync(RunSpec& s, void* user_stream, std::vector<Moments>* parts, lpmc_error* err) {
  if (s.devices.size() > 1) {
    std::vector<RunSpec> one(1, s);
    std::vector<std::vector<Moments>> out;
    const lpmc_status st = run_multi_device(one, s.devices, &out, err);
    if (st == LPMC_OK) *parts = std::move(out[0]);
    return st;
  }
  DeviceCtx* ctx = nullptr;
  int dev = -1;
  lpmc_status stt = get_ctx(s.device, &ctx, &dev, err);
  if (stt != LPMC_OK) return stt;
  DeviceGuard guard;
  cudaError_t e = guard.set(dev);
  if (e != cudaSuccess) return cuda_fail(err, e, "cudaSetDevice");
  std::lock_guard<std::mutex> lock(ctx->mu);
  cudaStream_t st = user_stream != nullptr ? static_cast<cudaStream_t>(user_stream) : ctx->stream;
  for (int attempt = 0; attempt < 2; ++attempt) {
    Enqueued q;
    e = enqueue_run(s, ctx->scratch, st, &q);
    if (e != cudaSuccess) return cuda_fail(err, e, "launch");
    bool rerun = false;
    stt = collect_run(s, ctx->scratch, st, q, parts, &rerun, err);
    if (stt != LPMC_OK) return stt;
    if (!rerun) {
      mask_legs(s, *parts);
      return ok(err);
    }
    s.arith = BarArith::kF64Round;  // exact emulation outside the native range
  }
  return fail(err, LPMC_RUNTIME_ERROR, "native range fallback did not converge");
}

// Independent runs on one device, concurrently: run i goes to pool stream
// i % kPoolStreams with that slot's buffers (reserved for the slot's largest
// run first), every run's read-back is enqueued behind its kernels, and the
// host waits once.  Results are then interpreted in list order, so the
// first failure reported is the one a serial loop would hit first; a run
// whose native legs left their range is re-run in the exact emulation.
lpmc_status run_many(std::vector<RunSpec>& specs, void* user_stream,
                     std::vector<std::vector<Moments>>* out, lpmc_error* err) {
  out->assign(specs.size(), {});
  if (specs.empty()) return ok(err);
  for (const RunSpec& s : specs)
    if (s.devices.size() > 1) return run_multi_device(specs, s.devices, out, err);
  DeviceCtx* ctx = nullptr;
  int dev = -1;
  lpmc_status stt = get_ctx(specs[0].device, &ctx, &dev, err);
  if (stt != LPMC_OK) return stt;
  DeviceGuard guard;
  cudaError_t e = guard.set(dev);
  if (e != cudaSuccess) return cuda_fail(err, e, "cudaSetDevice");
  std::lock_guard<std::mutex> lock(ctx->mu);
  StreamPool& P = ctx->pool;
  const size_t n = specs.size();
  const int used = static_cast<int>(std::min<size_t>(n, kPoolStreams));
  for (int k = 0; k < used && e == cudaSuccess; ++k)
    if (P.streams[k] == nullptr) e = cudaStreamCreateWithFlags(&P.streams[k], cudaStreamNonBlocking);
  if (e == cudaSuccess && P.start == nullptr)
    e = cudaEventCreateWithFlags(&P.start, cudaEventDisableTiming);
  if (e != cudaSuccess) return cuda_fail(err, e, "stream pool");
  // staging layout per run: key, range, 15 doubles per accumulator
  std::vector<size_t> off(n + 1, 0);
  for (size_t i = 0; i < n; ++i)
    off[i + 1] = off[i] + 2 + (specs[i].n_paths ? 15 * acc_count_of(specs[i]) : 0);
  if (off[n] > P.pinned_cap) {
    if (P.pinned != nullptr) cudaFreeHost(P.pinned);
    P.pinned = nullptr;
    P.pinned_cap = 0;
    e = cudaMallocHost(reinterpret_cast<void**>(&P.pinned), off[n] * sizeof(double));
    if (e != cudaSuccess) return cuda_fail(err, e, "pinned staging");
    P.pinned_cap = off[n];
  }
  for (size_t i = 0; i < n && e == cudaSuccess; ++i)
    if (specs[i].n_paths) e = reserve(specs[i], P.bufs[i % kPoolStreams]);
  if (e == cudaSuccess && user_stream != nullptr) {
    e = cudaEventRecord(P.start, static_cast<cudaStream_t>(user_stream));
    for (int k = 0; k < used && e == cudaSuccess; ++k) e = cudaStreamWaitEvent(P.streams[k], P.start, 0);
  }
  std::vector<Enqueued> q(n);
  for (size_t i = 0; i < n && e == cudaSuccess; ++i) {
    if (specs[i].n_paths == 0) continue;  // mlmc.hpp:75: nothing simulated
    const int k = static_cast<int>(i % kPoolStreams);
    double* stage = P.pinned + off[i];
    e = enqueue_run(specs[i], P.bufs[k], P.streams[k], &q[i]);
    if (e == cudaSuccess)
      e = enqueue_readback(q[i], P.bufs[k], P.streams[k], reinterpret_cast<unsigned long long*>(stage),
                           reinterpret_cast<unsigned int*>(stage + 1), stage + 2);
  }
  for (int k = 0; k < used; ++k) {
    const cudaError_t s2 = cudaStreamSynchronize(P.streams[k]);
    if (e == cudaSuccess) e = s2;
  }
  if (e != cudaSuccess) return cuda_fail(err, e, "level sampler");
  for (size_t i = 0; i < n; ++i) {
    if (specs[i].n_paths == 0) continue;
    const int k = static_cast<int>(i % kPoolStreams);
    const double* stage = P.pinned + off[i];
    unsigned long long key;
    unsigned int range;
    std::memcpy(&key, stage, sizeof key);
    std::memcpy(&range, stage + 1, sizeof range);
    bool rerun = false;
    stt = interpret_run(specs[i], acc_count(q[i]), key, range, stage + 2, &(*out)[i], &rerun, err);
    if (stt != LPMC_OK) return stt;
    if (rerun) {
      specs[i].arith = BarArith::kF64Round;
      Enqueued q2;
      e = enqueue_run(specs[i], P.bufs[k], P.streams[k], &q2);
      if (e != cudaSuccess) return cuda_fail(err, e, "fallback launch");
      stt = collect_run(specs[i], P.bufs[k], P.streams[k], q2, &(*out)[i], &rerun, err);
      if (stt != LPMC_OK) return stt;
    }
    mask_legs(specs[i], (*out)[i]);
  }
  return ok(err);
}

void fold(const std::vector<Moments>& parts, lpmc_moments* out3) {
  const NvtxRange range("lpmc fold");
  Moments acc[3];
  for (size_t i = 0; i < parts.size(); ++i) merge_into(acc[i % 3], parts[i]);
  for (int f = 0; f < 3; ++f) out3[f] = to_abi(acc[f]);
}

}  // namespace
}  // namespace lpmc_b200

using namespace lpmc_b200;

// ============================================================ C-ABI ========
extern "C" {

int32_t lpmc_abi_version(void) { return LPMC_B200_ABI_VERSION; }

int32_t lpmc_device_count(void) {
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess) return 0;
  int n = 0;
  for (int d = 0; d < count; ++d) {
    cudaDeviceProp p{};
    if (cudaGetDeviceProperties(&p, d) == cudaSuccess && p.major == 10) ++n;
  }
  return n;
}

uint64_t lpmc_launch_count(void) { return t_launches; }
void lpmc_reset_launch_count(void) { t_launches = 0; }

void lpmc_default_options(lpmc_options* o) {
  o->legs = LPMC_LEGS_ALL;
  o->payoff = LPMC_PAYOFF_TERMINAL;
  o->strike = 1.0;
  o->reduce = LPMC_REDUCE_TREE;
  o->device = -1;
  o->stream = nullptr;
  o->exact_z = LPMC_EXACT_Z_FAST;
  o->devices = nullptr;
  o->n_devices = 0;
  o->schedule = LPMC_SCHEDULE_AUTO;
  o->counter = 0;
}

void lpmc_default_cost_model(lpmc_cost_model* c) {  // mlmc.hpp:20-28
  c->cycles_exact_rng = 3.5;
  c->cycles_approx_rng_single = 0.5;
  c->cycles_approx_rng_half = 0.25;
  c->kahan_overhead_factor = 1.4;
  c->per_step_arithmetic = 0.0;
}

lpmc_status lpmc_round_to_precision(double x, int32_t m, double* out, lpmc_error* err) {
  if (out == nullptr) return fail(err, LPMC_INVALID_ARGUMENT, "null argument");
  if (m < 1) return fail(err, LPMC_INVALID_ARGUMENT, "mantissa_bits must be >= 1");
  if (!round_prec(x, m, out)) return fail(err, LPMC_DOMAIN_ERROR, "non-finite operand");
  return ok(err);
}

lpmc_status lpmc_invcdf_build(int32_t kind, int32_t K, double* bp, double* coeff, double* w_max,
                              double* step_w, double* tail, lpmc_error* err) {
  // InvCdfApprox::build (invcdf_approx.hpp:101-145), same op order.
  if (!valid_interval_count(K))
    return fail(err, LPMC_INVALID_ARGUMENT, "interval count must be a power of two >= 2");
  if (kind < 0 || kind > 2) return fail(err, LPMC_INVALID_ARGUMENT, "bad approximation kind");
  std::vector<double> nodes, weights;
  gauss_legendre_rule(32, nodes, weights);
  const double wm = std::min(static_cast<double>(K + 1), 45.0);
  const double sw = (wm - 1.0) / K;
  double left = 0.5;
  for (int j = 0; j < K; ++j) {
    const double w_hi = 1.0 + (j + 1) * sw;
    const double right = 1.0 - std::exp2(-w_hi);
    bp[j] = right;
    std::array<double, 4> c{0.0, 0.0, 0.0, 0.0};
    for (size_t i = 0; i < nodes.size(); ++i) {
      const double t = nodes[i];
      const double u = 0.5 * (left + right) + 0.5 * (right - left) * t;
      const double f = weights[i] * host_phi_inv(u);
      const double p2 = 1.5 * t * t - 0.5;
      const double p3 = t * (2.5 * t * t - 1.5);
      c[0] += 0.5 * f;
      if (kind != LPMC_APPROX_CONSTANT) c[1] += 1.5 * f * t;
      if (kind == LPMC_APPROX_CUBIC) {
        c[2] += 2.5 * f * p2;
        c[3] += 3.5 * f * p3;
      }
    }
    for (int k = 0; k < 4; ++k) coeff[4 * j + k] = c[k];
    left = right;
  }
  const double* last = coeff + 4 * (K - 1);
  *tail = last[0] + last[1] + last[2] + last[3];
  *w_max = wm;
  *step_w = sw;
  return ok(err);
}

// ---- host scheme utilities of the reference API (uniform.hpp, gaussian.hpp,
// quadrature.hpp, softfloat.hpp:129-136, invcdf_approx.hpp:150-185) --------
uint64_t lpmc_stream_word(uint64_t seed, uint64_t path_index, uint64_t counter) {
  // stream_word (uniform.hpp:22-27)
  uint64_t key = host_mix64(seed + 0x9e3779b97f4a7c15ull);
  key = host_mix64(key ^ host_mix64(path_index + 0xbf58476d1ce4e5b9ull));
  return host_mix64(host_mix64(key + counter * 0x94d049bb133111ebull));
}

double lpmc_stream_uniform(uint64_t seed, uint64_t path_index, uint64_t counter) {
  // UniformStream::next (uniform.hpp:38-41): the 53-bit draw offset by half a step
  return static_cast<double>(lpmc_stream_word(seed, path_index, counter) >> 11) * 0x1p-53 +
         0x1p-54;
}

double lpmc_normal_cdf(double x) { return 0.5 * std::erfc(-x * 0.7071067811865475244); }
double lpmc_normal_pdf(double x) { return 0.3989422804014326779 * std::exp(-0.5 * x * x); }

lpmc_status lpmc_exact_inv_cdf(double u, double* out, lpmc_error* err) {
  if (out == nullptr) return fail(err, LPMC_INVALID_ARGUMENT, "null argument");
  if (!(u > 0.0 && u < 1.0))  // gaussian.hpp:59-61
    return fail(err, LPMC_DOMAIN_ERROR, "exact_inv_cdf requires u in (0, 1)");
  *out = host_phi_inv(u);
  return ok(err);
}

double lpmc_inv_cdf_lower(double u) { return host_phi_inv_lower(u); }

lpmc_status lpmc_gauss_legendre(int32_t n, double* nodes, double* weights, lpmc_error* err) {
  if (n < 1 || nodes == nullptr || weights == nullptr)
    return fail(err, LPMC_INVALID_ARGUMENT, "need n >= 1 and output arrays");
  std::vector<double> x, w;
  gauss_legendre_rule(n, x, w);
  std::copy(x.begin(), x.end(), nodes);
  std::copy(w.begin(), w.end(), weights);
  return ok(err);
}

lpmc_status lpmc_ulp_spacing(double x, int32_t m, double* out, lpmc_error* err) {
  if (out == nullptr) return fail(err, LPMC_INVALID_ARGUMENT, "null argument");
  // ulp_spacing (softfloat.hpp:129-136)
  if (!std::isfinite(x)) return fail(err, LPMC_DOMAIN_ERROR, "non-finite operand");
  if (x == 0.0)
    return fail(err, LPMC_DOMAIN_ERROR, "ulp_spacing undefined at zero with an unbounded exponent");
  int e = 0;
  std::frexp(x, &e);
  *out = std::ldexp(1.0, e - 1 - m);
  return ok(err);
}

lpmc_status lpmc_moment_diagnostics(const lpmc_invcdf_table* t, int32_t p_max, double* out,
                                    lpmc_error* err) {
  // moment_diagnostics (invcdf_approx.hpp:150-185), same quadrature and order
  if (t == nullptr || out == nullptr) return fail(err, LPMC_INVALID_ARGUMENT, "null argument");
  if (p_max < 1 || p_max > 8)
    return fail(err, LPMC_INVALID_ARGUMENT, "moment order must be in [1, 8]");
  std::vector<double> nodes, weights;
  gauss_legendre_rule(32, nodes, weights);
  for (int p = 0; p < p_max; ++p) out[p] = 0.0;
  lpmc_status st = LPMC_OK;
  auto accumulate = [&](double a, double b) {
    for (size_t i = 0; i < nodes.size() && st == LPMC_OK; ++i) {
      const double u = 0.5 * (a + b) + 0.5 * (b - a) * nodes[i];
      double z = 0.0;
      st = lpmc_invcdf_eval(t, u, &z, err);
      const double wgt = 0.5 * (b - a) * weights[i];
      double zp = 1.0;
      for (int p = 0; p < p_max; ++p) {
        zp *= z;
        out[p] += wgt * zp;
      }
    }
  };
  double a = 0.5;
  for (int j = 0; j < t->interval_count && st == LPMC_OK; ++j) {
    const double b = t->breakpoints[j];
    accumulate(a, b);
    accumulate(1.0 - b, 1.0 - a);  // mirrored interval
    a = b;
  }
  if (st != LPMC_OK) return st;
  const double tail_mass = 1.0 - t->breakpoints[t->interval_count - 1];
  double zp_hi = 1.0, zp_lo = 1.0;
  for (int p = 0; p < p_max; ++p) {
    zp_hi *= t->tail_value;
    zp_lo *= -t->tail_value;
    out[p] += tail_mass * (zp_hi + zp_lo);
  }
  return ok(err);
}

lpmc_status lpmc_invcdf_eval(const lpmc_invcdf_table* t, double u, double* out, lpmc_error* err) {
  if (t == nullptr || out == nullptr) return fail(err, LPMC_INVALID_ARGUMENT, "null argument");
  // InvCdfApprox::operator() / eval_upper (invcdf_approx.hpp:44-90)
  if (!(u > 0.0 && u < 1.0))
    return fail(err, LPMC_DOMAIN_ERROR, "approx_inv_cdf requires u in (0, 1)");
  if (u == 0.5) {
    *out = 0.0;
    return ok(err);
  }
  const bool lower = u < 0.5;
  const double up = lower ? 1.0 - u : u;
  const int j_or_tail = reference_index(1.0 - up, t->interval_count, t->w_max, t->step_w);
  double r;
  if (j_or_tail == t->interval_count) {
    r = t->tail_value;
  } else {
    const int j = j_or_tail;
    const double a = j == 0 ? 0.5 : t->breakpoints[j - 1];
    const double b = t->breakpoints[j];
    double s = 2.0 * (up - a) / (b - a) - 1.0;
    if (s < -1.0) s = -1.0;
    if (s > 1.0) s = 1.0;
    const double* c = t->coeff + 4 * j;
    const double p2 = 1.5 * s * s - 0.5;
    const double p3 = s * (2.5 * s * s - 1.5);
    r = c[0] + c[1] * s + c[2] * p2 + c[3] * p3;
  }
  *out = lower ? -r : r;
  return ok(err);
}

void lpmc_moments_add(lpmc_moments* acc, double x) {  // stats.hpp:15-27
  const uint64_t prior = acc->n;
  acc->n += 1;
  const double dn = static_cast<double>(acc->n);
  const double delta = x - acc->mean;
  const double dl = delta / dn;
  const double dl2 = dl * dl;
  const double t1 = delta * dl * static_cast<double>(prior);
  acc->mean += dl;
  acc->m4 += t1 * dl2 * (dn * dn - 3.0 * dn + 3.0) + 6.0 * dl2 * acc->m2 - 4.0 * dl * acc->m3;
  acc->m3 += t1 * dl * (dn - 2.0) - 3.0 * dl * acc->m2;
  acc->m2 += t1;
}

void lpmc_moments_merge(lpmc_moments* acc, const lpmc_moments* other) {
  Moments a = from_abi(*acc);
  merge_into(a, from_abi(*other));
  *acc = to_abi(a);
}

void lpmc_fold_partials(const lpmc_moments* partials, uint64_t n_chunks, lpmc_moments* out) {
  const NvtxRange range("lpmc fold partials");
  Moments acc[3];
  for (uint64_t i = 0; i < 3 * n_chunks; ++i) merge_into(acc[i % 3], from_abi(partials[i]));
  for (int f = 0; f < 3; ++f) out[f] = to_abi(acc[f]);
}

void lpmc_level_stats_from_moments(const lpmc_moments* acc3, int32_t level,
                                   const lpmc_precision* prec, int32_t kahan,
                                   const lpmc_cost_model* cost_in, uint64_t n_paths,
                                   lpmc_level_stats* s) {
  // estimate_level_stats (mlmc.hpp:125-148); MomentAccumulator getters
  // (stats.hpp:56-82).
  lpmc_cost_model cost;
  lpmc_default_cost_model(&cost);
  if (cost_in != nullptr) cost = *cost_in;
  auto mean = [](const lpmc_moments& a) { return a.n ? a.mean : 0.0; };
  auto var = [](const lpmc_moments& a) { return a.n < 2 ? 0.0 : a.m2 / static_cast<double>(a.n - 1); };
  auto var_se = [&](const lpmc_moments& a) {
    if (a.n < 2) return 0.0;
    const double v = var(a);
    double spread = a.m4 / static_cast<double>(a.n) - v * v;
    if (spread < 0.0) spread = 0.0;
    return std::sqrt(spread / static_cast<double>(a.n));
  };
  const double n_fine = std::ldexp(1.0, level);
  const double steps = level == 0 ? n_fine : 1.5 * n_fine;
  s->level = level;
  s->mean_hat = mean(acc3[0]);
  s->v_hat = var(acc3[0]);
  s->v_hat_stderr = var_se(acc3[0]);
  s->mean_bar = mean(acc3[1]);
  s->v_bar = var(acc3[1]);
  s->v_bar_stderr = var_se(acc3[1]);
  s->mean_four = mean(acc3[2]);
  s->V_bar = var(acc3[2]);
  s->V_bar_stderr = var_se(acc3[2]);
  const double approx_cycles = prec->mantissa_bits <= 10 ? cost.cycles_approx_rng_half
                                                         : cost.cycles_approx_rng_single;
  s->c_hat = n_fine * cost.cycles_exact_rng + steps * cost.per_step_arithmetic;
  s->c_bar = n_fine * approx_cycles * (kahan ? cost.kahan_overhead_factor : 1.0) +
             steps * cost.per_step_arithmetic;
  s->C_bar = s->c_hat + s->c_bar;
  s->m_hat = s->m_bar = s->M_bar = n_paths;
}

lpmc_status lpmc_run_coupled_paths(const lpmc_gbm* model, int32_t level,
                                   const lpmc_precision* prec, const lpmc_invcdf_table* table,
                                   int32_t kahan, uint64_t n_paths, uint64_t seed,
                                   uint64_t path_base, const lpmc_options* opts,
                                   lpmc_moments* out, lpmc_error* err) {
  if (out == nullptr) return fail(err, LPMC_INVALID_ARGUMENT, "null argument");
  for (int f = 0; f < 3; ++f) out[f] = lpmc_moments{0, 0.0, 0.0, 0.0, 0.0};
  if (n_paths == 0) return ok(err);  // mlmc.hpp:75: no batches, nothing simulated
  RunSpec s;
  lpmc_status st = build_spec(model, level, prec, table, kahan, n_paths, seed, path_base, opts,
                              &s, err);
  if (st != LPMC_OK) return st;
  std::vector<Moments> parts;
  st = run_sync(s, opts ? opts->stream : nullptr, &parts, err);
  if (st != LPMC_OK) return st;
  Moments acc[3];
  for (size_t i = 0; i < parts.size(); ++i) merge_into(acc[i % 3], parts[i]);
  for (int f = 0; f < 3; ++f) out[f] = to_abi(acc[f]);
  return ok(err);
}

lpmc_status lpmc_estimate_level_stats(const lpmc_gbm* model, int32_t level,
                                      const lpmc_precision* prec,
                                      const lpmc_invcdf_table* table, int32_t kahan,
                                      uint64_t n_paths, uint64_t seed,
                                      const lpmc_cost_model* cost, uint64_t path_base,
                                      const lpmc_options* opts, lpmc_level_stats* out,
                                      lpmc_error* err) {
  if (out == nullptr) return fail(err, LPMC_INVALID_ARGUMENT, "null argument");
  if (n_paths < 2) return fail(err, LPMC_INVALID_ARGUMENT, "need at least 2 paths");  // mlmc.hpp:121
  lpmc_moments acc[3];
  lpmc_status st = lpmc_run_coupled_paths(model, level, prec, table, kahan, n_paths, seed,
                                          path_base, opts, acc, err);
  if (st != LPMC_OK) return st;
  lpmc_level_stats_from_moments(acc, level, prec, kahan, cost, n_paths, out);
  return ok(err);
}

lpmc_status lpmc_run_coupled_many(const lpmc_gbm* model, const lpmc_invcdf_table* table,
                                  uint64_t seed, const lpmc_run_desc* runs, uint64_t n_runs,
                                  const lpmc_options* opts, lpmc_moments* out, lpmc_error* err) {
  if (n_runs == 0) return ok(err);
  if (runs == nullptr || out == nullptr)
    return fail(err, LPMC_INVALID_ARGUMENT, "null run list or output");
  for (uint64_t i = 0; i < 3 * n_runs; ++i) out[i] = lpmc_moments{0, 0.0, 0.0, 0.0, 0.0};
  // Specs in list order; a run that cannot even be set up ends the list
  // there (a serial loop would throw at it, after the runs before it).
  std::vector<RunSpec> specs;
  specs.reserve(n_runs);
  lpmc_status setup = LPMC_OK;
  lpmc_error setup_err{};
  for (uint64_t i = 0; i < n_runs; ++i) {
    RunSpec s;
    if (runs[i].n_paths == 0) {  // run_coupled_paths simulates nothing (mlmc.hpp:75)
      s.device = opts != nullptr ? opts->device : -1;
    } else {
      setup = build_spec(model, runs[i].level, &runs[i].prec, table, runs[i].kahan,
                         runs[i].n_paths, seed, runs[i].path_base, opts, &s, &setup_err);
      if (setup != LPMC_OK) break;
    }
    specs.push_back(std::move(s));
  }
  std::vector<std::vector<Moments>> parts;
  lpmc_status st = run_many(specs, opts != nullptr ? opts->stream : nullptr, &parts, err);
  if (st != LPMC_OK) return st;
  if (setup != LPMC_OK) {
    if (err != nullptr) *err = setup_err;
    return setup;
  }
  for (size_t i = 0; i < specs.size(); ++i) fold(parts[i], out + 3 * i);
  return ok(err);
}

lpmc_status lpmc_run_coupled_many_partials(const lpmc_gbm* model, const lpmc_invcdf_table* table,
                                           uint64_t seed, const lpmc_run_desc* runs,
                                           uint64_t n_runs, const uint64_t* chunk_begin,
                                           const uint64_t* chunk_end, const lpmc_options* opts,
                                           lpmc_moments* out, lpmc_error* err) {
  if (n_runs == 0) return ok(err);
  if (runs == nullptr || out == nullptr || chunk_begin == nullptr || chunk_end == nullptr)
    return fail(err, LPMC_INVALID_ARGUMENT, "null run list, chunk range or output");
  lpmc_options o;
  lpmc_default_options(&o);
  if (opts != nullptr) o = *opts;
  o.reduce = LPMC_REDUCE_TREE;  // chunk partials are defined by the tree
  std::vector<RunSpec> specs;
  specs.reserve(n_runs);
  std::vector<uint64_t> off(n_runs + 1, 0);
  for (uint64_t i = 0; i < n_runs; ++i) {
    const uint64_t n_chunks = (runs[i].n_paths + LPMC_CHUNK_PATHS - 1) / LPMC_CHUNK_PATHS;
    if (chunk_end[i] > n_chunks || chunk_begin[i] > chunk_end[i])
      return fail(err, LPMC_INVALID_ARGUMENT, "chunk range outside the run");
    off[i + 1] = off[i] + 3 * (chunk_end[i] - chunk_begin[i]);
  }
  for (uint64_t i = 0; i < off[n_runs]; ++i) out[i] = lpmc_moments{0, 0.0, 0.0, 0.0, 0.0};
  lpmc_status setup = LPMC_OK;
  lpmc_error setup_err{};
  for (uint64_t i = 0; i < n_runs; ++i) {
    RunSpec s;
    if (runs[i].n_paths == 0 || chunk_begin[i] == chunk_end[i]) {
      s.device = o.device;  // nothing simulated on this rank
    } else {
      setup = build_spec(model, runs[i].level, &runs[i].prec, table, runs[i].kahan,
                         runs[i].n_paths, seed, runs[i].path_base, &o, &s, &setup_err);
      if (setup != LPMC_OK) break;
      s.chunk_begin = chunk_begin[i];
      s.chunk_end = chunk_end[i];
    }
    specs.push_back(std::move(s));
  }
  std::vector<std::vector<Moments>> parts;
  lpmc_status st = run_many(specs, o.stream, &parts, err);
  if (st != LPMC_OK) return st;
  if (setup != LPMC_OK) {
    if (err != nullptr) *err = setup_err;
    return setup;
  }
  for (size_t i = 0; i < specs.size(); ++i)
    for (size_t k = 0; k < parts[i].size() && off[i] + k < off[i + 1]; ++k)
      out[off[i] + k] = to_abi(parts[i][k]);
  return ok(err);
}

lpmc_status lpmc_run_two_way_paths(const lpmc_gbm* model, int32_t level,
                                   const lpmc_precision* prec, const lpmc_invcdf_table* table,
                                   int32_t kahan, uint64_t n_paths, uint64_t seed,
                                   uint64_t path_base, const lpmc_options* opts,
                                   lpmc_moments* out, lpmc_error* err) {
  if (out == nullptr) return fail(err, LPMC_INVALID_ARGUMENT, "null argument");
  *out = lpmc_moments{0, 0.0, 0.0, 0.0, 0.0};
  lpmc_options o;
  lpmc_default_options(&o);
  if (opts != nullptr) o = *opts;
  o.legs = LPMC_LEGS_FINE;
  lpmc_moments acc[3];
  const lpmc_status st = lpmc_run_coupled_paths(model, level, prec, table, kahan, n_paths, seed,
                                                path_base, &o, acc, err);
  if (st != LPMC_OK) return st;
  *out = acc[2];  // x_hat - x_bar
  return ok(err);
}

lpmc_status lpmc_allocate_samples(const lpmc_level_stats* stats, uint64_t n_levels, double eps,
                                  int32_t kind, uint64_t* primary, uint64_t* secondary,
                                  int32_t* degenerate, lpmc_error* err) {
  // allocate_samples (mlmc.hpp:165-195): same expressions, same order
  if (stats == nullptr || n_levels == 0) return fail(err, LPMC_INVALID_ARGUMENT, "no level stats");
  if (!(eps > 0.0)) return fail(err, LPMC_INVALID_ARGUMENT, "eps must be positive");
  if (kind != LPMC_ALLOCATION_STANDARD && kind != LPMC_ALLOCATION_NESTED)
    return fail(err, LPMC_INVALID_ARGUMENT, "bad allocation kind");
  const bool nested = kind == LPMC_ALLOCATION_NESTED;
  if (primary == nullptr || (nested && secondary == nullptr))
    return fail(err, LPMC_INVALID_ARGUMENT, "null allocation output");
  double s = 0.0;
  for (uint64_t i = 0; i < n_levels; ++i) {
    const lpmc_level_stats& st = stats[i];
    if (!nested) {
      s += std::sqrt(st.v_hat * st.c_hat);
    } else {
      s += std::sqrt(st.v_bar * st.c_bar) + std::sqrt(st.V_bar * st.C_bar);
    }
  }
  if (degenerate != nullptr) *degenerate = s == 0.0 ? 1 : 0;
  const double scale = 2.0 / (eps * eps) * s;
  for (uint64_t i = 0; i < n_levels; ++i) {
    const lpmc_level_stats& st = stats[i];
    const double v1 = nested ? st.v_bar : st.v_hat;
    const double c1 = nested ? st.c_bar : st.c_hat;
    const double m1 = v1 > 0.0 ? scale * std::sqrt(v1 / c1) : 0.0;
    primary[i] = std::max<uint64_t>(1, static_cast<uint64_t>(std::ceil(m1)));
    if (nested) {
      const double m2 = st.V_bar > 0.0 ? scale * std::sqrt(st.V_bar / st.C_bar) : 0.0;
      secondary[i] = std::max<uint64_t>(1, static_cast<uint64_t>(std::ceil(m2)));
    }
  }
  return ok(err);
}

lpmc_status lpmc_predicted_times(const lpmc_level_stats* stats, uint64_t n_levels, double eps,
                                 double* t_hat, double* t_bar, lpmc_error* err) {
  if (t_hat == nullptr || t_bar == nullptr) return fail(err, LPMC_INVALID_ARGUMENT, "null argument");
  // predicted_times (mlmc.hpp:202-213)
  if (stats == nullptr || n_levels == 0) return fail(err, LPMC_INVALID_ARGUMENT, "no level stats");
  if (!(eps > 0.0)) return fail(err, LPMC_INVALID_ARGUMENT, "eps must be positive");
  double s_hat = 0.0, s_bar = 0.0;
  for (uint64_t i = 0; i < n_levels; ++i) {
    const lpmc_level_stats& st = stats[i];
    s_hat += std::sqrt(st.v_hat * st.c_hat);
    s_bar += std::sqrt(st.v_bar * st.c_bar) + std::sqrt(st.V_bar * st.C_bar);
  }
  const double scale = 2.0 / (eps * eps);
  *t_hat = scale * s_hat * s_hat;
  *t_bar = scale * s_bar * s_bar;
  return ok(err);
}

lpmc_status lpmc_per_level_speedup(const lpmc_level_stats* s, double* value,
                                   int32_t* cost_ratio_only, lpmc_error* err) {
  if (s == nullptr || value == nullptr || cost_ratio_only == nullptr) return fail(err, LPMC_INVALID_ARGUMENT, "null argument");
  // per_level_speedup (mlmc.hpp:223-230)
  if (!(s->v_hat > 0.0) || !(s->c_hat > 0.0))
    return fail(err, LPMC_INVALID_ARGUMENT, "per_level_speedup needs v_hat, c_hat > 0");
  if (s->v_bar == 0.0) {
    *value = s->c_hat / s->c_bar;
    *cost_ratio_only = 1;
    return ok(err);
  }
  const double ratio = (s->v_bar * s->c_bar) / (s->v_hat * s->c_hat);
  const double mix = 1.0 + std::sqrt(s->V_bar * s->C_bar / (s->v_bar * s->c_bar));
  *value = 1.0 / (ratio * mix * mix);
  *cost_ratio_only = 0;
  return ok(err);
}

lpmc_status lpmc_run_nested_estimator(const lpmc_gbm* model, int32_t max_level,
                                      const lpmc_precision* prec,
                                      const lpmc_invcdf_table* table, int32_t kahan, double eps,
                                      uint64_t seed, const lpmc_cost_model* cost,
                                      uint64_t pilot_paths, const lpmc_options* opts,
                                      lpmc_estimator_result* out, lpmc_error* err) {
  // run_nested_estimator (mlmc.hpp:244-283)
  if (out == nullptr || prec == nullptr) return fail(err, LPMC_INVALID_ARGUMENT, "null argument");
  out->value = 0.0;
  out->eps = eps;
  out->t_hat = out->t_bar = 0.0;
  out->degenerate = 0;
  if (max_level < 0) return fail(err, LPMC_INVALID_ARGUMENT, "max level must be >= 0");
  if (pilot_paths < 2) return fail(err, LPMC_INVALID_ARGUMENT, "need at least 2 paths");  // :121
  const uint64_t levels = static_cast<uint64_t>(max_level) + 1;
  auto path_base = [](uint64_t l, uint64_t phase) { return (l << 40) | (phase << 36); };
  lpmc_options o;
  lpmc_default_options(&o);
  if (opts != nullptr) o = *opts;
  o.legs = LPMC_LEGS_ALL;  // the estimator needs all four legs

  std::vector<lpmc_run_desc> runs;
  for (uint64_t l = 0; l < levels; ++l)
    runs.push_back({static_cast<int32_t>(l), *prec, kahan, pilot_paths, path_base(l, 0)});
  std::vector<lpmc_moments> acc(3 * runs.size());
  lpmc_status st = lpmc_run_coupled_many(model, table, seed, runs.data(), runs.size(), &o,
                                         acc.data(), err);
  if (st != LPMC_OK) return st;
  std::vector<lpmc_level_stats> stats(levels);
  for (uint64_t l = 0; l < levels; ++l) {
    lpmc_level_stats_from_moments(&acc[3 * l], static_cast<int32_t>(l), prec, kahan, cost,
                                  pilot_paths, &stats[l]);
    if (out->pilot_stats != nullptr) out->pilot_stats[l] = stats[l];
  }
  std::vector<uint64_t> primary(levels), secondary(levels);
  int32_t degenerate = 0;
  st = lpmc_allocate_samples(stats.data(), levels, eps, LPMC_ALLOCATION_NESTED, primary.data(),
                             secondary.data(), &degenerate, err);
  if (st != LPMC_OK) return st;
  out->degenerate = degenerate;
  st = lpmc_predicted_times(stats.data(), levels, eps, &out->t_hat, &out->t_bar, err);
  if (st != LPMC_OK) return st;
  for (uint64_t l = 0; l < levels; ++l) {
    if (out->primary != nullptr) out->primary[l] = primary[l];
    if (out->secondary != nullptr) out->secondary[l] = secondary[l];
  }

  runs.clear();
  for (uint64_t l = 0; l < levels; ++l) {
    runs.push_back({static_cast<int32_t>(l), *prec, kahan, primary[l], path_base(l, 1)});
    runs.push_back({static_cast<int32_t>(l), *prec, kahan, secondary[l], path_base(l, 2)});
  }
  acc.assign(3 * runs.size(), lpmc_moments{});
  st = lpmc_run_coupled_many(model, table, seed, runs.data(), runs.size(), &o, acc.data(), err);
  if (st != LPMC_OK) return st;
  auto mean = [](const lpmc_moments& a) { return a.n ? a.mean : 0.0; };  // stats.hpp:57
  double value = 0.0;
  for (uint64_t l = 0; l < levels; ++l) {
    const lpmc_moments* two_way = &acc[6 * l];
    const lpmc_moments* four_way = &acc[6 * l + 3];
    const double contribution = mean(two_way[1]) + (mean(four_way[0]) - mean(four_way[1]));
    if (out->level_contributions != nullptr) out->level_contributions[l] = contribution;
    value += contribution;
  }
  out->value = value;
  return ok(err);
}

lpmc_status lpmc_level_partials(const lpmc_gbm* model, int32_t level,
                                const lpmc_precision* prec, const lpmc_invcdf_table* table,
                                int32_t kahan, uint64_t n_paths, uint64_t seed,
                                uint64_t path_base, uint64_t chunk_begin, uint64_t chunk_end,
                                const lpmc_options* opts, lpmc_moments* out, lpmc_error* err) {
  if (out == nullptr) return fail(err, LPMC_INVALID_ARGUMENT, "null argument");
  const uint64_t n_chunks = (n_paths + LPMC_CHUNK_PATHS - 1) / LPMC_CHUNK_PATHS;
  if (chunk_end > n_chunks || chunk_begin > chunk_end)
    return fail(err, LPMC_INVALID_ARGUMENT, "chunk range outside the run");
  if (chunk_begin == chunk_end) return ok(err);
  lpmc_options o;
  lpmc_default_options(&o);
  if (opts != nullptr) o = *opts;
  o.reduce = LPMC_REDUCE_TREE;  // chunk partials are defined by the tree
  RunSpec s;
  lpmc_status st = build_spec(model, level, prec, table, kahan, n_paths, seed, path_base, &o, &s, err);
  if (st != LPMC_OK) return st;
  s.chunk_begin = chunk_begin;
  s.chunk_end = chunk_end;
  std::vector<Moments> parts;
  st = run_sync(s, o.stream, &parts, err);
  if (st != LPMC_OK) return st;
  for (size_t i = 0; i < parts.size(); ++i) out[i] = to_abi(parts[i]);
  return ok(err);
}

lpmc_status lpmc_step_error_probe(const lpmc_gbm* model, int32_t level,
                                  const lpmc_precision* prec, const lpmc_invcdf_table* table,
                                  uint64_t n_samples, uint64_t seed, const lpmc_options* opts,
                                  lpmc_step_error_stats* out, lpmc_error* err) {
  if (out == nullptr) return fail(err, LPMC_INVALID_ARGUMENT, "null argument");
  // step_error_probe (sde.hpp:297-344)
  *out = lpmc_step_error_stats{0.0, 0.0, 0.0, 0.0, 0};
  if (prec != nullptr && prec->ieee_half)
    return fail(err, LPMC_INVALID_ARGUMENT, "step-error probe needs an emulated precision");
  if (level > 40) return fail(err, LPMC_INVALID_ARGUMENT, "level must be <= 40");
  const double nan = std::nan("");
  if (n_samples == 0) {  // no step taken: 0 / 0 (sde.hpp:338-342)
    *out = lpmc_step_error_stats{nan, nan, nan, nan, 0};
    return ok(err);
  }
  const uint64_t n_steps = level >= 0 ? (1ull << level) : 1;
  const uint64_t n_paths = (n_samples + n_steps - 1) / n_steps;
  const uint64_t last_steps = n_samples - (n_paths - 1) * n_steps;
  lpmc_options o;
  lpmc_default_options(&o);
  if (opts != nullptr) o = *opts;
  o.legs = LPMC_LEGS_BAR;
  RunSpec s;
  lpmc_status st = build_spec(model, level, prec, table, 0, n_paths, seed, 0, &o, &s, err);
  if (st != LPMC_OK) return st;
  DeviceCtx* ctx = nullptr;
  int dev = -1;
  st = get_ctx(s.device, &ctx, &dev, err);
  if (st != LPMC_OK) return st;
  DeviceGuard guard;
  cudaError_t e = guard.set(dev);
  if (e != cudaSuccess) return cuda_fail(err, e, "cudaSetDevice");
  std::lock_guard<std::mutex> lock(ctx->mu);
  cudaStream_t stream = o.stream != nullptr ? static_cast<cudaStream_t>(o.stream) : ctx->stream;
  Buffers& B = ctx->scratch;
  const uint64_t blocks = (n_paths + 255) / 256;
  std::vector<double> sums(4 * blocks);
  for (int attempt = 0; attempt < 2; ++attempt) {
    LevelArgs A = s.args;
    if ((e = B.err_key.ensure(1)) != cudaSuccess) break;
    if ((e = B.range_flag.ensure(1)) != cudaSuccess) break;
    if ((e = B.batch_acc.ensure(4 * blocks)) != cudaSuccess) break;
    if ((e = cudaMemsetAsync(B.err_key.ptr, 0xff, sizeof(unsigned long long), stream)) != cudaSuccess) break;
    if ((e = cudaMemsetAsync(B.range_flag.ptr, 0, sizeof(unsigned int), stream)) != cudaSuccess) break;
    A.err_key = B.err_key.ptr;
    A.range_flag = B.range_flag.ptr;
    A.table = nullptr;
    if (s.has_table) {
      if ((e = B.table.ensure(s.table.rows.size())) != cudaSuccess) break;
      if ((e = cudaMemcpyAsync(B.table.ptr, s.table.rows.data(), s.table.rows.size() * sizeof(double),
                               cudaMemcpyHostToDevice, stream)) != cudaSuccess)
        break;
      A.table = B.table.ptr;
    }
    if ((e = launch_step_error(A, s.arith, last_steps, B.batch_acc.ptr, stream)) != cudaSuccess) break;
    t_launches += 1;
    unsigned long long key = ~0ull;
    unsigned int range = 0;
    e = cudaMemcpyAsync(&key, B.err_key.ptr, sizeof key, cudaMemcpyDeviceToHost, stream);
    if (e == cudaSuccess) e = cudaMemcpyAsync(&range, B.range_flag.ptr, sizeof range, cudaMemcpyDeviceToHost, stream);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(sums.data(), B.batch_acc.ptr, 4 * blocks * sizeof(double),
                          cudaMemcpyDeviceToHost, stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
    if (e != cudaSuccess) break;
    if (range != 0 && (s.arith == BarArith::kF32 || s.arith == BarArith::kF32Round)) {
      s.arith = BarArith::kF64Round;  // exact emulation outside the native range
      continue;
    }
    if (key != ~0ull) {
      const int bits = s.args.err_step_bits;
      const uint64_t path = key >> (bits + 2);
      const int kind = static_cast<int>((key >> bits) & 3u);
      const uint64_t step = key & ((1ull << bits) - 1);
      if (kind == LPMC_FAIL_UNIFORM_IS_ONE)
        return fail(err, LPMC_DOMAIN_ERROR,
                    table != nullptr ? "approx_inv_cdf requires u in (0, 1)"
                                     : "exact_inv_cdf requires u in (0, 1)",
                    kind, path, step);
      return fail(err, LPMC_DOMAIN_ERROR, "non-finite operand", LPMC_FAIL_NONFINITE, path, step);
    }
    double tot[4] = {0.0, 0.0, 0.0, 0.0};
    for (uint64_t b = 0; b < blocks; ++b)
      for (int q = 0; q < 4; ++q) tot[q] += sums[4 * b + q];
    const double count = static_cast<double>(n_samples);
    *out = lpmc_step_error_stats{tot[0] / count, tot[1] / count, tot[2] / count, tot[3] / count,
                                 n_samples};
    return ok(err);
  }
  if (e != cudaSuccess) return cuda_fail(err, e, "step-error probe");
  return fail(err, LPMC_RUNTIME_ERROR, "native range fallback did not converge");
}

lpmc_status lpmc_simulate_paths(const lpmc_gbm* model, int32_t level, const lpmc_precision* prec,
                                const lpmc_invcdf_table* table, int32_t kahan, uint64_t n_paths,
                                uint64_t seed, uint64_t path_base, const lpmc_options* opts,
                                double* out4, double* z_out, lpmc_error* err) {
  if (out4 == nullptr) return fail(err, LPMC_INVALID_ARGUMENT, "null argument");
  if (n_paths == 0) return ok(err);
  if (n_paths > (1ull << 26)) return fail(err, LPMC_INVALID_ARGUMENT, "path dump limited to 2^26 paths");
  RunSpec s;
  lpmc_status st = build_spec(model, level, prec, table, kahan, n_paths, seed, path_base, opts, &s, err);
  if (st != LPMC_OK) return st;
  DeviceCtx* ctx = nullptr;
  int dev = -1;
  st = get_ctx(s.device, &ctx, &dev, err);
  if (st != LPMC_OK) return st;
  DeviceGuard guard;
  cudaError_t e = guard.set(dev);
  if (e != cudaSuccess) return cuda_fail(err, e, "cudaSetDevice");
  std::lock_guard<std::mutex> lock(ctx->mu);
  cudaStream_t stream = (opts && opts->stream) ? static_cast<cudaStream_t>(opts->stream) : ctx->stream;
  if (z_out != nullptr && (level > 32 || (n_paths << level) > (1ull << 32)))
    return fail(err, LPMC_INVALID_ARGUMENT, "Gaussian dump limited to 2^32 draws");
  const uint64_t zcount = z_out ? n_paths << level : 0;
  DevBuf<double> d_out, d_z;
  Buffers& B = ctx->scratch;
  for (int attempt = 0; attempt < 2; ++attempt) {
    if ((e = d_out.ensure(4 * n_paths)) != cudaSuccess) break;
    if (zcount && (e = d_z.ensure(zcount)) != cudaSuccess) break;
    if ((e = B.err_key.ensure(1)) != cudaSuccess) break;
    if ((e = B.range_flag.ensure(1)) != cudaSuccess) break;
    if ((e = cudaMemsetAsync(B.err_key.ptr, 0xff, sizeof(unsigned long long), stream)) != cudaSuccess)
      break;
    if ((e = cudaMemsetAsync(B.range_flag.ptr, 0, sizeof(unsigned int), stream)) != cudaSuccess) break;
    LevelArgs A = s.args;
    A.err_key = B.err_key.ptr;
    A.range_flag = B.range_flag.ptr;
    A.table = nullptr;
    if (s.has_table) {
      if ((e = B.table.ensure(s.table.rows.size())) != cudaSuccess) break;
      if ((e = cudaMemcpyAsync(B.table.ptr, s.table.rows.data(),
                               s.table.rows.size() * sizeof(double), cudaMemcpyHostToDevice,
                               stream)) != cudaSuccess)
        break;
      A.table = B.table.ptr;
    }
    A.batch0 = 0;
    A.n_batches = (n_paths + kBatch - 1) / kBatch;
    A.batch_acc = nullptr;
    A.path_diff = nullptr;
    A.path_out = d_out.ptr;
    A.z_out = zcount ? d_z.ptr : nullptr;
    // the dump of Gaussians is the fused kernel's; an explicit warp-per-path
    // request dumps that schedule's terminal values (parity of the schedule)
    const bool wpp = zcount == 0 && s.schedule == LPMC_SCHEDULE_WARP_PER_PATH && use_wpp(s);
    LaunchResult r = wpp ? launch_paths_wpp(A, s.arith, s.kahan, stream)
                         : launch_paths(A, s.arith, s.kahan, true, stream);
    t_launches += r.kernels;
    if (r.cuda_error != 0) {
      e = static_cast<cudaError_t>(r.cuda_error);
      break;
    }
    unsigned long long key = ~0ull;
    unsigned int range = 0;
    e = cudaMemcpyAsync(&key, B.err_key.ptr, sizeof key, cudaMemcpyDeviceToHost, stream);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(&range, B.range_flag.ptr, sizeof range, cudaMemcpyDeviceToHost, stream);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(out4, d_out.ptr, 4 * n_paths * sizeof(double), cudaMemcpyDeviceToHost,
                          stream);
    if (e == cudaSuccess && zcount)
      e = cudaMemcpyAsync(z_out, d_z.ptr, zcount * sizeof(double), cudaMemcpyDeviceToHost, stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
    if (e != cudaSuccess) break;
    if (range != 0 && (s.arith == BarArith::kF32 || s.arith == BarArith::kF32Round)) {
      s.arith = BarArith::kF64Round;
      continue;
    }
    d_out.release();
    d_z.release();
    if (key != ~0ull) return failure_from_key(s, key, err);
    return ok(err);
  }
  d_out.release();
  d_z.release();
  return cuda_fail(err, e, "path dump");
}

lpmc_status lpmc_device_math(int32_t op, const double* u, uint64_t n,
                             const lpmc_invcdf_table* table, double* out,
                             const lpmc_options* opts, lpmc_error* err) {
  if (n == 0) return ok(err);
  if (u == nullptr || out == nullptr) return fail(err, LPMC_INVALID_ARGUMENT, "null argument");
  if (op < 0 || op > 5 || op == 4) return fail(err, LPMC_INVALID_ARGUMENT, "bad math op");
  if (op == 1 && table == nullptr) return fail(err, LPMC_INVALID_ARGUMENT, "op 1 needs a table");
  HostTable ht;
  if (table != nullptr) {
    lpmc_status st = prepare_table(table, &ht, err);
    if (st != LPMC_OK) return st;
  }
  DeviceCtx* ctx = nullptr;
  int dev = -1;
  lpmc_status st = get_ctx(opts ? opts->device : -1, &ctx, &dev, err);
  if (st != LPMC_OK) return st;
  DeviceGuard guard;
  cudaError_t e = guard.set(dev);
  if (e != cudaSuccess) return cuda_fail(err, e, "cudaSetDevice");
  std::lock_guard<std::mutex> lock(ctx->mu);
  cudaStream_t stream = ctx->stream;
  DevBuf<double>& du = ctx->scratch.io_in;
  DevBuf<double>& dout = ctx->scratch.io_out;
  DevBuf<double>& dtab = ctx->scratch.table;
  if ((e = du.ensure(n)) == cudaSuccess && (e = dout.ensure(n)) == cudaSuccess &&
      (table == nullptr || (e = dtab.ensure(ht.rows.size())) == cudaSuccess)) {
    e = cudaMemcpyAsync(du.ptr, u, n * sizeof(double), cudaMemcpyHostToDevice, stream);
    if (e == cudaSuccess && table != nullptr)
      e = cudaMemcpyAsync(dtab.ptr, ht.rows.data(), ht.rows.size() * sizeof(double),
                          cudaMemcpyHostToDevice, stream);
    if (e != cudaSuccess) return cuda_fail(err, e, "inverse-CDF upload");
    LaunchResult r = launch_inv_cdf(du.ptr, n, table ? dtab.ptr : nullptr, ht.K, ht.degree,
                                    ht.dyadic, ht.stride, ht.simple, ht.tail, op, dout.ptr, stream);
    t_launches += r.kernels;
    e = static_cast<cudaError_t>(r.cuda_error);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(out, dout.ptr, n * sizeof(double), cudaMemcpyDeviceToHost, stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
  }
  if (e != cudaSuccess) return cuda_fail(err, e, "inv_cdf");
  return ok(err);
}

lpmc_status lpmc_density_histogram(const lpmc_invcdf_table* table, uint64_t seed,
                                   uint64_t n_samples, double z_max, double bin_width,
                                   int32_t n_bins, uint64_t* bins, const lpmc_options* opts,
                                   lpmc_error* err) {
  // the histogram loop of run_density_report (experiments.hpp:276-285)
  if (n_bins < 1 || bins == nullptr) return fail(err, LPMC_INVALID_ARGUMENT, "need at least one bin");
  if (!(bin_width > 0.0) || !std::isfinite(z_max))
    return fail(err, LPMC_INVALID_ARGUMENT, "bad histogram geometry");
  for (int32_t b = 0; b < n_bins; ++b) bins[b] = 0;
  if (n_samples == 0) return ok(err);
  HostTable ht;
  if (table != nullptr) {
    lpmc_status st = prepare_table(table, &ht, err);
    if (st != LPMC_OK) return st;
  }
  // UniformStream(seed, 0) (uniform.hpp:23-25): the key of path 0
  const uint64_t key = host_mix64(seed_key_of(seed) ^ host_mix64(0 + 0xbf58476d1ce4e5b9ull));
  DeviceCtx* ctx = nullptr;
  int dev = -1;
  lpmc_status st = get_ctx(opts ? opts->device : -1, &ctx, &dev, err);
  if (st != LPMC_OK) return st;
  DeviceGuard guard;
  cudaError_t e = guard.set(dev);
  if (e != cudaSuccess) return cuda_fail(err, e, "cudaSetDevice");
  std::lock_guard<std::mutex> lock(ctx->mu);
  cudaStream_t stream = ctx->stream;
  DevBuf<double>& dtab = ctx->scratch.table;
  DevBuf<unsigned long long>& dbins = ctx->scratch.counts;
  DevBuf<unsigned long long>& dtop = ctx->scratch.err_key;
  unsigned long long top = ~0ull;
  if ((e = dbins.ensure(static_cast<size_t>(n_bins))) == cudaSuccess &&
      (e = dtop.ensure(1)) == cudaSuccess &&
      (table == nullptr || (e = dtab.ensure(ht.rows.size())) == cudaSuccess)) {
    e = cudaMemsetAsync(dbins.ptr, 0, static_cast<size_t>(n_bins) * sizeof(unsigned long long),
                        stream);
    if (e == cudaSuccess) e = cudaMemsetAsync(dtop.ptr, 0xff, sizeof(unsigned long long), stream);
    if (e == cudaSuccess && table != nullptr)
      e = cudaMemcpyAsync(dtab.ptr, ht.rows.data(), ht.rows.size() * sizeof(double),
                          cudaMemcpyHostToDevice, stream);
    if (e != cudaSuccess) return cuda_fail(err, e, "density upload");
    LaunchResult r = launch_density(key, n_samples, table ? dtab.ptr : nullptr,
                                    static_cast<int>(ht.rows.size()), ht.K, ht.degree, ht.dyadic,
                                    ht.stride, ht.simple, ht.tail, z_max, bin_width, n_bins,
                                    opts != nullptr ? opts->exact_z : LPMC_EXACT_Z_FAST,
                                    dbins.ptr, dtop.ptr, stream);
    t_launches += r.kernels;
    e = static_cast<cudaError_t>(r.cuda_error);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(bins, dbins.ptr, static_cast<size_t>(n_bins) * sizeof(uint64_t),
                          cudaMemcpyDeviceToHost, stream);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(&top, dtop.ptr, sizeof top, cudaMemcpyDeviceToHost, stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
  }
  if (e != cudaSuccess) return cuda_fail(err, e, "density histogram");
  if (top != ~0ull)  // the reference throws at that draw
    return fail(err, LPMC_DOMAIN_ERROR,
                table != nullptr ? "approx_inv_cdf requires u in (0, 1)"
                                 : "exact_inv_cdf requires u in (0, 1)",
                LPMC_FAIL_UNIFORM_IS_ONE, 0, top);
  return ok(err);
}

lpmc_status lpmc_device_inv_cdf(const double* u, uint64_t n, const lpmc_invcdf_table* table,
                                double* out, const lpmc_options* opts, lpmc_error* err) {
  const bool glibc = opts != nullptr && opts->exact_z == LPMC_EXACT_Z_GLIBC;
  return lpmc_device_math(table ? 1 : (glibc ? 5 : 0), u, n, table, out, opts, err);
}

double lpmc_erfc_core(double t) {
  if (!(t >= 0.0 && t < math::kFastTMax)) return std::erfc(t);
  return math::erfc_fast(t, math::kMathTableHost);
}

lpmc_status lpmc_bar_arithmetic(const lpmc_gbm* model, int32_t level, const lpmc_precision* prec,
                                const lpmc_invcdf_table* table, int32_t kahan,
                                const lpmc_options* opts, int32_t* out, lpmc_error* err) {
  if (out == nullptr) return fail(err, LPMC_INVALID_ARGUMENT, "null argument");
  RunSpec s;
  const lpmc_status st = build_spec(model, level, prec, table, kahan, 256, 1, 0, opts, &s, err);
  if (st != LPMC_OK) return st;
  LevelArgs A = s.args;
  // the dispatcher's view: a table pointer is set at launch
  static const double kSome = 0.0;
  A.table = s.has_table ? &kSome : nullptr;
  *out = static_cast<int32_t>(s.arith) | (A.bar_pow2 ? LPMC_ARITH_POW2_FOLDED : 0) |
         (s.arith == BarArith::kF32Round && use_native_half(A, kahan != 0, false)
              ? LPMC_ARITH_NATIVE_BINARY16 : 0) |
         (s.arith == BarArith::kF32Round && use_native_bf16(A, false) ? LPMC_ARITH_NATIVE_BFLOAT16
                                                                      : 0);
  return ok(err);
}

double lpmc_phi_inv_direct_core(double v, int32_t* in_table) {
  bool tail = true;
  double z = std::nan("");
  if (v > 0.0 && v <= 0.5) z = math::phi_inv_direct(v, math::DirectTab{math::kDirectHost}, &tail);
  if (in_table != nullptr) *in_table = tail ? 0 : 1;
  // the table holds the upper half, -Phi^-1(v); +0 at v == 1/2 (gaussian.hpp:62)
  return tail ? std::nan("") : (z == 0.0 ? 0.0 : -z);
}

static_assert(LPMC_EXACT_Z_FAST == 0 && LPMC_EXACT_Z_GLIBC == 1, "dev::kZFast / kZGlibc");

double lpmc_glibc_math(int32_t op, double x, int32_t* ok) {
  bool good = true;
  double r = std::nan("");
  const double* t = math::kMathTableHost;
  switch (op) {
    case 0: r = glibc::exp(x, t, &good); break;
    case 1: r = glibc::log(x, t, &good); break;
    case 2: r = glibc::erfc(x, t, &good); break;
    case 3: r = glibc::inv_cdf(x, t, &good); break;
    default: good = false;
  }
  if (ok != nullptr) *ok = good ? 1 : 0;
  return r;
}

lpmc_status lpmc_measure_pipe_peaks(int32_t device, double* out4, lpmc_error* err) {
  if (out4 == nullptr) return fail(err, LPMC_INVALID_ARGUMENT, "null argument");
  DeviceCtx* ctx = nullptr;
  int dev = -1;
  lpmc_status st = get_ctx(device, &ctx, &dev, err);
  if (st != LPMC_OK) return st;
  DeviceGuard guard;
  cudaError_t e = guard.set(dev);
  if (e != cudaSuccess) return cuda_fail(err, e, "cudaSetDevice");
  std::lock_guard<std::mutex> lock(ctx->mu);
  e = static_cast<cudaError_t>(measure_pipe_peaks(out4));
  if (e != cudaSuccess) return cuda_fail(err, e, "pipe peaks");
  return ok(err);
}

// ------------------------------------------------------------- plans -------
struct lpmc_plan {
  RunSpec spec;
  Buffers buffers;
  Enqueued last;
  int device = -1;
  cudaStream_t own_stream = nullptr;
  cudaStream_t last_stream = nullptr;
  bool launched = false;
};

lpmc_status lpmc_plan_create(const lpmc_gbm* model, int32_t level, const lpmc_precision* prec,
                             const lpmc_invcdf_table* table, int32_t kahan, uint64_t n_paths,
                             uint64_t seed, uint64_t path_base, const lpmc_options* opts,
                             lpmc_plan** plan, lpmc_error* err) {
  const uint64_t n_chunks = (n_paths + LPMC_CHUNK_PATHS - 1) / LPMC_CHUNK_PATHS;
  return lpmc_plan_create_range(model, level, prec, table, kahan, n_paths, seed, path_base, 0,
                                n_chunks, opts, plan, err);
}

lpmc_status lpmc_plan_create_range(const lpmc_gbm* model, int32_t level,
                                   const lpmc_precision* prec, const lpmc_invcdf_table* table,
                                   int32_t kahan, uint64_t n_paths, uint64_t seed,
                                   uint64_t path_base, uint64_t chunk_begin, uint64_t chunk_end,
                                   const lpmc_options* opts, lpmc_plan** plan, lpmc_error* err) {
  if (plan == nullptr) return fail(err, LPMC_INVALID_ARGUMENT, "null argument");
  *plan = nullptr;
  if (n_paths == 0) return fail(err, LPMC_INVALID_ARGUMENT, "plan needs n_paths > 0");
  const uint64_t n_chunks = (n_paths + LPMC_CHUNK_PATHS - 1) / LPMC_CHUNK_PATHS;
  if (chunk_end > n_chunks || chunk_begin >= chunk_end)
    return fail(err, LPMC_INVALID_ARGUMENT, "chunk range outside the run");
  auto p = std::make_unique<lpmc_plan>();
  lpmc_status st = build_spec(model, level, prec, table, kahan, n_paths, seed, path_base, opts,
                              &p->spec, err);
  if (st != LPMC_OK) return st;
  if (chunk_begin != 0 || chunk_end != n_chunks) p->spec.reduce = LPMC_REDUCE_TREE;
  p->spec.chunk_begin = chunk_begin;
  p->spec.chunk_end = chunk_end;
  DeviceCtx* ctx = nullptr;
  st = get_ctx(p->spec.device, &ctx, &p->device, err);
  if (st != LPMC_OK) return st;
  DeviceGuard guard;
  cudaError_t e = guard.set(p->device);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&p->own_stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) return cuda_fail(err, e, "plan stream");
  // Pre-allocate by a dry enqueue on the plan's stream, then wait.
  Enqueued q;
  e = enqueue_run(p->spec, p->buffers, p->own_stream, &q);
  if (e == cudaSuccess) e = cudaStreamSynchronize(p->own_stream);
  if (e != cudaSuccess) return cuda_fail(err, e, "plan warm-up");
  t_launches -= static_cast<uint64_t>(q.kernels);
  *plan = p.release();
  return ok(err);
}

lpmc_status lpmc_plan_launch(lpmc_plan* p, void* stream, lpmc_error* err) {
  if (p == nullptr) return fail(err, LPMC_INVALID_ARGUMENT, "null argument");
  DeviceGuard guard;
  cudaError_t e = guard.set(p->device);
  if (e != cudaSuccess) return cuda_fail(err, e, "cudaSetDevice");
  cudaStream_t st = stream != nullptr ? static_cast<cudaStream_t>(stream) : p->own_stream;
  e = enqueue_run(p->spec, p->buffers, st, &p->last);
  if (e != cudaSuccess) return cuda_fail(err, e, "plan launch");
  p->last_stream = st;
  p->launched = true;
  return ok(err);
}

lpmc_status lpmc_plan_collect(lpmc_plan* p, lpmc_moments* out, lpmc_error* err) {
  if (p == nullptr || out == nullptr) return fail(err, LPMC_INVALID_ARGUMENT, "null argument");
  if (!p->launched) return fail(err, LPMC_INVALID_ARGUMENT, "plan was not launched");
  DeviceGuard guard;
  cudaError_t e = guard.set(p->device);
  if (e != cudaSuccess) return cuda_fail(err, e, "cudaSetDevice");
  std::vector<Moments> parts;
  bool rerun = false;
  lpmc_status st = collect_run(p->spec, p->buffers, p->last_stream, p->last, &parts, &rerun, err);
  if (st != LPMC_OK) return st;
  if (rerun) {
    RunSpec s = p->spec;
    s.arith = BarArith::kF64Round;
    Enqueued q;
    e = enqueue_run(s, p->buffers, p->last_stream, &q);
    if (e != cudaSuccess) return cuda_fail(err, e, "fallback launch");
    st = collect_run(s, p->buffers, p->last_stream, q, &parts, &rerun, err);
    if (st != LPMC_OK) return st;
  }
  mask_legs(p->spec, parts);
  fold(parts, out);
  p->launched = false;
  return ok(err);
}

lpmc_status lpmc_plan_collect_partials(lpmc_plan* p, lpmc_moments* out, lpmc_error* err) {
  if (p == nullptr || out == nullptr) return fail(err, LPMC_INVALID_ARGUMENT, "null argument");
  if (!p->launched) return fail(err, LPMC_INVALID_ARGUMENT, "plan was not launched");
  if (p->spec.reduce != LPMC_REDUCE_TREE)
    return fail(err, LPMC_INVALID_ARGUMENT, "partials need the tree reduction");
  DeviceGuard guard;
  cudaError_t e = guard.set(p->device);
  if (e != cudaSuccess) return cuda_fail(err, e, "cudaSetDevice");
  std::vector<Moments> parts;
  bool rerun = false;
  lpmc_status st = collect_run(p->spec, p->buffers, p->last_stream, p->last, &parts, &rerun, err);
  if (st != LPMC_OK) return st;
  if (rerun) {
    RunSpec s = p->spec;
    s.arith = BarArith::kF64Round;
    Enqueued q;
    e = enqueue_run(s, p->buffers, p->last_stream, &q);
    if (e != cudaSuccess) return cuda_fail(err, e, "fallback launch");
    st = collect_run(s, p->buffers, p->last_stream, q, &parts, &rerun, err);
    if (st != LPMC_OK) return st;
  }
  mask_legs(p->spec, parts);
  for (size_t i = 0; i < parts.size(); ++i) out[i] = to_abi(parts[i]);
  p->launched = false;
  return ok(err);
}

uint64_t lpmc_plan_chunk_count(const lpmc_plan* p) { return p->spec.chunk_end - p->spec.chunk_begin; }

int32_t lpmc_plan_kernels_per_launch(const lpmc_plan* p) {
  const uint64_t chunks = p->spec.chunk_end - p->spec.chunk_begin;
  const uint64_t slice = p->spec.reduce == LPMC_REDUCE_SEQUENTIAL ? kSeqSliceChunks : kSliceChunks;
  return static_cast<int32_t>(2 * ((chunks + slice - 1) / slice));
}

void lpmc_plan_destroy(lpmc_plan* p) {
  if (p == nullptr) return;
  DeviceGuard guard;
  guard.set(p->device);
  if (p->own_stream != nullptr) {
    cudaStreamSynchronize(p->own_stream);
    cudaStreamDestroy(p->own_stream);
  }
  p->buffers.release();
  delete p;
}

}  // extern "C"
