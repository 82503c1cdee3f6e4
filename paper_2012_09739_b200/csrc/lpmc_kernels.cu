// sm_100a kernels of the MLMC level-correction sampler.
//
// One thread owns one path (two for the IEEE-half2 legs) for the whole level:
// the counter RNG key, four EM states, two Kahan compensations and the two
// pending coarse increments live in registers; nothing per step touches
// memory.  A 256-path batch is one CTA (the reference's kBatch, mlmc.hpp:74);
// the CTA reduces its 256 differences to central moments with a fixed
// two-pass warp-shuffle tree, and a second kernel merges 1024 batch
// accumulators per chunk with Pebay's update in a fixed binary tree.  The host
// then folds chunks in index order (mlmc.hpp:108-110), so the result is
// independent of how chunks are spread over GPUs.
//
// Compiled with -fmad=false: the reference rounds every operation separately
// (sde.hpp:60-116 on a binary64 carrier without FMA), so no
// multiply-add may be contracted anywhere on this path.
//
// Reference cross-walk (file:line under /root/reference/proj/include/lpmc):
//   mix64 / stream_word / next      uniform.hpp:13-41
//   exact_inv_cdf (Acklam+Newton)   gaussian.hpp:14-65
//   InvCdfApprox::operator()        invcdf_approx.hpp:44-90
//   round_to_precision / fp_*       softfloat.hpp:69-111
//   em_step* / kahan_accumulate     sde.hpp:60-116
//   simulate_coupled                sde.hpp:211-284
//   MomentAccumulator add/merge     stats.hpp:15-54

#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "lpmc_internal.h"
#include "lpmc_math.cuh"

namespace lpmc_b200 {
namespace {

constexpr int kBatch = 256;
constexpr int kChunkBatches = 1024;
constexpr int kChunkThreads = 512;
constexpr uint64_t kTopDraw = 0x1FFFFFFFFFFFFFull;  // (w >> 11) that rounds u to 1.0
constexpr uint64_t kNoFail = ~0ull;

enum : uint32_t { kStageDraw = 0, kStageHatFine = 1, kStageBarFine = 2, kStageHatCoarse = 3,
                  kStageBarCoarse = 4 };
enum : uint32_t { kKindU1 = 1, kKindNonFinite = 2, kKindState = 3 };

// ---------------------------------------------------------------- RNG ------
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z ^= z >> 33;
  z *= 0xff51afd7ed558ccdull;
  z ^= z >> 33;
  z *= 0xc4ceb9fe1a85ec53ull;
  z ^= z >> 33;
  return z;
}

// ------------------------------------------------ exact inverse CDF --------
// math::phi_inv (lpmc_math.cuh): Acklam + one Newton step with a
// constant-bank erfc; the erfcx coefficient table is staged in shared memory.
using math::phi_inv;
constexpr int kErfcxWords = math::kErfcxRows * math::kErfcxN;

__device__ __forceinline__ void stage_erfcx(double* s_erfcx) {
  for (int i = threadIdx.x; i < kErfcxWords; i += blockDim.x) s_erfcx[i] = math::kErfcxTable[i];
}

// ------------------------------------------- approximate inverse CDF -------
struct TableView {
  const double* a;    // left endpoints
  const double* w;    // 2^(j+2) (dyadic) or b_j - a_j
  const double* c0;
  const double* c1;
  const double* c2;
  const double* c3;
  const double* thr;  // v-thresholds (general K)
  int K, degree, dyadic;
  double tail;
};

__device__ __forceinline__ TableView table_view(const double* base, int K, int degree, int dyadic,
                                                double tail) {
  TableView t;
  t.a = base;
  t.w = base + K;
  t.c0 = base + 2 * K;
  t.c1 = base + 3 * K;
  t.c2 = base + 4 * K;
  t.c3 = base + 5 * K;
  t.thr = base + 6 * K;
  t.K = K;
  t.degree = degree;
  t.dyadic = dyadic;
  t.tail = tail;
  return t;
}

// InvCdfApprox::operator() (invcdf_approx.hpp:44-90).  The interval index is
// read from the exponent of v = 1 - u' for dyadic tables (exactly the
// reference's floor(-log2 v) on the 2^-53 grid), or found in a
// host-computed threshold table that reproduces the reference's log2-based
// index on every representable v (general K).
__device__ __forceinline__ double approx_inv(const TableView& t, double u) {
  const bool lower = u < 0.5;
  const double up = lower ? 1.0 - u : u;  // fl(1-u) for the lower half (:47-49)
  const double v = 1.0 - up;              // exact (Sterbenz)
  int j;
  bool tail;
  if (t.dyadic) {
    const uint64_t vb = static_cast<uint64_t>(__double_as_longlong(v));
    const int e = static_cast<int>(vb >> 52) - 1023;
    const int fl = (vb & 0xFFFFFFFFFFFFFull) == 0 ? -e : -e - 1;  // floor(-log2 v)
    tail = fl >= t.K + 1;
    j = min(max(fl - 1, 0), t.K - 1);
  } else {
    int lo = 0, hi = t.K - 1;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (v <= t.thr[mid]) lo = mid + 1; else hi = mid;
    }
    j = lo;
    tail = v <= t.thr[t.K - 1];
  }
  double r;
  if (tail) {
    r = t.tail;
  } else {
    const double a = t.a[j];
    const double span2 = 2.0 * (up - a);
    double s = t.dyadic ? span2 * t.w[j] : span2 / t.w[j];
    s = s - 1.0;
    s = s < -1.0 ? -1.0 : s;
    s = s > 1.0 ? 1.0 : s;
    r = t.c0[j] + t.c1[j] * s;
    if (t.degree == 3 || r == 0.0) {  // r == 0: keep the reference's signed-zero result
      const double p2 = 1.5 * s * s - 0.5;
      const double p3 = s * (2.5 * s * s - 1.5);
      r = r + t.c2[j] * p2 + t.c3[j] * p3;
    }
  }
  r = lower ? -r : r;
  return u == 0.5 ? 0.0 : r;
}

// ----------------------------------------------- rounding helpers ---------
// Round-to-nearest-even of a binary64 value to m+1 significant bits by
// integer arithmetic on its bit pattern (== round_to_precision, softfloat.hpp:
// 69-80, for normal operands; binary64 subnormals are scaled like frexp/ldexp).
__device__ __forceinline__ double rne64(double x, uint32_t d, uint64_t half_m1, uint64_t keep) {
  uint64_t b = static_cast<uint64_t>(__double_as_longlong(x));
  if (((b >> 52) & 0x7ff) == 0 && (b << 1) != 0) {
    const double y = x * 0x1p64;
    uint64_t c = static_cast<uint64_t>(__double_as_longlong(y));
    c = (c + half_m1 + ((c >> d) & 1ull)) & keep;
    return __longlong_as_double(static_cast<long long>(c)) * 0x1p-64;
  }
  b = (b + half_m1 + ((b >> d) & 1ull)) & keep;
  return __longlong_as_double(static_cast<long long>(b));
}

__device__ __forceinline__ float rne32(float x, uint32_t d, uint32_t half_m1, uint32_t keep) {
  uint32_t b = __float_as_uint(x);
  b = (b + half_m1 + ((b >> d) & 1u)) & keep;
  return __uint_as_float(b);
}

__device__ __forceinline__ bool nonfinite64(double x) {
  return (__double2hiint(x) & 0x7ff00000) == 0x7ff00000;
}
__device__ __forceinline__ bool nonfinite32(float x) {
  return (__float_as_uint(x) & 0x7f800000u) == 0x7f800000u;
}
// Native fp32 legs are bit-exact with the unbounded-exponent reference while
// no intermediate is subnormal or overflows; the host pre-checks the
// constants and the kernel keeps states in [2^-32, 2^33) (SURVEY.md §7 "hard
// parts").  Outside it the host re-runs the
// level with the exact kF64Round emulation.
__device__ __forceinline__ bool out_of_native_range(float x) {
  const uint32_t b = __float_as_uint(x) & 0x7fffffffu;
  const uint32_t e = b >> 23;
  return b != 0 && (e - (127u - 32u)) > 64u;
}

// ------------------------------------------------------ bar arithmetic -----
// Each policy: T (state type), NP (paths per thread), mul/add/sub in the
// target precision, lift(z[NP]) = R(z) packed, get(x, p) -> double, bad(x)
// -> bitmask of non-finite lanes, range(x) -> native-range violation.

struct ArithCarrier {  // m >= 52
  using T = double;
  static constexpr int NP = 1;
  static constexpr bool kIeee = false;
  __device__ explicit ArithCarrier(const LevelArgs&) {}
  __device__ T c(double d, uint16_t) const { return d; }
  __device__ T zero() const { return 0.0; }
  __device__ T mul(T a, T b) const { return __dmul_rn(a, b); }
  __device__ T add(T a, T b) const { return __dadd_rn(a, b); }
  __device__ T sub(T a, T b) const { return __dsub_rn(a, b); }
  __device__ T lift(const double (&z)[1]) const { return z[0]; }
  __device__ double get(T x, int) const { return x; }
  __device__ uint32_t bad(T x) const { return nonfinite64(x) ? 1u : 0u; }
  __device__ bool range(T) const { return false; }
};

struct ArithF32 {  // m == 23, native
  using T = float;
  static constexpr int NP = 1;
  static constexpr bool kIeee = false;
  __device__ explicit ArithF32(const LevelArgs&) {}
  __device__ T c(double d, uint16_t) const { return static_cast<float>(d); }  // exact
  __device__ T zero() const { return 0.0f; }
  __device__ T mul(T a, T b) const { return __fmul_rn(a, b); }
  __device__ T add(T a, T b) const { return __fadd_rn(a, b); }
  __device__ T sub(T a, T b) const { return __fsub_rn(a, b); }
  __device__ T lift(const double (&z)[1]) const { return __double2float_rn(z[0]); }
  __device__ double get(T x, int) const { return static_cast<double>(x); }
  __device__ uint32_t bad(T x) const { return nonfinite32(x) ? 1u : 0u; }
  __device__ bool range(T x) const { return out_of_native_range(x); }
};

struct ArithF32Round {  // m <= 10: fp32 op, then RNE to m+1 bits
  using T = float;
  static constexpr int NP = 1;
  static constexpr bool kIeee = false;
  uint32_t d, half_m1, keep;
  uint32_t d64;
  uint64_t half_m1_64, keep64;
  __device__ explicit ArithF32Round(const LevelArgs& A) {
    d = 23u - static_cast<uint32_t>(A.mantissa_bits);
    half_m1 = (1u << (d - 1)) - 1u;
    keep = ~((1u << d) - 1u);
    d64 = 52u - static_cast<uint32_t>(A.mantissa_bits);
    half_m1_64 = (1ull << (d64 - 1)) - 1ull;
    keep64 = ~((1ull << d64) - 1ull);
  }
  __device__ T c(double dd, uint16_t) const { return static_cast<float>(dd); }
  __device__ T zero() const { return 0.0f; }
  __device__ T mul(T a, T b) const { return rne32(__fmul_rn(a, b), d, half_m1, keep); }
  __device__ T add(T a, T b) const { return rne32(__fadd_rn(a, b), d, half_m1, keep); }
  __device__ T sub(T a, T b) const { return rne32(__fsub_rn(a, b), d, half_m1, keep); }
  // R(z) from the full binary64 value (a single rounding, softfloat.hpp:69)
  __device__ T lift(const double (&z)[1]) const {
    return __double2float_rn(rne64(z[0], d64, half_m1_64, keep64));
  }
  __device__ double get(T x, int) const { return static_cast<double>(x); }
  __device__ uint32_t bad(T x) const { return nonfinite32(x) ? 1u : 0u; }
  __device__ bool range(T x) const { return out_of_native_range(x); }
};

struct ArithF64Round {  // any m < 52: binary64 op, then integer RNE (exact emulation)
  using T = double;
  static constexpr int NP = 1;
  static constexpr bool kIeee = false;
  uint32_t d;
  uint64_t half_m1, keep;
  __device__ explicit ArithF64Round(const LevelArgs& A) {
    d = 52u - static_cast<uint32_t>(A.mantissa_bits);
    half_m1 = (1ull << (d - 1)) - 1ull;
    keep = ~((1ull << d) - 1ull);
  }
  __device__ T c(double dd, uint16_t) const { return dd; }
  __device__ T zero() const { return 0.0; }
  __device__ T mul(T a, T b) const { return rne64(__dmul_rn(a, b), d, half_m1, keep); }
  __device__ T add(T a, T b) const { return rne64(__dadd_rn(a, b), d, half_m1, keep); }
  __device__ T sub(T a, T b) const { return rne64(__dsub_rn(a, b), d, half_m1, keep); }
  __device__ T lift(const double (&z)[1]) const { return rne64(z[0], d, half_m1, keep); }
  __device__ double get(T x, int) const { return x; }
  __device__ uint32_t bad(T x) const { return nonfinite64(x) ? 1u : 0u; }
  __device__ bool range(T) const { return false; }
};

struct ArithHalf2 {  // native IEEE binary16, two paths per thread
  using T = __half2;
  static constexpr int NP = 2;
  static constexpr bool kIeee = true;
  __device__ explicit ArithHalf2(const LevelArgs&) {}
  __device__ T c(double, uint16_t bits) const {
    const __half h = __ushort_as_half(bits);
    return __halves2half2(h, h);
  }
  __device__ T zero() const { return __float2half2_rn(0.0f); }
  __device__ T mul(T a, T b) const { return __hmul2_rn(a, b); }
  __device__ T add(T a, T b) const { return __hadd2_rn(a, b); }
  __device__ T sub(T a, T b) const { return __hsub2_rn(a, b); }
  __device__ T lift(const double (&z)[2]) const {
    return __halves2half2(__double2half(z[0]), __double2half(z[1]));
  }
  __device__ double get(T x, int p) const {
    return static_cast<double>(__half2float(p == 0 ? __low2half(x) : __high2half(x)));
  }
  __device__ uint32_t bad(T x) const {
    const uint32_t b = *reinterpret_cast<const uint32_t*>(&x);
    return (((b & 0x7c00u) == 0x7c00u) ? 1u : 0u) | (((b & 0x7c000000u) == 0x7c000000u) ? 2u : 0u);
  }
  __device__ bool range(T) const { return false; }
};

// --------------------------------------------------------- block tree ------
// Fixed reduction of a 256-path batch: slot s = threadIdx.x + p*blockDim.x;
// per 32-slot group an xor butterfly, then an xor butterfly over the 8 group
// sums.  Pass 1 gives the mean, pass 2 the central power sums.  Restated
// bit-for-bit in oracle/lpmc_oracle.c (batch_acc).
__device__ __forceinline__ double warp_sum(double x, int first) {
  for (int k = first; k >= 1; k >>= 1) x = __dadd_rn(x, __shfl_xor_sync(0xffffffffu, x, k));
  return x;
}

template <int NP>
__device__ void batch_moments(const double (&vh)[NP], const double (&vb)[NP],
                              const bool (&valid)[NP], int count, double* out15) {
  __shared__ double s_grp[9][8];
  __shared__ double s_mean[3];
  constexpr int kWarps = kBatch / NP / 32;
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  double v[3][NP];
#pragma unroll
  for (int p = 0; p < NP; ++p) {
    v[0][p] = valid[p] ? vh[p] : 0.0;
    v[1][p] = valid[p] ? vb[p] : 0.0;
    v[2][p] = valid[p] ? __dsub_rn(vh[p], vb[p]) : 0.0;
  }
#pragma unroll
  for (int f = 0; f < 3; ++f)
#pragma unroll
    for (int p = 0; p < NP; ++p) {
      const double s = warp_sum(v[f][p], 16);
      if (lane == 0) s_grp[f][warp + p * kWarps] = s;
    }
  __syncthreads();
  if (warp == 0) {
#pragma unroll
    for (int f = 0; f < 3; ++f) {
      const double g = warp_sum(lane < 8 ? s_grp[f][lane] : 0.0, 4);
      if (lane == 0) s_mean[f] = __ddiv_rn(g, static_cast<double>(count));
    }
  }
  __syncthreads();
  double mean[3] = {s_mean[0], s_mean[1], s_mean[2]};
#pragma unroll
  for (int f = 0; f < 3; ++f)
#pragma unroll
    for (int p = 0; p < NP; ++p) {
      const double dv = valid[p] ? __dsub_rn(v[f][p], mean[f]) : 0.0;
      const double d2 = __dmul_rn(dv, dv);
      const double d3 = __dmul_rn(d2, dv);
      const double d4 = __dmul_rn(d2, d2);
      const double s2 = warp_sum(d2, 16);
      const double s3 = warp_sum(d3, 16);
      const double s4 = warp_sum(d4, 16);
      if (lane == 0) {
        s_grp[3 * f + 0][warp + p * kWarps] = s2;
        s_grp[3 * f + 1][warp + p * kWarps] = s3;
        s_grp[3 * f + 2][warp + p * kWarps] = s4;
      }
    }
  __syncthreads();
  if (warp == 0) {
#pragma unroll
    for (int q = 0; q < 9; ++q) {
      const double g = warp_sum(lane < 8 ? s_grp[q][lane] : 0.0, 4);
      if (lane == 0) out15[5 * (q / 3) + 2 + (q % 3)] = g;
    }
    if (lane == 0) {
#pragma unroll
      for (int f = 0; f < 3; ++f) {
        out15[5 * f + 0] = static_cast<double>(count);
        out15[5 * f + 1] = mean[f];
      }
    }
  }
}

// --------------------------------------------------- the path kernel -------
__device__ __forceinline__ void note_fail(uint64_t& fk, bool bad, uint64_t n, uint32_t stage) {
  if (bad) {
    const uint64_t ord = (n << 3) | stage;
    fk = ord < fk ? ord : fk;
  }
}

template <class Arith, bool KAHAN, int LEGS, bool APPROX>
__global__ void __launch_bounds__(kBatch / Arith::NP, 3 * Arith::NP)
    level_kernel(const __grid_constant__ LevelArgs A) {
  using T = typename Arith::T;
  constexpr int NP = Arith::NP;
  constexpr bool kHat = (LEGS & 1) != 0;
  constexpr bool kBar = (LEGS & 2) != 0;
  constexpr bool kNeedExact = kHat || !APPROX;

  extern __shared__ double s_table[];
  __shared__ double s_erfcx[kNeedExact ? kErfcxWords : 1];
  if constexpr (kNeedExact) stage_erfcx(s_erfcx);
  TableView tab{};
  if constexpr (APPROX) {
    for (int i = threadIdx.x; i < kTableRows * A.K; i += blockDim.x) s_table[i] = A.table[i];
    tab = table_view(s_table, A.K, A.degree, A.dyadic, A.tail);
  }
  __syncthreads();

  const Arith ar(A);
  const uint64_t batch = A.batch0 + blockIdx.x;
  const uint64_t first = batch * kBatch;
  const uint64_t left = A.n_paths - first;
  const int count = left < kBatch ? static_cast<int>(left) : kBatch;

  uint64_t local[NP];
  bool valid[NP];
  uint64_t kc[NP];    // key + counter * C3, strength-reduced (uniform.hpp:25)
  uint64_t fk[NP];    // first failure ord of the path
  double xhf[NP], xhc[NP];
#pragma unroll
  for (int p = 0; p < NP; ++p) {
    const int slot = threadIdx.x + p * blockDim.x;
    local[p] = first + slot;
    valid[p] = slot < count;
    kc[p] = mix64(A.seed_key ^ mix64(A.path_base + local[p] + 0xbf58476d1ce4e5b9ull));
    fk[p] = kNoFail;
    xhf[p] = A.x0;
    xhc[p] = A.x0;
  }
  const T mu_l = ar.c(A.mu_l, A.h_mu), sg_l = ar.c(A.sigma_l, A.h_sigma);
  const T dtf_l = ar.c(A.dtf_l, A.h_dtf), sdtf_l = ar.c(A.sdtf_l, A.h_sdtf);
  const T dtc_l = ar.c(A.dtc_l, A.h_dtc);
  T xbf = ar.c(A.x0_l, A.h_x0);
  T xbc = xbf;
  T cmpf = ar.zero(), cmpc = ar.zero();
  bool range_bad = false;
  const uint64_t zstride = 1ull << A.level;

  // One uniform per path -> exact Z (hat legs, or bar legs without a table),
  // approximate Z~, and R(Z~) packed for the bar legs (sde.hpp:256-258).
  auto draw = [&](uint64_t n, double (&z)[NP], T& zb) {
    double zl[NP];
#pragma unroll
    for (int p = 0; p < NP; ++p) {
      const uint64_t w = mix64(mix64(kc[p]));
      kc[p] += 0x94d049bb133111ebull;
      const uint64_t top = w >> 11;
      note_fail(fk[p], top == kTopDraw, n, kStageDraw);
      const double u = __dadd_rn(__dmul_rn(__ull2double_rn(top), 0x1p-53), 0x1p-54);
      z[p] = kNeedExact ? phi_inv(u, s_erfcx) : 0.0;
      if (A.z_out != nullptr && valid[p]) A.z_out[local[p] * zstride + n] = z[p];
      if constexpr (APPROX) {
        zl[p] = approx_inv(tab, u);
      } else {
        zl[p] = z[p];
      }
    }
    if constexpr (kBar) zb = ar.lift(zl);
  };

  // em_step (sde.hpp:60-68), carrier
  auto hat_fine = [&](const double (&z)[NP], uint64_t n) {
#pragma unroll
    for (int p = 0; p < NP; ++p) {
      const double x = xhf[p];
      const double drift = __dmul_rn(__dmul_rn(A.mu, x), A.dtf);
      const double diff = __dmul_rn(__dmul_rn(__dmul_rn(A.sigma, x), A.sdtf), z[p]);
      xhf[p] = __dadd_rn(x, __dadd_rn(drift, diff));
      note_fail(fk[p], nonfinite64(xhf[p]), n, kStageHatFine);
    }
  };
  // em_step / em_step_kahan (sde.hpp:60-68, 96-105) in the bar precision
  auto bar_fine = [&](T zb, uint64_t n) {
    const T x = xbf;
    const T drift = ar.mul(ar.mul(mu_l, x), dtf_l);
    const T diff = ar.mul(ar.mul(ar.mul(sg_l, x), sdtf_l), zb);
    const T inc = ar.add(drift, diff);
    if constexpr (KAHAN) {  // kahan_accumulate (sde.hpp:85-92)
      const T y = ar.sub(inc, cmpf);
      const T s = ar.add(x, y);
      cmpf = ar.sub(ar.sub(s, x), y);
      xbf = s;
    } else {
      xbf = ar.add(x, inc);
    }
    const uint32_t m = ar.bad(xbf);
#pragma unroll
    for (int p = 0; p < NP; ++p) note_fail(fk[p], (m >> p) & 1u, n, kStageBarFine);
    range_bad |= ar.range(xbf);
  };
  // em_step_dw / em_step_kahan_dw (sde.hpp:72-80, 107-116)
  auto coarse = [&](const double (&z0)[NP], const double (&z1)[NP], T zb0, T zb1, uint64_t n) {
    if constexpr (kHat) {
#pragma unroll
      for (int p = 0; p < NP; ++p) {
        const double dw = __dadd_rn(__dmul_rn(A.sdtf, z0[p]), __dmul_rn(A.sdtf, z1[p]));
        const double x = xhc[p];
        const double drift = __dmul_rn(__dmul_rn(A.mu, x), A.dtc);
        const double diff = __dmul_rn(__dmul_rn(A.sigma, x), dw);
        xhc[p] = __dadd_rn(x, __dadd_rn(drift, diff));
        note_fail(fk[p], nonfinite64(xhc[p]), n, kStageHatCoarse);
      }
    }
    if constexpr (kBar) {
      const T dw = ar.add(ar.mul(sdtf_l, zb0), ar.mul(sdtf_l, zb1));
      const T x = xbc;
      const T drift = ar.mul(ar.mul(mu_l, x), dtc_l);
      const T diff = ar.mul(ar.mul(sg_l, x), dw);
      const T inc = ar.add(drift, diff);
      if constexpr (KAHAN) {
        const T y = ar.sub(inc, cmpc);
        const T s = ar.add(x, y);
        cmpc = ar.sub(ar.sub(s, x), y);
        xbc = s;
      } else {
        xbc = ar.add(x, inc);
      }
      const uint32_t m = ar.bad(xbc);
#pragma unroll
      for (int p = 0; p < NP; ++p) note_fail(fk[p], (m >> p) & 1u, n, kStageBarCoarse);
      range_bad |= ar.range(xbc);
    }
  };

  if (A.level == 0) {  // sde.hpp:237-249: one draw, fine legs only, coarse := 0
    double z[NP];
    T zb = ar.zero();
    draw(0, z, zb);
    if constexpr (kHat) hat_fine(z, 0);
    if constexpr (kBar) bar_fine(zb, 0);
  } else {
    const uint64_t halves = 1ull << (A.level - 1);
    for (uint64_t m = 0; m < halves; ++m) {  // sde.hpp:251-277
      double z0[NP], z1[NP];
      T zb0 = ar.zero(), zb1 = ar.zero();
      draw(2 * m, z0, zb0);
      draw(2 * m + 1, z1, zb1);
      if constexpr (kHat) hat_fine(z0, 2 * m);
      if constexpr (kBar) bar_fine(zb0, 2 * m);
      if constexpr (kHat) hat_fine(z1, 2 * m + 1);
      if constexpr (kBar) bar_fine(zb1, 2 * m + 1);
      coarse(z0, z1, zb0, zb1, 2 * m + 1);
    }
  }

  // terminal values -> payoff -> per-path differences (mlmc.hpp:86-90)
  double dh[NP], db[NP];
#pragma unroll
  for (int p = 0; p < NP; ++p) {
    const double hf = kHat ? xhf[p] : 0.0;
    const double hc = (kHat && A.level > 0) ? xhc[p] : 0.0;
    const double bf = kBar ? ar.get(xbf, p) : 0.0;
    const double bc = (kBar && A.level > 0) ? ar.get(xbc, p) : 0.0;
    if (A.path_out != nullptr && valid[p]) {
      double* o = A.path_out + 4 * local[p];
      o[0] = hf;
      o[1] = hc;
      o[2] = bf;
      o[3] = bc;
    }
    double pf_h = hf, pc_h = hc, pf_b = bf, pc_b = bc;
    if (A.payoff == 1) {
      pf_h = fmax(__dsub_rn(hf, A.strike), 0.0);
      pf_b = fmax(__dsub_rn(bf, A.strike), 0.0);
      pc_h = A.level > 0 ? fmax(__dsub_rn(hc, A.strike), 0.0) : 0.0;
      pc_b = A.level > 0 ? fmax(__dsub_rn(bc, A.strike), 0.0) : 0.0;
    }
    dh[p] = kHat ? __dsub_rn(pf_h, pc_h) : 0.0;
    db[p] = kBar ? __dsub_rn(pf_b, pc_b) : 0.0;
    if (valid[p] && fk[p] != kNoFail) {
      const uint64_t n = fk[p] >> 3;
      const uint32_t stage = static_cast<uint32_t>(fk[p] & 7u);
      uint32_t kind = stage == kStageDraw ? kKindU1 : kKindNonFinite;
      if (Arith::kIeee && (stage == kStageBarFine || stage == kStageBarCoarse)) kind = kKindState;
      const uint64_t step = n < (1ull << 22) ? n : (1ull << 22) - 1;
      atomicMin(A.err_key, static_cast<unsigned long long>((local[p] << 24) |
                                                           (static_cast<uint64_t>(kind) << 22) |
                                                           step));
    }
  }
  if (range_bad) atomicOr(A.range_flag, 1u);

  if (A.path_diff != nullptr) {
#pragma unroll
    for (int p = 0; p < NP; ++p)
      if (valid[p]) {
        const uint64_t r = local[p] - A.batch0 * kBatch;  // slice-relative
        A.path_diff[2 * r + 0] = dh[p];
        A.path_diff[2 * r + 1] = db[p];
      }
  }
  if (A.batch_acc != nullptr) {
    batch_moments<NP>(dh, db, valid, count, A.batch_acc + 15 * blockIdx.x);
  }
}

// ----------------------------------------------------------- moments -------
struct Acc {
  double n, mean, m2, m3, m4;
};

// MomentAccumulator::merge (stats.hpp:29-54), same expression trees.
__device__ __forceinline__ void acc_merge(Acc& a, const Acc& b) {
  if (b.n == 0.0) return;
  if (a.n == 0.0) {
    a = b;
    return;
  }
  const double na = a.n, nb = b.n;
  const double n = na + nb;
  const double d = b.mean - a.mean;
  const double d2 = d * d;
  const double m2 = a.m2 + b.m2 + d2 * na * nb / n;
  const double m3 = a.m3 + b.m3 + d2 * d * na * nb * (na - nb) / (n * n) +
                    3.0 * d * (na * b.m2 - nb * a.m2) / n;
  const double m4 = a.m4 + b.m4 + d2 * d2 * na * nb * (na * na - na * nb + nb * nb) / (n * n * n) +
                    6.0 * d2 * (na * na * b.m2 + nb * nb * a.m2) / (n * n) +
                    4.0 * d * (na * b.m3 - nb * a.m3) / n;
  a.mean = a.mean + d * nb / n;
  a.m2 = m2;
  a.m3 = m3;
  a.m4 = m4;
  a.n = n;
}

// MomentAccumulator::add (stats.hpp:15-27), same expression trees.
__device__ __forceinline__ void acc_add(Acc& a, double x) {
  const double before = a.n;
  const double dn = a.n + 1.0;
  a.n = dn;
  const double delta = x - a.mean;
  const double dl = delta / dn;
  const double dl2 = dl * dl;
  const double t1 = delta * dl * before;
  a.mean = a.mean + dl;
  a.m4 = a.m4 + (t1 * dl2 * (dn * dn - 3.0 * dn + 3.0) + 6.0 * dl2 * a.m2 - 4.0 * dl * a.m3);
  a.m3 = a.m3 + (t1 * dl * (dn - 2.0) - 3.0 * dl * a.m2);
  a.m2 = a.m2 + t1;
}

__device__ __forceinline__ Acc load_acc(const double* p) { return Acc{p[0], p[1], p[2], p[3], p[4]}; }
__device__ __forceinline__ void store_acc(double* p, const Acc& a) {
  p[0] = a.n;
  p[1] = a.mean;
  p[2] = a.m2;
  p[3] = a.m3;
  p[4] = a.m4;
}

// Chunk tree: 1024 batch slots (empty past the end), pairwise Pebay merges.
__global__ void __launch_bounds__(kChunkThreads)
    chunk_reduce_kernel(const double* __restrict__ batch_acc, uint64_t n_batches,
                        double* __restrict__ chunk_acc) {
  __shared__ Acc s[kChunkThreads];
  const uint64_t b0 = static_cast<uint64_t>(blockIdx.x) * kChunkBatches;
  const int t = threadIdx.x;
  for (int f = 0; f < 3; ++f) {
    Acc a{0, 0, 0, 0, 0}, b{0, 0, 0, 0, 0};
    const uint64_t i0 = b0 + 2 * t, i1 = b0 + 2 * t + 1;
    if (i0 < n_batches) a = load_acc(batch_acc + 15 * i0 + 5 * f);
    if (i1 < n_batches) b = load_acc(batch_acc + 15 * i1 + 5 * f);
    acc_merge(a, b);
    s[t] = a;
    __syncthreads();
    for (int width = kChunkThreads / 2; width >= 1; width >>= 1) {
      Acc r{0, 0, 0, 0, 0};
      if (t < width) {
        r = s[2 * t];
        acc_merge(r, s[2 * t + 1]);
      }
      __syncthreads();
      if (t < width) s[t] = r;
      __syncthreads();
    }
    if (t == 0) store_acc(chunk_acc + 15 * blockIdx.x + 5 * f, s[0]);
    __syncthreads();
  }
}

// Reference order: one thread per (batch, family) adds its <= 256 values in
// path order, exactly run_batch's loop (mlmc.hpp:78-93).
__global__ void sequential_batch_kernel(const double* __restrict__ path_diff, uint64_t n_paths,
                                        double* __restrict__ batch_acc) {
  const uint64_t idx = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint64_t n_batches = (n_paths + kBatch - 1) / kBatch;
  if (idx >= 3 * n_batches) return;
  const uint64_t b = idx / 3;
  const int f = static_cast<int>(idx % 3);
  Acc a{0, 0, 0, 0, 0};
  const uint64_t end = (b + 1) * kBatch < n_paths ? (b + 1) * kBatch : n_paths;
  for (uint64_t i = b * kBatch; i < end; ++i) {
    const double h = path_diff[2 * i], br = path_diff[2 * i + 1];
    acc_add(a, f == 0 ? h : (f == 1 ? br : __dsub_rn(h, br)));
  }
  store_acc(batch_acc + 15 * b + 5 * f, a);
}

// op 0: exact Gaussian (product path), 1: approximate (table), 2: the
// reference's formula on libdevice, 3: erfc core on t in [0, 6.5).
__global__ void inv_cdf_kernel(const double* __restrict__ u, uint64_t n,
                               const double* __restrict__ table, int K, int degree, int dyadic,
                               double tail, int op, double* __restrict__ out) {
  __shared__ double s_erfcx[kErfcxWords];
  stage_erfcx(s_erfcx);
  __syncthreads();
  const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double x = u[i];
  double r = 0.0;
  if (op == 0) {
    r = phi_inv(x, s_erfcx);
  } else if (op == 1) {
    const TableView t = table_view(table, K, degree, dyadic, tail);
    r = approx_inv(t, x);
  } else if (op == 2) {
    r = math::phi_inv_libdevice(x);
  } else {
    r = math::erfc_fast(x, s_erfcx);
  }
  out[i] = r;
}

// ------------------------------------------------------ pipe peaks ---------
// Roofline denominators for this non-tensor path: many independent
// dependency chains per thread so the pipe, not latency, is the limit.
// One "op" = one lane-operation (one SASS instruction x 32 lanes / 32).
constexpr int kPeakChains = 8;
constexpr int kPeakIters = 4096;

__global__ void __launch_bounds__(256) peak_fp64_kernel(double seed, double* sink) {
  double a[kPeakChains];
#pragma unroll
  for (int c = 0; c < kPeakChains; ++c) a[c] = seed + threadIdx.x + c;
  const double m = 1.0000000001, k = 1e-9;
  for (int i = 0; i < kPeakIters; ++i) {
#pragma unroll
    for (int c = 0; c < kPeakChains; ++c) a[c] = __fma_rn(a[c], m, k);
  }
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < kPeakChains; ++c) s += a[c];
  if (s == 12345.678) sink[0] = s;
}

__global__ void __launch_bounds__(256) peak_fp32_kernel(float seed, float* sink) {
  float a[kPeakChains];
#pragma unroll
  for (int c = 0; c < kPeakChains; ++c) a[c] = seed + threadIdx.x + c;
  const float m = 1.0001f, k = 1e-7f;
  for (int i = 0; i < kPeakIters; ++i) {
#pragma unroll
    for (int c = 0; c < kPeakChains; ++c) a[c] = __fmaf_rn(a[c], m, k);
  }
  float s = 0.0f;
#pragma unroll
  for (int c = 0; c < kPeakChains; ++c) s += a[c];
  if (s == 12345.678f) sink[0] = s;
}

__global__ void __launch_bounds__(256) peak_half2_kernel(float seed, float* sink) {
  __half2 a[kPeakChains];
#pragma unroll
  for (int c = 0; c < kPeakChains; ++c) a[c] = __float2half2_rn(seed + 0.001f * (threadIdx.x + c));
  const __half2 m = __float2half2_rn(1.0001f), k = __float2half2_rn(1e-4f);
  for (int i = 0; i < kPeakIters; ++i) {
#pragma unroll
    for (int c = 0; c < kPeakChains; ++c) a[c] = __hfma2(a[c], m, k);
  }
  float s = 0.0f;
#pragma unroll
  for (int c = 0; c < kPeakChains; ++c) s += __low2float(a[c]) + __high2float(a[c]);
  if (s == 12345.678f) sink[0] = s;
}

__global__ void __launch_bounds__(256) peak_imad64_kernel(uint64_t seed, uint64_t* sink) {
  uint64_t a[kPeakChains];
#pragma unroll
  for (int c = 0; c < kPeakChains; ++c) a[c] = seed + threadIdx.x + c;
  for (int i = 0; i < kPeakIters / 4; ++i) {
#pragma unroll
    for (int c = 0; c < kPeakChains; ++c) a[c] = a[c] * 0xff51afd7ed558ccdull + 0x9e3779b97f4a7c15ull;
  }
  uint64_t s = 0;
#pragma unroll
  for (int c = 0; c < kPeakChains; ++c) s ^= a[c];
  if (s == 12345) sink[0] = s;
}

// ------------------------------------------------------------ dispatch -----
constexpr int kMaxTableK = 1024;
constexpr int kMaxDynSmem = kTableRows * kMaxTableK * 8;

template <class Arith, bool KAHAN, int LEGS, bool APPROX>
cudaError_t configure_one() {
  return cudaFuncSetAttribute(level_kernel<Arith, KAHAN, LEGS, APPROX>,
                              cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxDynSmem);
}

template <class Arith, bool KAHAN, int LEGS, bool APPROX>
cudaError_t launch_one(const LevelArgs& A, cudaStream_t s) {
  const size_t smem = APPROX ? static_cast<size_t>(kTableRows) * A.K * sizeof(double) : 0;
  level_kernel<Arith, KAHAN, LEGS, APPROX>
      <<<static_cast<unsigned>(A.n_batches), kBatch / Arith::NP, smem, s>>>(A);
  return cudaGetLastError();
}

template <class Arith, bool KAHAN, int LEGS>
cudaError_t pick_approx(const LevelArgs& A, cudaStream_t s) {
  return A.table != nullptr ? launch_one<Arith, KAHAN, LEGS, true>(A, s)
                            : launch_one<Arith, KAHAN, LEGS, false>(A, s);
}

template <class Arith, bool KAHAN>
cudaError_t pick_legs(const LevelArgs& A, cudaStream_t s) {
  if (A.legs == 1) return launch_one<ArithCarrier, false, 1, false>(A, s);
  if (A.legs == 2) return pick_approx<Arith, KAHAN, 2>(A, s);
  return pick_approx<Arith, KAHAN, 3>(A, s);
}

template <class Arith>
cudaError_t pick_kahan(const LevelArgs& A, bool kahan, cudaStream_t s) {
  return kahan ? pick_legs<Arith, true>(A, s) : pick_legs<Arith, false>(A, s);
}

template <class Arith>
cudaError_t configure_arith() {
  cudaError_t e = cudaSuccess;
  auto acc = [&](cudaError_t x) { if (e == cudaSuccess) e = x; };
  acc(configure_one<Arith, false, 2, true>());
  acc(configure_one<Arith, true, 2, true>());
  acc(configure_one<Arith, false, 3, true>());
  acc(configure_one<Arith, true, 3, true>());
  return e;
}

}  // namespace

int configure_kernels() {
  // math constants live in an uninitialised __constant__ block (see
  // lpmc_math.cuh): upload them for the current device first
  cudaError_t e = cudaMemcpyToSymbol(math::kMath, math::kMathHost, sizeof(math::kMathHost));
  if (e == cudaSuccess) e = configure_arith<ArithCarrier>();
  if (e == cudaSuccess) e = configure_arith<ArithF32>();
  if (e == cudaSuccess) e = configure_arith<ArithF32Round>();
  if (e == cudaSuccess) e = configure_arith<ArithF64Round>();
  if (e == cudaSuccess) e = configure_arith<ArithHalf2>();
  return static_cast<int>(e);
}

LaunchResult launch_paths(const LevelArgs& A, BarArith arith, bool kahan, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaError_t e = cudaSuccess;
  switch (arith) {
    case BarArith::kCarrier: e = pick_kahan<ArithCarrier>(A, kahan, s); break;
    case BarArith::kF32: e = pick_kahan<ArithF32>(A, kahan, s); break;
    case BarArith::kF32Round: e = pick_kahan<ArithF32Round>(A, kahan, s); break;
    case BarArith::kF64Round: e = pick_kahan<ArithF64Round>(A, kahan, s); break;
    case BarArith::kHalf2: e = pick_kahan<ArithHalf2>(A, kahan, s); break;
  }
  return {static_cast<int>(e), 1};
}

LaunchResult launch_chunk_reduce(const double* batch_acc, uint64_t n_batches, uint64_t n_chunks,
                                 double* chunk_acc, void* stream) {
  chunk_reduce_kernel<<<static_cast<unsigned>(n_chunks), kChunkThreads, 0,
                        static_cast<cudaStream_t>(stream)>>>(batch_acc, n_batches, chunk_acc);
  return {static_cast<int>(cudaGetLastError()), 1};
}

LaunchResult launch_sequential_batches(const double* path_diff, uint64_t n_paths,
                                       double* batch_acc, void* stream) {
  const uint64_t n_batches = (n_paths + kBatch - 1) / kBatch;
  const uint64_t threads = 3 * n_batches;
  const unsigned blocks = static_cast<unsigned>((threads + 127) / 128);
  sequential_batch_kernel<<<blocks, 128, 0, static_cast<cudaStream_t>(stream)>>>(
      path_diff, n_paths, batch_acc);
  return {static_cast<int>(cudaGetLastError()), 1};
}

int measure_pipe_peaks(double* out4) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  void* sink = nullptr;
  cudaError_t e = cudaMalloc(&sink, 64);
  if (e != cudaSuccess) return static_cast<int>(e);
  cudaEvent_t t0, t1;
  cudaEventCreate(&t0);
  cudaEventCreate(&t1);
  const unsigned blocks = static_cast<unsigned>(sms) * 8u;
  const double lanes = static_cast<double>(blocks) * 256.0;
  for (int which = 0; which < 4 && e == cudaSuccess; ++which) {
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(t0);
      switch (which) {
        case 0: peak_fp64_kernel<<<blocks, 256>>>(1.0, static_cast<double*>(sink)); break;
        case 1: peak_fp32_kernel<<<blocks, 256>>>(1.0f, static_cast<float*>(sink)); break;
        case 2: peak_half2_kernel<<<blocks, 256>>>(1.0f, static_cast<float*>(sink)); break;
        default: peak_imad64_kernel<<<blocks, 256>>>(1ull, static_cast<uint64_t*>(sink)); break;
      }
      cudaEventRecord(t1);
      e = cudaEventSynchronize(t1);
      float ms = 0.0f;
      cudaEventElapsedTime(&ms, t0, t1);
      if (rep > 0 && ms < best) best = ms;  // rep 0 warms up
    }
    const double iters = which == 3 ? kPeakIters / 4 : kPeakIters;
    // lane-operations per second (one FMA = one op; half2: 2 lanes per op)
    const double ops = lanes * iters * kPeakChains * (which == 2 ? 2.0 : 1.0);
    out4[which] = ops / (best * 1e-3);
  }
  cudaEventDestroy(t0);
  cudaEventDestroy(t1);
  cudaFree(sink);
  if (e == cudaSuccess) e = cudaGetLastError();
  return static_cast<int>(e);
}

LaunchResult launch_inv_cdf(const double* u, uint64_t n, const double* table, int K, int degree,
                            int dyadic, double tail, int op, double* out, void* stream) {
  const unsigned blocks = static_cast<unsigned>((n + 255) / 256);
  inv_cdf_kernel<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      u, n, table, K, degree, dyadic, tail, op, out);
  return {static_cast<int>(cudaGetLastError()), 1};
}

}  // namespace lpmc_b200
