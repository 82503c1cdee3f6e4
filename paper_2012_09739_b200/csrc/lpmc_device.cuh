// Device building blocks of the level sampler (shared by every kernel TU):
// counter RNG, approximate inverse CDF, emulated rounding, bar-leg arithmetic
// policies, the fixed batch-moment tree and the Pebay merge.
//
// Reference cross-walk (file:line under /root/reference/proj/include/lpmc):
//   mix64 / stream_word / next      uniform.hpp:13-41
//   InvCdfApprox::operator()        invcdf_approx.hpp:44-90
//   round_to_precision / fp_*       softfloat.hpp:69-111
//   MomentAccumulator add/merge     stats.hpp:15-54
#pragma once

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "lpmc_internal.h"
#include "lpmc_math.cuh"

namespace lpmc_b200 {
namespace dev {

constexpr int kBatch = 256;
constexpr int kChunkBatches = 1024;
constexpr int kChunkThreads = 512;
constexpr uint64_t kTopDraw = 0x1FFFFFFFFFFFFFull;  // (w >> 11) that rounds u to 1.0
constexpr uint64_t kNoFail = ~0ull;
constexpr int kMathWords = math::kMathTableWords;  // incl. the glibc-mode tables
constexpr int kFastMathWords = math::kGlibcOff;     // the fast mode's tables only
constexpr uint64_t kHalfDraw = 1ull << 52;  // (w >> 11) that rounds u to exactly 1/2

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

// key of path i: mix64(mix64(seed + phi) ^ mix64(i + c2)) (uniform.hpp:23-24),
// the first factor hoisted by the host (LevelArgs::seed_key).
__device__ __forceinline__ uint64_t path_key(uint64_t seed_key, uint64_t path) {
  return mix64(seed_key ^ mix64(path + 0xbf58476d1ce4e5b9ull));
}

// The draw b = w >> 11 of u = b 2^-53 + 2^-54 with w = mix64(mix64(key + ctr
// c3)); the running kc = key + ctr c3 is strength-reduced (uniform.hpp:25,
// :38-41).  The hot loop keeps b, not u: everything the transforms take
// from u is derived from it; the half-plane tests are then integer compares
// on its high word instead of FP64 compares.
// b == kTopDraw: u rounds to 1 (the reference throws, gaussian.hpp:60);
// b == kHalfDraw: u rounds to exactly 1/2 (both transforms return exactly 0).
constexpr uint64_t kCounterStep = 0x94d049bb133111ebull;  // uniform.hpp:26
__device__ __forceinline__ uint64_t next_draw(uint64_t& kc) {
  const uint64_t w = mix64(mix64(kc));
  kc += kCounterStep;
  return w >> 11;
}

// (double)b 2^-53 + 2^-54 (uniform.hpp:40): b < 2^53 converts exactly and the
// product by 2^-53 is exact, so the reference's one rounding (of the sum) is
// the FMA's one rounding -- bitwise, one FP64 operation fewer.
__device__ __forceinline__ double uniform_of(uint64_t b) {
  return __fma_rn(__ull2double_rn(b), 0x1p-53, 0x1p-54);
}

// erfcx records + 2^(j/64) pairs into (16-byte aligned) shared memory
__device__ __forceinline__ void stage_math(double* s_math, int words = kMathWords) {
  for (int i = threadIdx.x; i < words; i += blockDim.x) s_math[i] = math::kMathTable[i];
}

// the fast mode's tables in the lane-private layout (math::LaneTab)
constexpr int kLaneWords = math::kLaneWords;
__device__ __forceinline__ void stage_lane(double* s_lane) {
  for (int i = threadIdx.x; i < kLaneWords; i += blockDim.x)
    s_lane[i] = math::kMathTable[math::lane_source(i)];
}

// ------------------------------------------- approximate inverse CDF -------
// Shared-memory table.  Dyadic layout (K <= 32): one 6-double record per
// interval {3 - 2^(j+3), 2^(j+3), c0, c1, c2, c3} (128-bit loads).  General
// layout: one record of `stride` doubles per interval, {a_j, b_j - a_j, c0,
// c1} (degree 1) or {.., c2, c3} (degree 3), then the K v-thresholds, then
// 1 / step_w.
struct TableView {
  const double* base;
  int stride, K, degree, dyadic, simple;
  double tail;
  uint32_t saddr = 0;  // shared-space address of `base` (the level kernel's reversed copy)
};

// 128-bit load from a shared-space address (no generic-to-shared conversion
// in the hot loop: the address is a uniform base plus the record offset)
__device__ __forceinline__ math::D2 lds2(uint32_t saddr) {
  math::D2 r;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(r.a), "=d"(r.b) : "r"(saddr));
  return r;
}

// InvCdfApprox::operator() (invcdf_approx.hpp:44-90).
//  * dyadic tables (K <= 32, w_max = K+1): the reference's j = floor(-log2 v)
//    - 1 read from the exponent of v = 1 - u' (exact on the 2^-53 grid,
//    SURVEY.md §A3); u' in [a_j, b_j) with a_j = 1 - 2^-(j+1), b_j - a_j =
//    2^-(j+2), so t in [-1, 1) and the reference's clamps are no-ops.  Its
//    t = RN(2 (u' - a_j) / (b_j - a_j) - 1) has only that last rounding
//    (u' - a_j is exact by Sterbenz, the rest are powers of two), and the
//    exact value is u' 2^(j+3) - (2^(j+3) - 3): one FMA, bitwise equal.
//  * general K: index from host thresholds that reproduce the reference's
//    log2-based index on every representable v; division and clamps as the
//    reference.
//  * `simple` (host-proved: every c0 != 0 and c2 = c3 = +0): the reference's
//    (c0 + c1 t) + 0 p2 + 0 p3 equals c0 + c1 t including the sign of zero.
//  * lower: u < 1/2 (the sampler passes the integer test on its draw).
//  * EXACT_HALF: exactly 0 at u = 1/2; the hot loop replays such draws.
//  * TAB == kTabDyadicLinear: the host proved dyadic && simple && degree 1
//    (every BASELINE table): the same arithmetic without the run-time kind
//    tests, so a draw's approximate Gaussian is straight-line code.
enum : int { kTabNone = 0, kTabDyadicLinear = 1, kTabGeneric = 2 };

template <bool EXACT_HALF = true, int TAB = kTabGeneric>
__device__ __forceinline__ double approx_inv(const TableView& t, double u, bool lower) {
  const double up = lower ? 1.0 - u : u;  // fl(1-u) for the lower half (:47-49)
  double r;
  if constexpr (TAB == kTabDyadicLinear) {
    // floor(-log2 v), v = 1 - u' (exact, Sterbenz), needs the binade of v with
    // an exact power of two counted into the binade below.  u' and v sit on
    // the 2^-53 grid, so (1 - 2^-53) - u' = v - 2^-53 is exact and has that
    // binade: a power of two drops into the binade below, any other grid
    // point of a binade stays (it is at least one grid step above the
    // binade's start).  v = 2^-53 gives 0 (exponent field 0: the last tail
    // record, which is the reference's j = 52), v = 0 (u' == 1: u == 1, where
    // the reference throws and the path is replayed checked; or the smallest
    // draw u = 2^-54, whose 1 - u rounds to 1 and which the reference maps to
    // the tail value) gives -2^-53, whose sign bit sends the unsigned minimum
    // to the last tail record too.  One FP64 subtraction and a shift instead
    // of a subtraction, a 64-bit decrement and a shift.  Records j >= K are the
    // host's tail records (c0 = tail, c1 = 0: tail + 0 * s = tail), so neither
    // the reference's clamp nor its tail test needs an instruction.
    const double vm = __dsub_rn(0x1.fffffffffffffp-1, up);
    const uint32_t eb = static_cast<uint32_t>(__double2hiint(vm)) >> 20;
    const uint32_t j = min(1021u - eb, static_cast<uint32_t>(kDyadicRecords - 1));
    LPMC_DCHECK(j < static_cast<uint32_t>(kDyadicRecords));
    const double* b = t.base + 6 * j;
    const math::D2 cw = math::load2(b);
    const math::D2 c01 = math::load2(b + 2);
    const double s = __fma_rn(up, cw.b, cw.a);
    r = __dadd_rn(c01.a, __dmul_rn(c01.b, s));
    r = math::flip_sign(r, lower);
    if constexpr (EXACT_HALF) r = u == 0.5 ? 0.0 : r;
    return r;
  }
  const double v = 1.0 - up;              // exact (Sterbenz)
  if (t.dyadic) {
    const uint64_t vb = static_cast<uint64_t>(__double_as_longlong(v));
    const int e = static_cast<int>(vb >> 52) - 1023;
    const int fl = (vb & 0xFFFFFFFFFFFFFull) == 0 ? -e : -e - 1;  // floor(-log2 v) >= 1
    const int j = min(fl - 1, t.K - 1);
    LPMC_DCHECK(j >= 0 && j < t.K);
    const double* b = t.base + 6 * j;
    const math::D2 cw = math::load2(b);
    const math::D2 c01 = math::load2(b + 2);
    const double s = __fma_rn(up, cw.b, cw.a);
    r = __dadd_rn(c01.a, __dmul_rn(c01.b, s));
    if (t.degree == 3 || (!t.simple && r == 0.0)) {
      const math::D2 c23 = math::load2(b + 4);
      const double p2 = 1.5 * s * s - 0.5;
      const double p3 = s * (2.5 * s * s - 1.5);
      r = r + c23.a * p2 + c23.b * p3;
    }
    r = fl >= t.K + 1 ? t.tail : r;  // w >= w_max: clamped tail
  } else {
    // J(v) = #{k in 1..K : v <= T_k} with the host thresholds T_k = thr[k-1]
    // (non-increasing); J == K is the tail.  Start from a float estimate of
    // the reference's floor((-log2 v - 1) / step_w) and walk to the exact J
    // (the walk alone is correct; the estimate makes it one or two compares).
    const int W = t.stride;  // record width: 4 (degree 1) or 6 (degree 3)
    const double* thr = t.base + W * t.K;
    const float inv_step = __double2float_rn(thr[t.K]);  // 1 / step_w, after T_K
    const float w = -__log2f(__double2float_rn(v));
    const float je = floorf((w - 1.0f) * inv_step);
    int J = je < 0.0f ? 0 : (je > static_cast<float>(t.K) ? t.K : static_cast<int>(je));
    while (J < t.K && v <= thr[J]) ++J;
    while (J > 0 && v > thr[J - 1]) --J;
    const int j = J < t.K ? J : t.K - 1;
    LPMC_DCHECK(J >= 0 && J <= t.K && j >= 0 && j < t.K);
    const double* rec = t.base + W * j;
    const math::D2 ad = math::load2(rec);       // a_j, b_j - a_j
    const math::D2 c01 = math::load2(rec + 2);  // c0, c1
    double s = (2.0 * (up - ad.a)) / ad.b;
    s = s - 1.0;
    s = s < -1.0 ? -1.0 : s;
    s = s > 1.0 ? 1.0 : s;
    r = c01.a + c01.b * s;
    if (t.degree == 3 || (!t.simple && r == 0.0)) {
      // degree-1 tables have c2 = c3 = +0 (invcdf_approx.hpp:124-133)
      const math::D2 c23 = t.degree == 3 ? math::load2(rec + 4) : math::D2{0.0, 0.0};
      const double p2 = 1.5 * s * s - 0.5;
      const double p3 = s * (2.5 * s * s - 1.5);
      r = r + c23.a * p2 + c23.b * p3;
    }
    r = J >= t.K ? t.tail : r;
  }
  r = math::flip_sign(r, lower);
  if constexpr (EXACT_HALF) r = u == 0.5 ? 0.0 : r;
  return r;
}

// The dyadic-linear evaluation of the unchecked hot loop from the
// reflected draw: up = u > 1/2 ? u : fl(1 - u), sgn = 0x80000000 where the
// result is negated (u < 1/2), both shared with the exact transform.
// t is the kernel's REVERSED copy of the dyadic table (kRunCopyRecords
// records, staged by the level kernel): record r = e' - 969 holds interval
// j = 52 - r for r <= 52 (e' the biased exponent of v - 2^-53, see
// approx_inv), record 53 the tail value -- so the index is one shift-add and
// one unsigned minimum with immediates (v - 2^-53 <= 0: the wrapped or
// sign-carrying e' lands on record 53 or record 0, both tail records).
constexpr int kRunCopyRecords = kDyadicRecords + 1;
constexpr int kRunCopyWords = kRunCopyRecords * kDyadicRecord;
__device__ __forceinline__ int run_copy_source(int r) {  // forward record of reversed record r
  return r < kDyadicRecords ? kDyadicRecords - 1 - r : kDyadicRecords - 1;
}
__device__ __forceinline__ double approx_inv_up(const TableView& t, double up, uint32_t sgn) {
  const double vm = __dsub_rn(0x1.fffffffffffffp-1, up);  // see approx_inv
  const uint32_t r = min((static_cast<uint32_t>(__double2hiint(vm)) >> 20) - (1021u - 52u),
                         static_cast<uint32_t>(kRunCopyRecords - 1));
  LPMC_DCHECK(r < static_cast<uint32_t>(kRunCopyRecords) && t.saddr != 0u);
  const uint32_t b = t.saddr + r * (kDyadicRecord * 8u);
  const math::D2 cw = lds2(b);
  const math::D2 c01 = lds2(b + 16u);
  const double s = __fma_rn(up, cw.b, cw.a);
  return math::flip_sign_mask(__dadd_rn(c01.a, __dmul_rn(c01.b, s)), sgn);
}

template <bool EXACT_HALF = true, int TAB = kTabGeneric>
__device__ __forceinline__ double approx_inv(const TableView& t, double u) {
  return approx_inv<EXACT_HALF, TAB>(t, u, u < 0.5);
}

// u < 1/2 <=> b < 2^52 <=> high word < 2^20
__device__ __forceinline__ bool draw_lower(uint64_t b) {
  return static_cast<uint32_t>(b >> 32) < (1u << 20);
}

// ----------------------------------------------- rounding helpers ---------
// RNE of a binary64 value to m+1 significant bits by integer arithmetic on
// its pattern (== round_to_precision, softfloat.hpp:69-80, for normal
// operands; binary64 subnormals are scaled the way frexp/ldexp handle them).
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

// ------------------------------------------------- packed fp32 pairs ------
// (-DLPMC_PAIR, A/B only.)  sm_100 executes two fp32 lanes per instruction
// (FFMA2).  Measured on the C4 kernels: 7 % fewer warp-instructions, but
// FFMA2 holds the FMA pipe twice as long and the kernels ran 0-3 % slower
// (DESIGN.md section 8), so the scalar form is the default.  Every packed op is
// an fma.rn.f32x2 whose addend/multiplier constants come from the launch
// parameters (LevelArgs::f2_neg0 / f2_neg1), never immediates: with known
// constants ptxas fuses a multiply and a following add into one FFMA2 even
// though each is written with .rn, which would change the rounding.
// a * b + (-0) is the correctly rounded product (the sign of a zero product
// is kept); c + (-1) x is the correctly rounded difference c - x.
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ uint64_t pack2(float lo, float hi) {
  uint64_t d;
  asm("mov.b64 %0, {%1, %2};" : "=l"(d) : "f"(lo), "f"(hi));
  return d;
}
__device__ __forceinline__ float lo2(uint64_t v) {
  float a, b;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
  (void)b;
  return a;
}
__device__ __forceinline__ float hi2(uint64_t v) {
  float a, b;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
  (void)a;
  return b;
}

// ------------------------------------------------------ bar arithmetic -----
// Policies: T (state type), NP (paths per thread), mul/add/sub in the target
// precision, lift(z[NP]) = R(z) packed, get(x, p) -> double, bad(x) ->
// bitmask of non-finite lanes.  Native fp32 policies also track the state
// exponent range: they are bit-exact with the unbounded-exponent reference
// while states stay in [2^-32, 2^33) (no intermediate can then be subnormal
// or overflow); otherwise the host re-runs
// the level in the exact kF64Round emulation.
struct RangeNone {
  __device__ void track(__nv_bfloat16) {}
  __device__ void track(double) {}
  __device__ void track(float) {}
  __device__ void track(__half2) {}
  __device__ bool bad() const { return false; }
};
// |x| in [2^-32, 2^33) <=> (bits(|x|) - bits(2^-32)) < bits(2^33) - bits(2^-32)
// unsigned (a smaller |x| wraps to a huge value): one running maximum
// (LOP3 + VIADDMNMX per state update).
struct RangeF32 {
  static constexpr uint32_t kLo = 0x2f800000u, kHi = 0x50000000u;
  uint32_t worst = 0u;
  __device__ void track(float x) {
    worst = max(worst, (__float_as_uint(x) & 0x7fffffffu) - kLo);
  }
  __device__ bool bad() const { return worst >= kHi - kLo; }
};

// Guard of the folded binary64 legs (step_hat_pw, and step_bar_pw on the
// carrier arithmetic): |x| in [2^-300, 2^300] <=> (high word of |x|) - hw(2^-300) < hw(2^300) -
// hw(2^-300) unsigned; zero, subnormal and non-finite values are outside.
struct RangeF64 {
  static constexpr uint32_t kLo = (1023u - 300u) << 20, kHi = (1023u + 300u) << 20;
  uint32_t worst = 0u;
  __device__ void track(double x) {
    worst = max(worst, (static_cast<uint32_t>(__double2hiint(x)) & 0x7fffffffu) - kLo);
  }
  __device__ bool bad() const { return worst >= kHi - kLo; }
};

struct ArithCarrier {  // m >= 52
  using T = double;
  using Range = RangeF64;  // only the folded instances (PW) depend on it
  static constexpr int NP = 1;
  static constexpr bool kScaled = false;  // see ArithHalfScaled
  using Replay = ArithCarrier;
  static constexpr bool kRangeReplays = true;  // a path outside the guard is replayed (else: the launch is re-run)
  static constexpr bool kIeee = false;
  static constexpr bool kPair = false;  // no packed fp32 pairs (see ArithF32)
  // power-of-two step folding like the carrier (hat) legs: exact inside
  // RangeF64, checked on every state update; a path outside is replayed
  static constexpr bool kPow2 = true;
  __device__ explicit ArithCarrier(const LevelArgs&) {}
  __device__ T c(double d, uint16_t) const { return d; }
  __device__ T zero() const { return 0.0; }
  __device__ T mul(T a, T b) const { return __dmul_rn(a, b); }
  __device__ T add(T a, T b) const { return __dadd_rn(a, b); }
  __device__ T sub(T a, T b) const { return __dsub_rn(a, b); }
  __device__ T lift(const double (&z)[1]) const { return z[0]; }
  __device__ double get(T x, int) const { return x; }
  __device__ uint32_t bad(T x) const { return nonfinite64(x) ? 1u : 0u; }
};

struct ArithF32 {  // m == 23, native
  using T = float;
  using Range = RangeF32;
  static constexpr int NP = 1;
  static constexpr bool kScaled = false;  // see ArithHalfScaled
  using Replay = ArithF32;
  static constexpr bool kRangeReplays = false;  // a path outside the guard is replayed (else: the launch is re-run)
  static constexpr bool kIeee = false;
  // mul2: two independent products of one leg step in one FFMA2 (bitwise
  // the two scalar products)
#ifdef LPMC_PAIR  // A/B only: measured slower
  static constexpr bool kPair = true;
#else
  static constexpr bool kPair = false;
#endif
  static constexpr bool kPow2 = true;  // native range guard: step_bar_pw is exact
  uint64_t n0, n1, p1;
  __device__ explicit ArithF32(const LevelArgs& A)
      : n0(A.f2_neg0), n1(A.f2_neg1), p1(A.f2_neg1 & 0x7fffffff7fffffffull) {}
  __device__ uint64_t mul2(uint64_t a, uint64_t b) const { return ffma2(a, b, n0); }
  __device__ uint64_t add2(uint64_t a, uint64_t b) const { return ffma2(a, p1, b); }
  __device__ uint64_t sub2(uint64_t a, uint64_t b) const { return ffma2(b, n1, a); }
  __device__ float one() const { return lo2(p1); }  // +1.0f the compiler cannot fold
  __device__ T c(double d, uint16_t) const { return static_cast<float>(d); }  // exact
  __device__ T zero() const { return 0.0f; }
  __device__ T mul(T a, T b) const { return __fmul_rn(a, b); }
  __device__ T add(T a, T b) const { return __fadd_rn(a, b); }
  __device__ T sub(T a, T b) const { return __fsub_rn(a, b); }
  __device__ T lift(const double (&z)[1]) const { return __double2float_rn(z[0]); }
  __device__ double get(T x, int) const { return static_cast<double>(x); }
  __device__ uint32_t bad(T x) const { return nonfinite32(x) ? 1u : 0u; }
};

struct ArithF32Round {  // m <= 10: fp32 op (correctly rounded), then RNE to m+1 bits
  using T = float;
  using Range = RangeF32;
  static constexpr int NP = 1;
  static constexpr bool kScaled = false;  // see ArithHalfScaled
  using Replay = ArithF32Round;
  static constexpr bool kRangeReplays = false;  // a path outside the guard is replayed (else: the launch is re-run)
  static constexpr bool kIeee = false;
  uint32_t d, half_m1, keep;
  uint32_t d64;
  uint64_t half_m1_64, keep64;
  float split;     // 2^d + 1: Veltkamp's splitter
  double split64;  // 2^d64 + 1
#if defined(LPMC_PAIR) && !defined(LPMC_F32R_INT)
  static constexpr bool kPair = true;  // mul2: packed product + packed Veltkamp split
#else
  static constexpr bool kPair = false;
#endif
  static constexpr bool kPow2 = true;  // native range guard: step_bar_pw is exact
  uint64_t n0, n1, p1, split2;
  __device__ explicit ArithF32Round(const LevelArgs& A)
      : n0(A.f2_neg0), n1(A.f2_neg1), p1(A.f2_neg1 & 0x7fffffff7fffffffull) {
    d = 23u - static_cast<uint32_t>(A.mantissa_bits);
    half_m1 = (1u << (d - 1)) - 1u;
    keep = ~((1u << d) - 1u);
    split = static_cast<float>((1u << d) + 1u);  // exact: d <= 22
    d64 = 52u - static_cast<uint32_t>(A.mantissa_bits);
    half_m1_64 = (1ull << (d64 - 1)) - 1ull;
    keep64 = ~((1ull << d64) - 1ull);
    split64 = static_cast<double>((1ull << d64) + 1ull);  // exact: d64 <= 51
    split2 = pack2(split, split);
  }
  __device__ T c(double dd, uint16_t) const { return static_cast<float>(dd); }
  __device__ T zero() const { return 0.0f; }
  // RNE of a normal fp32 value to 24 - d = m + 1 significant bits.  Veltkamp's
  // split c = x (2^d + 1), x - (c - x)... as c - (c - x) in round-to-nearest-
  // even fp32 is that rounding, ties to even included, for m + 1 >= 2 bits
  // and no overflow/underflow (the native range guard):
  // three FMA-pipe operations instead of four integer ones (tests/
  // test_veltkamp.py checks it against the integer RNE, ties included).
  __device__ T rn(T x) const {
#ifdef LPMC_F32R_INT
    return rne32(x, d, half_m1, keep);
#else
    const float c = __fmul_rn(x, split);
    return __fsub_rn(c, __fsub_rn(c, x));
#endif
  }
  __device__ T mul(T a, T b) const { return rn(__fmul_rn(a, b)); }
  __device__ T add(T a, T b) const { return rn(__fadd_rn(a, b)); }
  __device__ T sub(T a, T b) const { return rn(__fsub_rn(a, b)); }
  // rn of both halves: c = x s, c - (c - x) as packed FFMA2s (see ffma2)
  __device__ uint64_t rn2(uint64_t x) const {
    const uint64_t c = ffma2(x, split2, n0);
    return ffma2(ffma2(x, n1, c), n1, c);
  }
  __device__ uint64_t mul2(uint64_t a, uint64_t b) const { return rn2(ffma2(a, b, n0)); }
  __device__ uint64_t add2(uint64_t a, uint64_t b) const { return rn2(ffma2(a, p1, b)); }
  __device__ uint64_t sub2(uint64_t a, uint64_t b) const { return rn2(ffma2(b, n1, a)); }
  __device__ float one() const { return lo2(p1); }
  // R(z) from the full binary64 value: one rounding (softfloat.hpp:69)
  // (Veltkamp in binary64: Gaussians are 0 or normal and |z| < 40)
  __device__ T lift(const double (&z)[1]) const {
#ifdef LPMC_F32R_INT
    return __double2float_rn(rne64(z[0], d64, half_m1_64, keep64));
#else
    const double c = __dmul_rn(z[0], split64);
    return __double2float_rn(__dsub_rn(c, __dsub_rn(c, z[0])));
#endif
  }
  __device__ double get(T x, int) const { return static_cast<double>(x); }
  __device__ uint32_t bad(T x) const { return nonfinite32(x) ? 1u : 0u; }
};

struct ArithF64Round {  // any m < 52: binary64 op, then integer RNE (exact emulation)
  using T = double;
  using Range = RangeNone;
  static constexpr int NP = 1;
  static constexpr bool kScaled = false;  // see ArithHalfScaled
  using Replay = ArithF64Round;
  static constexpr bool kRangeReplays = false;  // a path outside the guard is replayed (else: the launch is re-run)
  static constexpr bool kIeee = false;
  static constexpr bool kPair = false;
  static constexpr bool kPow2 = false;
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
};

struct ArithHalf2 {  // native IEEE binary16, two paths per thread
  using T = __half2;
  using Range = RangeNone;
  static constexpr int NP = 2;
  static constexpr bool kScaled = false;  // see ArithHalfScaled
  using Replay = ArithHalf2;
  static constexpr bool kRangeReplays = false;  // a path outside the guard is replayed (else: the launch is re-run)
  static constexpr bool kIeee = true;
  static constexpr bool kPair = false;  // already two paths per half2 op
  static constexpr bool kPow2 = false;
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
};

// The reference's m = 7 (bf16: RNE to 8 significant bits, unbounded exponent)
// on NATIVE bfloat16 arithmetic: bfloat16 has fp32's exponent range, so the
// native fp32 policies' range guard ([2^-32, 2^33) states, host-bounded
// constants: no intermediate is subnormal or overflows) makes one
// HMUL2.BF16 / HADD2.BF16 per reference operation exact -- no scaling, unlike
// binary16 below -- instead of an fp32 operation plus a three-operation
// Veltkamp split.  Production launches in the fast mode; dumps, glibc mode
// and the warp-per-path schedule run the fp32-carried emulation
// (ArithF32Round), which also replays suspect paths; a launch that leaves the
// range is re-run in the binary64 emulation like the other native policies.
struct RangeBf16 {
  static constexpr uint32_t kLo = 0x2f80u, kHi = 0x5000u;  // 2^-32, 2^33 (top halves of fp32)
  uint32_t worst = 0u;
  __device__ void track(__nv_bfloat16 x) {
    worst = max(worst, (static_cast<uint32_t>(__bfloat16_as_ushort(x)) & 0x7fffu) - kLo);
  }
  __device__ bool bad() const { return worst >= kHi - kLo; }
};

struct ArithBf16 {
  using T = __nv_bfloat16;
  using Range = RangeBf16;
  using Replay = ArithF32Round;
  static constexpr int NP = 1;
  static constexpr bool kScaled = false;
  static constexpr bool kRangeReplays = false;  // a path outside the guard is replayed (else: the launch is re-run)
  static constexpr bool kIeee = false;
  static constexpr bool kPair = false;
  static constexpr bool kPow2 = true;  // native range guard: step_bar_pw is exact
  double split64;  // 2^45 + 1: Veltkamp's splitter for R(z) in binary64
  __device__ explicit ArithBf16(const LevelArgs&) : split64(35184372088833.0) {}
  // constants are already rounded to 8 bits on the host: exact conversions
  __device__ T c(double d, uint16_t) const { return __float2bfloat16_rn(static_cast<float>(d)); }
  __device__ T zero() const { return __ushort_as_bfloat16(0u); }
  __device__ T mul(T a, T b) const { return __hmul_rn(a, b); }
  __device__ T add(T a, T b) const { return __hadd_rn(a, b); }
  __device__ T sub(T a, T b) const { return __hsub_rn(a, b); }
  // R(z) from the full binary64 value: one rounding (softfloat.hpp:69) by
  // Veltkamp's split in binary64, then exact conversions
  __device__ T lift(const double (&z)[1]) const {
    const double c = __dmul_rn(z[0], split64);
    return __float2bfloat16_rn(__double2float_rn(__dsub_rn(c, __dsub_rn(c, z[0]))));
  }
  __device__ double get(T x, int) const { return static_cast<double>(__bfloat162float(x)); }
  __device__ uint32_t bad(T x) const {
    return (__bfloat16_as_ushort(x) & 0x7f80u) == 0x7f80u ? 1u : 0u;
  }
};

// The reference's m = 10 emulation (RNE to 11 significant bits, unbounded
// exponent; softfloat.hpp:69-111) on NATIVE binary16 arithmetic: one HMUL2 /
// HFMA2 per reference operation instead of an fp32 operation plus a
// three-operation Veltkamp split.  binary16's exponent range is far narrower
// than the values of a step (mu x dt ~ 1e-5 is subnormal), so every quantity
// is carried with a static power-of-two scale chosen on the host (LevelArgs::
// hs_*; scaling by a power of two commutes with rounding while the scaled
// value is a normal binary16 number).  With mu_l = mu_m 2^e_mu, sigma_l =
// sg_m 2^e_sg, sqrt_dt_l = sdt_m 2^e_sdt (mantissas in [1, 2): exact binary16),
// dt_l = 2^e_dt, the approximate Gaussian delivered as zs = R(z) 2^kz (the
// table's c0, c1 are pre-scaled at staging; the conversion F2F.F16.F64 is the
// reference's one rounding), e_d = e_sg + e_sdt - kz:
//   a = R(x mu_m)                          = R(mu_l x) 2^-e_mu
//   c = R(R(x sg_m) sdt_m)                 = R(R(sigma_l x) sqrt_dt_l) 2^-(e_sg+e_sdt)
//   e = R(c zs)                            = diff 2^-e_d
//   i = fma(a, P1, e),  P1 = 2^(e_mu+e_dt-e_d) = 4   (kz is chosen for this)
//                                          = R(drift + diff) 2^-e_d
//   x' = fma(i, P2, x), P2 = 2^e_d         = R(x + inc)
// and the coarse step with dW 2^(kz-e_sdt) = R(R(sdt_m zs0) + R(sdt_m zs1)),
// P1c = 8 (2 dt).  Exactness ("native binary16"):
//  * |x| in [2^-4, 2^14) before and after every step (RangeH, per update)
//    -- then a, R(x sg_m), c are normal;
//  * a scaled Gaussian below 2^-14 is subnormal and carries fewer than 11
//    bits.  In the fine step that only perturbs a subnormal e (next item).
//    In the coarse dW = R(w0 + w1), w = R(sdt_m zs), it is absorbed when the
//    other term is at least 2^-2 (|w| < 2^-13.5 is below half an ulp of it),
//    so a harmful pair has |w0 w1| < 2^-15.5; RangeH::trackw flags the coarse
//    steps with |R(w0 w1)| < 2^-15 (probability ~2e-9 per step; a first
//    version that flagged every pair below 2^-2 replayed 5e-4 of the level-12
//    paths, 14 % of the batches, and gave the native gain back).  dW itself,
//    a sum of multiples of 2^-24, is exact whenever it is below 2^-14;
//  * e may be subnormal (fewer than 11 bits): then |e| < 2^-14 <= 2^-10 |x|,
//    below half an ulp of a P1 (>= 4 |x| 2^-12), so i = a P1 whatever e's
//    last bits are; i itself is a sum of multiples of 2^-24, exact whenever
//    it is below 2^-14; x' = fma(i, P2, x) rounds the exact x + inc once.
// Overflow gives inf, which is absorbing and caught at the end of the path.
// A path that fails any of these is replayed in the fp32-carried emulation
// (Replay = ArithF32Round, bitwise the reference), so the result never
// depends on the guard -- only the speed does.  With or without Kahan
// compensation (ArithHalfScaled::kahan), dyadic-linear tables or none.
// State of ArithHalfScaled: X = (x_fine, x_coarse) in one binary16 pair; the
// guard tracks both lanes at once (packed min / max of |X|) and, per coarse
// step, the larger of the two scaled increments.  NaN is invisible to min / max and
// inf to nothing: non-finite states are absorbing and caught at the end of
// the path (bad()).
struct RangeH {
  __half2 lo = __halves2half2(__ushort_as_half(0x7bffu), __ushort_as_half(0x7bffu));
  __half2 hi = __halves2half2(__ushort_as_half(0u), __ushort_as_half(0u));
  __half wmin = __ushort_as_half(0x7bffu);  // min over coarse steps of |R(w0 w1)|
  __device__ void track(__half2 X) {
    const __half2 a = __habs2(X);
    lo = __hmin2(lo, a);
    hi = __hmax2(hi, a);
  }
  __device__ void trackw(__half2 w) {
    wmin = __hmin(wmin, __habs(__hmul_rn(__low2half(w), __high2half(w))));
  }
  __device__ void track(float) {}
  __device__ void track(double) {}
  // |x| in [2^-4, 2^14) on both lanes; every coarse step had |w0 w1| >= 2^-15
  __device__ bool bad() const {
    const uint32_t l = *reinterpret_cast<const uint32_t*>(&lo);
    const uint32_t h = *reinterpret_cast<const uint32_t*>(&hi);
    constexpr uint32_t kLo = (15u - 4u) << 10, kHi = (15u + 14u) << 10;
    return (l & 0xffffu) < kLo || (l >> 16) < kLo || (h & 0xffffu) >= kHi || (h >> 16) >= kHi ||
           __half_as_ushort(wmin) < 0x0200u;  // 2^-15 (a binary16 subnormal: 512 2^-24)
  }
};

struct ArithHalfScaled {
  using T = __half2;  // states: (fine, coarse); Gaussians: low lane
  using Range = RangeH;
  using Replay = ArithF32Round;
  static constexpr int NP = 1;
  static constexpr bool kScaled = true;
  static constexpr bool kRangeReplays = true;  // a path outside the guard is replayed (else: the launch is re-run)
  static constexpr bool kIeee = false;
  static constexpr bool kPair = false;
  static constexpr bool kPow2 = true;  // PW instances fold the carrier legs (step_hat_pw)
  __half2 musg, mu2, sg2, sdt2, sdt_one, p1_2, p1_p1c, p2_2, q1_2, q2_2;
  double zscale;
  __device__ explicit ArithHalfScaled(const LevelArgs& A) : zscale(A.hs_zscale) {
    const __half q1 = __ushort_as_half(A.hs_q1), q2 = __ushort_as_half(A.hs_q2);
    q1_2 = __halves2half2(q1, q1);
    q2_2 = __halves2half2(q2, q2);
    const __half mu = __ushort_as_half(A.hs_mu), sg = __ushort_as_half(A.hs_sigma);
    const __half sd = __ushort_as_half(A.hs_sdt), one = __ushort_as_half(0x3c00u);
    const __half p1 = __ushort_as_half(A.hs_p1), p1c = __ushort_as_half(A.hs_p1c);
    const __half p2 = __ushort_as_half(A.hs_p2);
    musg = __halves2half2(mu, sg);
    mu2 = __halves2half2(mu, mu);
    sg2 = __halves2half2(sg, sg);
    sdt2 = __halves2half2(sd, sd);
    sdt_one = __halves2half2(sd, one);
    p1_2 = __halves2half2(p1, p1);
    p1_p1c = __halves2half2(p1, p1c);
    p2_2 = __halves2half2(p2, p2);
  }
  __device__ T c(double, uint16_t bits) const {  // x0 (exact): both legs start there
    const __half h = __ushort_as_half(bits);
    return __halves2half2(h, h);
  }
  __device__ T zero() const { return __halves2half2(__ushort_as_half(0u), __ushort_as_half(0u)); }
  // z arrives pre-scaled by 2^kz from the scaled table copy; exact Gaussians
  // (no table) are scaled here
  __device__ T lift(const double (&z)[1]) const {
    const __half h = __double2half(z[0]);
    return __halves2half2(h, h);
  }
  __device__ T lift_exact(const double (&z)[1]) const {
    const __half h = __double2half(__dmul_rn(z[0], zscale));
    return __halves2half2(h, h);
  }
  __device__ double get(T x, int lane) const {
    return static_cast<double>(__half2float(lane == 0 ? __low2half(x) : __high2half(x)));
  }
  __device__ uint32_t bad(T x) const {
    const uint32_t b = *reinterpret_cast<const uint32_t*>(&x);
    return ((b & 0x7c00u) == 0x7c00u || (b & 0x7c000000u) == 0x7c000000u) ? 1u : 0u;
  }
  // kahan_accumulate (sde.hpp:85-92) on scaled values: the increment is
  // inc = i P2 and the compensation is carried as cs = comp / P2, so
  //   ys = R(i - cs)                   = R(inc - comp) / P2
  //   s  = fma(ys, P2, x)              = R(sum + y)
  //   t  = R(s - x)                      (a multiple of 2^-14: normal or 0)
  //   cs = fma(t Q1, Q2, -ys), Q1 Q2 = 1 / P2   = R(R(s - x) - y) / P2
  // (t Q1 is an exact scaling; 1/P2 may exceed binary16's range, hence two
  // factors).  Differences below 2^-14 are multiples of 2^-24 and exact, in
  // the reference as well (they have at most 10 bits).  Returns s.
  __device__ T kahan(T x, T i, T& cs) const {
    const T ys = __hsub2_rn(i, cs);
    const T s = __hfma2(ys, p2_2, x);
    const T t = __hsub2_rn(s, x);
    cs = __hfma2(__hmul2_rn(t, q1_2), q2_2, __hneg2(ys));
    return s;
  }
  // em_step / em_step_kahan (sde.hpp:60-68, :95-104) of the fine leg (lane 0
  // of X, lane 0 of the compensation pair); returns the new x_fine in both
  // lanes (and, with Kahan, the new compensation in both lanes of csf)
  template <bool KAHAN>
  __device__ T fine_value(T X, T zs, T& csf) const {
    const T xf = __low2half2(X);
    const T ab = __hmul2_rn(xf, musg);                      // (R(x mu_m), R(x sg_m))
    const T cc = __hmul2_rn(__high2half2(ab), sdt2);        // R(R(x sg_m) sdt_m)
    const T e = __hmul2_rn(cc, __low2half2(zs));
    const T i = __hfma2(__low2half2(ab), p1_2, e);
    if constexpr (KAHAN) {
      csf = __low2half2(csf);
      return kahan(xf, i, csf);
    } else {
      return __hfma2(i, p2_2, xf);
    }
  }
  // one fine step alone (level 0, the two-way sampler): lane 1 is kept
  template <bool KAHAN>
  __device__ void fine(T& X, T& CS, T zs, Range& r) const {
    T csf = CS;
    const T xf1 = fine_value<KAHAN>(X, zs, csf);
    X = __halves2half2(__low2half(xf1), __high2half(X));
    if constexpr (KAHAN) CS = __halves2half2(__low2half(csf), __high2half(CS));
    r.track(X);
  }
  // fine step n (zs0), then fine step n + 1 (zs1) and the coarse step as one
  // pair: em_step and em_step_dw (sde.hpp:60-79) with dW = sqrt_dt z0 +
  // sqrt_dt z1 (sde.hpp:261-264); the coarse lane multiplies by an exact 1
  // where the fine lane takes sdt_m
  template <bool KAHAN>
  __device__ void coarse_step(T& X, T& CS, T zs0, T zs1, Range& r) const {
    const T Z = __halves2half2(__low2half(zs0), __low2half(zs1));
    T csf = CS;
    const T xf1 = fine_value<KAHAN>(X, zs0, csf);
    r.track(xf1);
    const T X1 = __halves2half2(__low2half(xf1), __high2half(X));
    if constexpr (KAHAN) CS = __halves2half2(__low2half(csf), __high2half(CS));
    const T a = __hmul2_rn(X1, mu2);
    const T b = __hmul2_rn(X1, sg2);
    const T w = __hmul2_rn(Z, sdt2);                                   // (w0, w1)
    r.trackw(w);
    const T dw = __hadd2_rn(__low2half2(w), __high2half2(w));          // both lanes
    const T cc = __hmul2_rn(b, sdt_one);                               // (R(b sdt_m), b)
    const T e = __hmul2_rn(cc, __halves2half2(__high2half(Z), __low2half(dw)));  // (zs1, dW)
    const T i = __hfma2(a, p1_p1c, e);
    if constexpr (KAHAN) {
      X = kahan(X1, i, CS);
    } else {
      X = __hfma2(i, p2_2, X1);
    }
    r.track(X);
  }
  // unused generic interface (step_bar is never instantiated for this policy)
  __device__ T mul(T a, T b) const { return __hmul2_rn(a, b); }
  __device__ T add(T a, T b) const { return __hadd2_rn(a, b); }
  __device__ T sub(T a, T b) const { return __hsub2_rn(a, b); }
};

// --------------------------------------------------------- block tree ------
// Fixed reduction of a 256-path batch: slot s = threadIdx.x + p*blockDim.x;
// per 32-slot group an xor butterfly, then an xor butterfly over the 8 group
// sums.  Pass 1 gives the mean, pass 2 the central power sums.  Restated
// bit for bit in oracle/lpmc_oracle.c (batch_acc).
__device__ __forceinline__ double warp_sum(double x, int first) {
  for (int k = first; k >= 1; k >>= 1) x = __dadd_rn(x, __shfl_xor_sync(0xffffffffu, x, k));
  return x;
}

// GROUPS > 1 (the persistent level kernel): GROUPS independent batches per
// CTA, one per group of kBatch / NP threads; `tid` is the thread's index in
// its group, `grp` the group; the groups synchronise on their own named
// barriers (1 + grp) and use their own scratch rows.
template <int GROUPS>
__device__ __forceinline__ void group_sync(int grp) {
  if constexpr (GROUPS == 1) {
    __syncthreads();
  } else {
    asm volatile("bar.sync %0, %1;" ::"r"(1 + grp), "r"(static_cast<int>(blockDim.x) / GROUPS) : "memory");
  }
}

template <int NP, int GROUPS = 1>
__device__ void batch_moments(const double (&vh)[NP], const double (&vb)[NP],
                              const bool (&valid)[NP], int count, double* out15,
                              int tid = static_cast<int>(threadIdx.x), int grp = 0) {
  __shared__ double s_grp_all[GROUPS][9][8];
  __shared__ double s_mean_all[GROUPS][3];
  double(&s_grp)[9][8] = s_grp_all[grp];
  double(&s_mean)[3] = s_mean_all[grp];
  constexpr int kWarps = kBatch / NP / 32;
  const int lane = tid & 31;
  const int warp = tid >> 5;
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
      LPMC_DCHECK(warp + p * kWarps < 8);
      if (lane == 0) s_grp[f][warp + p * kWarps] = s;
    }
  group_sync<GROUPS>(grp);
  if (warp == 0) {
#pragma unroll
    for (int f = 0; f < 3; ++f) {
      const double g = warp_sum(lane < 8 ? s_grp[f][lane] : 0.0, 4);
      if (lane == 0) s_mean[f] = __ddiv_rn(g, static_cast<double>(count));
    }
  }
  group_sync<GROUPS>(grp);
  const double mean[3] = {s_mean[0], s_mean[1], s_mean[2]};
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
  group_sync<GROUPS>(grp);
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
  // persistent callers: the next batch's first pass rewrites s_grp rows 0..2
  // only after its own first barrier, which every thread of the group reaches
  // after reading s_mean and the final rows above -- except warp 0's reads of
  // rows 0..8 just above, hence one more barrier.
  if constexpr (GROUPS > 1) group_sync<GROUPS>(grp);
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

}  // namespace dev
}  // namespace lpmc_b200
