// Device math for the exact Gaussian (gaussian.hpp:26-65: Acklam's rational
// + one Newton step on libm's erfc), restated for the sm_100a issue budget.
//
// Round 2: the default transform is ONE TABLE LOOKUP -- phi_inv_direct: a
// degree-8 polynomial of Phi^-1 on 16 sub-intervals per binade of
// v = min(u, 1 - u) (tools/fit_direct.py, lpmc_direct_coef.h), 10 FP64
// operations per draw, 0.42 eps (v/pdf + |z|) from the true value
// (DirectTab: flat; LaneDirectTab: eight lane-private copies, conflict-free
// gathers in the persistent level kernel).  Draws below the table (v < 2^-15,
// 6e-5 of them) take round 1's transform, which the rest of this header
// describes, out of line (phi_inv_lower_tail); -DLPMC_HALLEY_Z rebuilds it
// everywhere (A/B).
//
// Why not libdevice: its erfc/exp keep their polynomial coefficients as
// 64-bit literals, which ptxas rematerialises through uniform moves on every
// loop iteration (136 UMOV per warp-step, 24% of all issue slots in the v0
// kernel, profiles/r01_v0_summary.md), and their range branches diverge.
// Here every coefficient is a constant-bank operand (__constant__) or a
// shared-memory load.
//
// Round 1's transform ("below the table"):
//  * The reference refines Acklam's x0 (1.15e-9) by one Newton step.  Here
//    x0 comes from an fp32 polynomial in log2(v (1 - v)) (~4e-7 relative,
//    tools/fit_x0f.py) and one Halley step x0 - r (1 - x0 r / 2),
//    r = (Phi(x0) - v) / pdf(x0), whose error K e0^3 stays below 1% of an ulp
//    of Z: the same root, to the same last-ulp noise of the erfc evaluation.
//  * r needs Phi(x0) to ~1 ulp of v, and 1/pdf to ~1e-12 only.  Phi(x0) =
//    erfc(t)/2, t = -x0/sqrt(2), with erfc(t) = 2^k p(r) G(t): t^2 split
//    exactly by FMA, exp(-t^2) = 2^k p(r) from a 64-entry 2^(j/64) hi/lo
//    table and a degree-4 expm1 polynomial, and G = erfcx by 104 degree-8
//    piecewise polynomials on intervals of 1/16 with the constant term as
//    hi + lo (tools/fit_math.py).  1/pdf is sqrt(2 pi) 2^-k / p(r): the same
//    exponential, no second exp, no division.  Table indices come from the
//    low words of shifted FMAs (no F2I/I2F conversions).
//  * t >= kDevTMax (6.5: u < 1e-20, never drawn by the sampler) takes a
//    libdevice slow path out of line.
//  * -DLPMC_X0_ACKLAM restores Acklam's binary64 x0 + Newton (A/B only,
//    tools/gpu_ab_x0.sh).
//
// All functions are __host__ __device__ so the host hooks (lpmc_erfc_core,
// lpmc_phi_inv_direct_core; tests/test_math_host.py) can check them on the
// CPU against mpmath; they use only IEEE fma/mul/add and integer bit
// operations, hence are bitwise the same there.
#pragma once

#include <cstdint>
#include <cstring>
#include <cmath>

#include "lpmc_glibc_coef.h"
#if defined(LPMC_ERFCX_W8)
#include "lpmc_math_coef_w8.h"  // erfcx on 1/8 intervals, degree 9 (A/B)
#elif defined(LPMC_ERFCX_W4)
#include "lpmc_math_coef_w4.h"  // erfcx on 1/4 intervals, degree 11 (A/B)
#else
#include "lpmc_math_coef.h"
#endif
#include "lpmc_x0f_coef.h"
#include "lpmc_direct_coef.h"

#ifdef __CUDACC__
#define LPMC_HD __host__ __device__ __forceinline__
#else
#define LPMC_HD inline
#endif

// -DLPMC_DEVICE_CHECKS (test builds only -- compute-sanitizer is not
// available on the B200 pool): bounds checks on every table, shared-memory
// and output index; a failed check prints the condition and traps the kernel,
// so the calling test fails loudly (tools/gpu_checks.sh).
#if defined(LPMC_DEVICE_CHECKS) && defined(__CUDA_ARCH__)
#define LPMC_DCHECK(c)                                                                 \
  do {                                                                                 \
    if (!(c)) {                                                                        \
      printf("LPMC_DCHECK failed %s:%d: %s (block %d thread %d)\n", __FILE__, __LINE__, #c, \
             static_cast<int>(blockIdx.x), static_cast<int>(threadIdx.x));             \
      __trap();                                                                        \
    }                                                                                  \
  } while (0)
#else
#define LPMC_DCHECK(c) \
  do {                 \
  } while (0)
#endif

namespace lpmc_b200 {
namespace math {

LPMC_HD double fmad(double a, double b, double c) {
#ifdef __CUDA_ARCH__
  return __fma_rn(a, b, c);
#else
  return std::fma(a, b, c);
#endif
}

LPMC_HD uint64_t bits(double x) {
#ifdef __CUDA_ARCH__
  return static_cast<uint64_t>(__double_as_longlong(x));
#else
  uint64_t b;
  std::memcpy(&b, &x, 8);
  return b;
#endif
}

LPMC_HD double from_bits(uint64_t b) {
#ifdef __CUDA_ARCH__
  return __longlong_as_double(static_cast<long long>(b));
#else
  double x;
  std::memcpy(&x, &b, 8);
  return x;
#endif
}

// neg ? -x : x as one XOR on the high word (a select of the sign mask and a
// LOP3 instead of a DADD and two selects).
LPMC_HD double flip_sign(double x, bool neg) {
  return from_bits(bits(x) ^ (neg ? 0x8000000000000000ull : 0ull));
}
// x with the high word XORed by `mask` (0 or 0x80000000, computed once per
// draw and shared by both transforms)
LPMC_HD double flip_sign_mask(double x, uint32_t mask) {
  return from_bits(bits(x) ^ (static_cast<uint64_t>(mask) << 32));
}

// 1/d to ~1 ulp: hardware seed (MUFU.RCP64H) + two Newton steps.
LPMC_HD double rcp_refined(double d) {
#ifdef __CUDA_ARCH__
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
  double e = fmad(-d, r, 1.0);
  r = fmad(r, e, r);
  e = fmad(-d, r, 1.0);
  return fmad(r, e, r);
#else
  return 1.0 / d;
#endif
}

// 1/d to ~2^-44: seed + one Newton step (for the Newton correction only).
LPMC_HD double rcp_coarse(double d) {
#ifdef __CUDA_ARCH__
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
  const double e = fmad(-d, r, 1.0);
  return fmad(r, e, r);
#else
  return 1.0 / d;
#endif
}

// sqrt(y), y > 0, to ~2^-44 (Acklam tail only).
LPMC_HD double sqrt_coarse(double y) {
#ifdef __CUDA_ARCH__
  double r;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(y));
  const double h = 0.5 * y;
  r = r * fmad(-h * r, r, 1.5);
  return y * r;
#else
  return std::sqrt(y);
#endif
}

// Scalar coefficients, one constant block.  On the device it is deliberately
// NOT statically initialised: ptxas constant-folds initialised __constant__
// data back into 64-bit immediates (uniform-register moves again); uploaded
// at context creation (upload_math_constants), uses become constant loads.
enum : int {
  kOffAckA = 0,                     // Acklam central numerator a0..a5   (gaussian.hpp:28-30)
  kOffAckB = 6,                     // Acklam central denominator b0..b4 (:31-33)
  kOffAckC = 11,                    // Acklam tail numerator c0..c5      (:34-36)
  kOffAckD = 17,                    // Acklam tail denominator d0..d3    (:37-38)
  kOffLogS = 21,                    // 2/(2i+1), i = 0..6: log(m) = s sum s^2i 2/(2i+1)
  kOffExpm1 = 28,                   // expm1(r)/r, LPMC_EXPM1_DEG + 1 terms
  kOffMisc = kOffExpm1 + LPMC_EXPM1_DEG + 1,
  kLog2eN = kOffMisc + 0,           // 64 log2(e)
  kLn2HiN = kOffMisc + 1,           // ln2/64 split: 32 significant bits (k * hi exact)
  kLn2LoN = kOffMisc + 2,
  kLn2 = kOffMisc + 3,
  kInvSqrt2 = kOffMisc + 4,         // gaussian.hpp:15 literal
  kSqrt2Pi = kOffMisc + 5,
  kTailU = kOffMisc + 6,            // Acklam's u_low = 0.02425 (gaussian.hpp:38)
  kSpare = kOffMisc + 7,
  kMathCount = kOffMisc + 8
};

static const double kMathHost[kMathCount] = {
    -3.969683028665376e+01, 2.209460984245205e+02, -2.759285104469687e+02,
    1.383577518672690e+02, -3.066479806614716e+01, 2.506628277459239e+00,
    -5.447609879822406e+01, 1.615858368580409e+02, -1.556989798598866e+02,
    6.680131188771972e+01, -1.328068155288572e+01,
    -7.784894002430293e-03, -3.223964580411365e-01, -2.400758277161838e+00,
    -2.549732539343734e+00, 4.374664141464968e+00, 2.938163982698783e+00,
    7.784695709041462e-03, 3.224671290700398e-01, 2.445134137142996e+00,
    3.754408661907416e+00,
    2.0, 2.0 / 3.0, 2.0 / 5.0, 2.0 / 7.0, 2.0 / 9.0, 2.0 / 11.0, 2.0 / 13.0,
    LPMC_EXPM1_COEF_LIST,
    92.332482616893657 / 64.0 * LPMC_EXP_N,   // N log2(e) (power-of-two scalings: exact)
    6.93147180369123816490e-01 / LPMC_EXP_N,  // exact scaling of the 32-bit ln2 head
    1.90821492927058770002e-10 / LPMC_EXP_N,
    6.93147180559945309417e-01, 0.7071067811865475244, 2.5066282746310002, 0.02425, 0.0};

constexpr int kErfcxRow = LPMC_ERFCX_ROW;
constexpr int kErfcxN = LPMC_ERFCX_INTERVALS;
constexpr int kErfcxWords = kErfcxRow * kErfcxN;
constexpr int kExpN = LPMC_EXP_N;
constexpr int kExpWords = 2 * kExpN;
constexpr int kExpShift = kExpN == 64 ? 6 : kExpN == 32 ? 5 : kExpN == 16 ? 4 : 3;
static_assert(1 << kExpShift == kExpN, "exp table size must be 8, 16, 32 or 64");
constexpr int kGlibcOff = kErfcxWords + kExpWords;  // glibc exp and log tables (lpmc_glibc.cuh)
constexpr int kGlibcWords = 512;
constexpr int kMathTableWords = kGlibcOff + kGlibcWords;  // one shared-memory block
constexpr double kFastTMax = 6.5;  // the erfcx intervals cover [0, 6.5) (host core)

// The direct table of the fast exact Gaussian (tools/fit_direct.py):
// Phi^-1 on [2^-(B+1), 1/2] as degree-8 polynomials on 16 sub-intervals per
// binade, the record index read off v's high word.
constexpr int kDirectRow = LPMC_DIRECT_ROW;
constexpr int kDirectN = LPMC_DIRECT_N;
constexpr int kDirectWords = kDirectRow * kDirectN;
constexpr int kDirectShift = 20 - LPMC_DIRECT_S;  // high-word bits below the index
constexpr uint32_t kDirectBase = static_cast<uint32_t>(1023 - (LPMC_DIRECT_B + 1)) << LPMC_DIRECT_S;
static_assert(LPMC_DIRECT_DEG == 8 && LPMC_DIRECT_ROW == 10, "phi_inv_direct reads c8..c1, c0_lo, c0_hi as five quads");

// erfcx records, the 2^(j/64) hi/lo pairs, the glibc exp and log tables (host copy)
alignas(16) static const double kDirectHost[kDirectWords] = {LPMC_DIRECT_COEF_LIST};
static const double kMathTableHost[kMathTableWords] = {LPMC_ERFCX_COEF_LIST, LPMC_EXP_TAB_LIST,
                                                       LPMC_GLIBC_EXP_TAB, LPMC_GLIBC_LOG_TAB};

#ifdef __CUDACC__
// TU-local (static): every kernel translation unit has its own copy and
// uploads it in its configure function (upload_math_constants).
static __constant__ double kMath[kMathCount];
static __device__ __align__(16) const double kMathTable[kMathTableWords] = {
    LPMC_ERFCX_COEF_LIST, LPMC_EXP_TAB_LIST, LPMC_GLIBC_EXP_TAB, LPMC_GLIBC_LOG_TAB};

static __device__ __align__(16) const double kDirectTable[kDirectWords] = {LPMC_DIRECT_COEF_LIST};

static inline cudaError_t upload_math_constants() {
  return cudaMemcpyToSymbol(kMath, kMathHost, sizeof(kMathHost));
}
#endif

#ifdef __CUDA_ARCH__
#define LPMC_K(i) kMath[i]
#else
#define LPMC_K(i) kMathHost[i]
#endif

// two adjacent doubles of a 16-byte aligned table (one 128-bit load)
struct D2 {
  double a, b;
};
LPMC_HD D2 load2(const double* p) {
#ifdef __CUDA_ARCH__
  const double2 v = *reinterpret_cast<const double2*>(p);
  return D2{v.x, v.y};
#else
  return D2{p[0], p[1]};
#endif
}

// Table layouts of the erfcx records and the 2^(j/64) pairs.
//  * FlatTab: the records one after another (host, the erfc-core diagnostic
//    and the small kernels: inverse-CDF diagnostics, step-error probe,
//    density histogram).
//  * LaneTab (device, the level and warp-per-path kernels): eight
//    lane-private copies, transposed so that quad q of record j of copy c
//    sits at 16-byte index (j Q + q) 8 + c (Q quads per record) and every
//    lane reads copy c = lane % 8.  The eight lanes of each quarter-warp
//    phase of a 128-bit shared load then hit eight different bank quads
//    whatever records they gather: conflict-free by construction, with no
//    extra instruction (the copy offset is hoisted into the per-thread base
//    pointer; the record stride and the quad offsets are immediates).  Only
//    the records for t < 3 are staged (99.998 % of the sampler's draws); a
//    draw with t >= 3 takes the out-of-line libdevice path that serves
//    t >= 6.5 with the flat layout (newton_fast's `slow`).  kDevTMax is one
//    value for every kernel of a build (3 with -DLPMC_LANE_TABLES, else 6.5),
//    so all kernels compute the same Z.
struct FlatTab {
  const double* t;
  static constexpr int kRec = kErfcxRow;  // doubles between records
  static constexpr int kStep = 1;         // in-record offset multiplier
  static constexpr int kExpStride = 2;    // doubles between exp entries
  static constexpr int kNRec = kErfcxN;
  LPMC_HD const double* erfcx() const { return t; }
  LPMC_HD const double* expt() const { return t + kErfcxWords; }
};

constexpr int kLaneCopies = 8;
#ifdef LPMC_LANE_TABLES
constexpr double kDevTMax = 3.0;  // device fast path: erfcx records for t < 3
#else
constexpr double kDevTMax = kFastTMax;  // the flat table covers [0, 6.5)
#endif
constexpr int kHotRec = 3 * LPMC_ERFCX_PER_UNIT;  // lane layout: records for t < 3
static_assert(kErfcxRow % 2 == 0 && kHotRec <= kErfcxN, "lane layout needs whole quads");
constexpr int kLaneErfcxWords = kHotRec * kErfcxRow * kLaneCopies;
constexpr int kLaneWords = kLaneErfcxWords + kExpWords * kLaneCopies;

struct LaneTab {
  const double* e;  // copy c of the erfcx records (base + 2c)
  const double* x;  // copy c of the exp pairs
  static constexpr int kRec = kErfcxRow * kLaneCopies;
  static constexpr int kStep = kLaneCopies;
  static constexpr int kExpStride = 2 * kLaneCopies;
  static constexpr int kNRec = kHotRec;
  LPMC_HD const double* erfcx() const { return e; }
  LPMC_HD const double* expt() const { return x; }
};

// The direct table: flat (kDirectHost / kDirectTable or a shared-memory copy:
// the small kernels, the warp-per-path kernel, the host) or eight
// lane-private copies in shared memory (the persistent level kernel): quad q
// of record j of copy c at 16-byte index (5 j + q) 8 + c, every lane reads
// copy c = lane % 8, so the eight lanes of each quarter-warp phase of a
// 128-bit load hit eight different bank quads whatever records they gather
// -- conflict-free by construction, no extra instruction (the copy offset
// sits in the per-thread base pointer, record stride and quad offsets are
// immediates).  225 records x 80 B x 8 = 144 KB: one table per SM.
struct DirectTab {
  const double* t;
  static constexpr int kRec = kDirectRow;  // doubles between records
  static constexpr int kStep = 1;          // in-record offset multiplier
};
struct LaneDirectTab {
  const double* t;  // copy c (base + 2 c)
  uint32_t saddr;   // its shared-space address (device: loads without a generic pointer)
  static constexpr int kRec = kDirectRow * kLaneCopies;
  static constexpr int kStep = kLaneCopies;
};
// quad q (0..4) of record j
LPMC_HD D2 direct_quad(const DirectTab& tab, uint32_t j, int q) {
  return load2(tab.t + j * DirectTab::kRec + 2 * q);
}
LPMC_HD D2 direct_quad(const LaneDirectTab& tab, uint32_t j, int q) {
#ifdef __CUDA_ARCH__
  D2 r;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];"
               : "=d"(r.a), "=d"(r.b)
               : "r"(tab.saddr + j * (LaneDirectTab::kRec * 8u) + q * (LaneDirectTab::kStep * 16u)));
  return r;
#else
  return load2(tab.t + j * LaneDirectTab::kRec + 2 * q * LaneDirectTab::kStep);
#endif
}
constexpr int kLaneDirectWords = kDirectWords * kLaneCopies;
// source word of lane-layout word i: 16 doubles = 8 copies of one quad
LPMC_HD int lane_direct_source(int i) { return 2 * (i >> 4) + (i & 1); }

// -Phi^-1(v) = Phi^-1(1 - v) >= 0 for v in [2^-(B+1), 1/2] (v == 1/2: the
// all-zero record, +0 exactly, gaussian.hpp:62): the table holds the upper
// half, so the exact and the approximate transform (invcdf_approx.hpp:47-49)
// flip their signs on the same predicate, u < 1/2.  Record index = exponent and top S mantissa
// bits of v; t = v - midpoint is exact (both in one binade; the midpoint is
// v's bit pattern with the low mantissa bits replaced by 100...0).
// *tail: v below the table (probability 2^-B per draw); the value returned
// for such a lane comes from the zero record and is never used.
// Error: <= 0.42 eps (v/phi(z) + |z|) (tools/fit_direct.py --check): the
// final addition's half ulp; the interpolation error is ~1 % of it.
template <class V>
LPMC_HD double phi_inv_direct(double v, const V& tab, bool* tail) {
  const uint32_t hi = static_cast<uint32_t>(bits(v) >> 32);
  const uint32_t idx = (hi >> kDirectShift) - kDirectBase;
  *tail = idx >= static_cast<uint32_t>(kDirectN);  // below the table: idx wrapped
  const uint32_t j = idx < static_cast<uint32_t>(kDirectN - 1) ? idx : static_cast<uint32_t>(kDirectN - 1);
  LPMC_DCHECK(j < static_cast<uint32_t>(kDirectN));
  const uint32_t hc = (hi & ~((1u << kDirectShift) - 1u)) | (1u << (kDirectShift - 1));
  const double t = v - from_bits(static_cast<uint64_t>(hc) << 32);
  const D2 a = direct_quad(tab, j, 0), b = direct_quad(tab, j, 1), c = direct_quad(tab, j, 2);
  const D2 d = direct_quad(tab, j, 3);
  const D2 e = direct_quad(tab, j, 4);  // c0_lo, c0_hi
  double p = fmad(a.a, t, a.b);
  p = fmad(p, t, b.a);
  p = fmad(p, t, b.b);
  p = fmad(p, t, c.a);
  p = fmad(p, t, c.b);
  p = fmad(p, t, d.a);
  p = fmad(p, t, d.b);
  p = fmad(p, t, e.a);  // + c0_lo
  return p + e.b;       // + c0_hi
}

// source word of lane-layout word i (staging; host tests use it too)
LPMC_HD int lane_source(int i) {
  const int half = i & 1, quad = i >> 4;  // 16 doubles = 8 copies of one quad
  if (i < kLaneErfcxWords) return 2 * quad + half;
  return kErfcxWords + 2 * ((i - kLaneErfcxWords) >> 4) + half;
}

// exp(-(th + tl)) = 2^k p, p in [2^-1/2, 2^1/2], th in [0, 700]:
// kf = round(-64 th log2 e) = 64 k + j, r = -th - kf ln2/64 (exact head),
// p = 2^(j/64) (1 + r P(r)) with the table value as hi + lo.
struct ExpSplit {
  double p;
  int k;
};

template <class V>
LPMC_HD ExpSplit exp_neg(double th, double tl, const V& tab) {
  const double kShift = 6755399441055744.0;  // 1.5 * 2^52 (an encodable immediate)
  const double ks = fmad(-th, LPMC_K(kLog2eN), kShift);
  const double kd = ks - kShift;
  const int kf = static_cast<int>(static_cast<uint32_t>(bits(ks)));  // = (int)kd, no F2I
  double r = fmad(kd, -LPMC_K(kLn2HiN), -th);  // exact
  r = fmad(kd, -LPMC_K(kLn2LoN), r);
  r = r - tl;
  double q = LPMC_K(kOffExpm1 + LPMC_EXPM1_DEG);
#ifdef __CUDA_ARCH__
#pragma unroll
#endif
  for (int i = LPMC_EXPM1_DEG - 1; i >= 0; --i) q = fmad(q, r, LPMC_K(kOffExpm1 + i));
  q = q * r;  // expm1(r)
  const D2 t2 = load2(tab.expt() + V::kExpStride * (kf & (kExpN - 1)));
  const double p = t2.a + fmad(t2.a, q, t2.b);
  return ExpSplit{p, kf >> kExpShift};
}

// erfcx(t) for t in [0, 6.5) (FlatTab) or [0, 3) (LaneTab): interval record
// j (width 1/LPMC_ERFCX_PER_UNIT), highest power first.
template <class V>
LPMC_HD double erfcx_piecewise(double t, const V& tab) {
  constexpr int D = LPMC_ERFCX_DEG;
  constexpr double kPerUnit = LPMC_ERFCX_PER_UNIT;
  constexpr int S = V::kStep;
#ifdef __CUDA_ARCH__
  // j = floor(t kPerUnit) from the low word of a round-down FMA onto 2^52
  // (no F2I/I2F conversions); s = t - (j + 1/2) / kPerUnit, both steps exact.
  const double js = __fma_rd(t, kPerUnit, 4503599627370496.0);
  const double jd = js - 4503599627370496.0;
  const uint32_t ju = static_cast<uint32_t>(bits(js));
  const int j = static_cast<int>(ju < V::kNRec - 1 ? ju : V::kNRec - 1);
  const double s = fmad(jd, -1.0 / kPerUnit, t) - 0.5 / kPerUnit;
#else
  int j = static_cast<int>(t * kPerUnit);
  j = j < V::kNRec - 1 ? j : V::kNRec - 1;
  const double s = t - (j + 0.5) * (1.0 / kPerUnit);  // exact: j < 2^10, power-of-two width
#endif
  LPMC_DCHECK(j >= 0 && j < V::kNRec);
  const double* rec = tab.erfcx() + V::kRec * j;  // c_D, ..., c_1, c0 hi, c0 lo
  D2 c = load2(rec);
  double q = fmad(c.a, s, c.b);  // c_D s + c_{D-1}
  if constexpr (D % 2 == 0) {
#ifdef __CUDA_ARCH__
#pragma unroll
#endif
    for (int i = 2; i < D; i += 2) {  // c_{D-2} .. c_1
      c = load2(rec + S * i);
      q = fmad(q, s, c.a);
      q = fmad(q, s, c.b);
    }
    c = load2(rec + S * D);  // c0 hi, c0 lo
    return c.a + fmad(q, s, c.b);
  } else {
#ifdef __CUDA_ARCH__
#pragma unroll
#endif
    for (int i = 2; i < D - 1; i += 2) {  // c_{D-2} .. c_2
      c = load2(rec + S * i);
      q = fmad(q, s, c.a);
      q = fmad(q, s, c.b);
    }
    c = load2(rec + S * (D - 1));  // c1, c0 hi
    q = fmad(q, s, c.a);
    const D2 lo = load2(rec + S * (D + 1));  // c0 lo, pad
    return c.b + fmad(q, s, lo.a);
  }
}

// 2^k x for |k| <= 1022 and a normal result (the fast path has |k| <= 62).
LPMC_HD double scale(double x, int k) {
  return x * from_bits(static_cast<uint64_t>(1023 + k) << 52);
}

// erfc(t), 0 <= t < 6.5 (host/device identical).
LPMC_HD double erfc_fast(double t, const double* tab) {
  const FlatTab ft{tab};
  const double th = t * t;
  const double tl = fmad(t, t, -th);
  const ExpSplit e = exp_neg(th, tl, ft);
  return scale(e.p * erfcx_piecewise(t, ft), e.k);
}

#ifdef __CUDACC__
// per-thread view of the staged lane layout (copy = lane % 8)
__device__ __forceinline__ LaneTab lane_tab(const double* s) {
  const int c = 2 * static_cast<int>(threadIdx.x & (kLaneCopies - 1));
  return LaneTab{s + c, s + kLaneErfcxWords + c};
}
#endif

#ifdef __CUDACC__
// The reference's own formula on libdevice (slow path, t >= kDevTMax only).
__device__ __forceinline__ double phi_inv_lower_libdevice(double u) {
  double x;
  if (u < 0.02425) {
    const double q = sqrt(-2.0 * log(u));
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
  const double resid = 0.5 * erfc(-x * 0.7071067811865475244) - u;
  const double dens = 0.3989422804014326779 * exp(-0.5 * x * x);
  return x - resid / dens;
}

// log(u) for normal u > 0 to ~1e-13 absolute (Acklam tail only).
__device__ __forceinline__ double log_coarse(double u) {
  const uint64_t b = bits(u);
  int e = static_cast<int>(b >> 52) - 1023;
  uint64_t mb = (b & 0x000FFFFFFFFFFFFFull) | 0x3FF0000000000000ull;  // m in [1, 2)
  if (mb > 0x3FF6A09E667F3BCDull) {  // m > sqrt(2): use m/2, e+1
    mb -= 0x0010000000000000ull;
    e += 1;
  }
  const double m = from_bits(mb);
  const double f = m - 1.0;
  const double s = f * rcp_coarse(2.0 + f);
  const double s2 = s * s;
  double p = LPMC_K(kOffLogS + 6);
#pragma unroll
  for (int i = 5; i >= 0; --i) p = fmad(p, s2, LPMC_K(kOffLogS + i));
  return fmad(static_cast<double>(e), LPMC_K(kLn2), s * p);
}

// Acklam's initial approximation (gaussian.hpp:26-51) for v in (0, 1/2], to
// ~1e-12 relative of the reference's x0 (Newton squares that away).
// Central branch, v >= 0.02425: evaluated branch-free for every draw.
__device__ __forceinline__ double acklam_central(double v) {
  const double q = v - 0.5;
  const double r = q * q;
  double num = LPMC_K(kOffAckA);
#pragma unroll
  for (int i = 1; i < 6; ++i) num = fmad(num, r, LPMC_K(kOffAckA + i));
  double den = LPMC_K(kOffAckB);
#pragma unroll
  for (int i = 1; i < 5; ++i) den = fmad(den, r, LPMC_K(kOffAckB + i));
  den = fmad(den, r, 1.0);
  return (num * q) * rcp_refined(den);
}

// Tail branch, v < 0.02425 (4.85% of draws).
__device__ __forceinline__ double acklam_tail(double v) {
  const double q = sqrt_coarse(-2.0 * log_coarse(v));
  double num = LPMC_K(kOffAckC);
#pragma unroll
  for (int i = 1; i < 6; ++i) num = fmad(num, q, LPMC_K(kOffAckC + i));
  double den = LPMC_K(kOffAckD);
#pragma unroll
  for (int i = 1; i < 4; ++i) den = fmad(den, q, LPMC_K(kOffAckD + i));
  den = fmad(den, q, 1.0);
  return num * rcp_refined(den);
}

// The Newton step of gaussian.hpp:52-53, x0 - (Phi(x0) - v) / pdf(x0), with
// Phi(x0) = erfc(t)/2 and t = (-x0) * (1/sqrt 2) rounded as the reference
// rounds it.  *slow is set when t >= kDevTMax (6.5: v < 1e-20, outside the
// sampler's range; 3 with the lane layout: v < 1.1e-5); the caller then
// redoes that draw on libdevice (the value computed here for such a lane is
// garbage but never used, and no operation traps).
// mtab = the staged math table (erfcx records, then 2^(j/64)).
template <class V>
__device__ __forceinline__ double newton_fast(double x0, double v, const V& mtab, bool* slow) {
  const double t = -x0 * LPMC_K(kInvSqrt2);
  *slow = !(t < kDevTMax);
  const double th = t * t;
  const double tl = fmad(t, t, -th);
  const ExpSplit e = exp_neg(th, tl, mtab);
  const double pg = e.p * erfcx_piecewise(t, mtab);
  // resid = 0.5 erfc(t) - v = 2^k (pg/2 - v 2^-k); 1/pdf(x0) = sqrt(2 pi)
  // exp(t^2) = 2^-k sqrt(2 pi) / p.  Both power-of-two factors cancel, and
  // power-of-two scaling commutes with rounding, so this is bitwise
  // x0 - RN(RN(cdf - v) RN(sqrt(2 pi) 2^-k / p)) with two fewer FP64 ops.
  // v 2^-k: an exponent add (v is normal: v >= 2^-54, |k| <= 62).
  const double v_k = from_bits(bits(v) - (static_cast<uint64_t>(static_cast<int64_t>(e.k)) << 52));
  const double resid_k = fmad(pg, 0.5, -v_k);
#ifdef LPMC_X0_ACKLAM
  return x0 - resid_k * (LPMC_K(kSqrt2Pi) * rcp_coarse(e.p));
#else
  // Halley: x0 - r (1 - x0 r / 2), r = resid / pdf.  From the fp32 initial
  // guess (|e0| <= 4.3e-7 |x|) the error K e0^3, K = (x^2 + 2)/12, stays
  // below 1% of an ulp of Z for |x| <= 5 (Newton alone would leave e0^2 x/2).
  const double r = resid_k * (LPMC_K(kSqrt2Pi) * rcp_coarse(e.p));
  const double c = fmad(-0.5 * x0, r, 1.0);
  return fmad(-r, c, x0);
#endif
}

// exact_inv_cdf (gaussian.hpp:59-65) for D independent draws of one thread.
// The central rational runs for all draws; the tail rational (log, sqrt)
// runs in warp-uniform passes, one pending tail draw per lane per pass, so a
// warp pays for it about once per coarse step instead of once per draw with
// one lane active.  Must be called by every active lane of the warp.
// Stage 1: Acklam x0 of the reflected v = min(u, 1 - u) (gaussian.hpp:63)
// (central for all, tail pass for the rest).
#ifndef LPMC_X0_ACKLAM
// Initial guess in fp32 (tools/fit_x0f.py): x0 = q G(y), q = v - 1/2 exact in
// binary64, y = log2(v (1 - v)) from one MUFU.LG2, G a degree-8 polynomial
// with float immediates (v >= 2^-10), or degree 12 in sqrt(-y) in the tail
// (0.2 % of draws: a warp-uniform pass per draw slot).  ~4e-7 relative, which
// the Halley step in newton_fast squares and cubes away.  Replaces Acklam's
// binary64 rational (19 FP64 operations + a reciprocal, and a log/sqrt tail
// pass for 4.85 % of draws) by 2 FP64 operations and ~12 fp32/MUFU ones.
__device__ __forceinline__ float x0f_central(float x) {
  constexpr float c[LPMC_X0F_DEG_C + 1] = {LPMC_X0F_COEF_C};  // immediates after unrolling
  float p = c[LPMC_X0F_DEG_C];
#pragma unroll
  for (int i = LPMC_X0F_DEG_C - 1; i >= 0; --i) p = __fmaf_rn(p, x, c[i]);
  return p;
}

__device__ __forceinline__ float x0f_tail(float x) {
  constexpr float c[LPMC_X0F_DEG_T + 1] = {LPMC_X0F_COEF_T};
  float p = c[LPMC_X0F_DEG_T];
#pragma unroll
  for (int i = LPMC_X0F_DEG_T - 1; i >= 0; --i) p = __fmaf_rn(p, x, c[i]);
  return p;
}

template <int D>
__device__ __forceinline__ void phi_inv_stage1(const double (&v)[D], double (&x0)[D]) {
  float y[D], g[D];
  uint32_t pend = 0;
#pragma unroll
  for (int d = 0; d < D; ++d) {
    const float vf = __double2float_rn(v[d]);
    y[d] = __log2f(__fmaf_rn(-vf, vf, vf));  // log2(v (1 - v))
    g[d] = x0f_central(__fsub_rn(y[d], LPMC_X0F_Y_MID));
    if (vf < LPMC_X0F_SPLIT) pend |= 1u << d;
  }
  const unsigned mask = __activemask();
  if (__any_sync(mask, pend != 0)) {
#pragma unroll
    for (int d = 0; d < D; ++d) {
      if (__any_sync(mask, (pend >> d) & 1u)) {
        const float ny = -y[d];
        const float s = __fmul_rn(ny, rsqrtf(ny));
        const float gt = x0f_tail(__fsub_rn(s, LPMC_X0F_S_MID));
        if ((pend >> d) & 1u) g[d] = gt;
      }
    }
  }
#pragma unroll
  for (int d = 0; d < D; ++d) x0[d] = (v[d] - 0.5) * static_cast<double>(g[d]);
}
#else
template <int D>
__device__ __forceinline__ void phi_inv_stage1(const double (&v)[D], double (&x0)[D]) {
  uint32_t pend = 0;
#pragma unroll
  for (int d = 0; d < D; ++d) {
    x0[d] = acklam_central(v[d]);
    if (v[d] < LPMC_K(kTailU)) pend |= 1u << d;
  }
  const unsigned mask = __activemask();
  while (__any_sync(mask, pend != 0)) {
    double vs = 0.01;  // lanes with nothing pending evaluate a harmless value
#pragma unroll
    for (int d = D - 1; d >= 0; --d)
      if (pend & (1u << d)) vs = v[d];
    const double xt = acklam_tail(vs);
    const uint32_t low = pend & (0u - pend);
#pragma unroll
    for (int d = 0; d < D; ++d)
      if (low == (1u << d)) x0[d] = xt;
    pend &= pend - 1u;
  }
}
#endif

// Out of line: keeps the never-taken libdevice path out of the hot loop's
// instruction footprint (one copy per kernel instead of one per draw).
static __device__ __noinline__ double phi_inv_lower_slow(double v) {
  return phi_inv_lower_libdevice(v);
}

// The draws below the direct table (v < 2^-(B+1), 2^-B of all draws): the
// fp32 initial guess + Halley step on the erfc, tables read from global
// memory (L1/L2 hits).  Out of line, one copy per kernel.
static __device__ __noinline__ double phi_inv_lower_tail(double v) {
  const double vv[1] = {v};
  double x0[1];
  phi_inv_stage1<1>(vv, x0);
  bool slow;
  const double z = newton_fast(x0[0], v, FlatTab{kMathTable}, &slow);
  return slow ? phi_inv_lower_libdevice(v) : z;
}

// Stage 2: the Newton step, libdevice fix-up of out-of-range draws, sign
// (bit d of `neg`: u > 1/2).  EXACT_HALF: exactly 0 where bit d of `half`
// (u == 1/2, gaussian.hpp:62).  The hot loop instead flags such a draw
// (probability 2^-53) and has the path replayed with EXACT_HALF, which keeps
// two selects per draw out of the loop.
struct NoMid {
  __device__ __forceinline__ void operator()() const {}
};

// exact_inv_cdf for D reflected draws from the direct table: polynomial
// evaluation for all, the tail fix-up behind one combined branch, sign: the
// table holds the upper half, so the value is negated where sgn[d] =
// 0x80000000 (u < 1/2) and kept where it is 0.  u == 1/2 needs no special
// case (the zero record, +0 with sgn 0).  `mid` runs in the same basic block
// as the polynomial evaluations.
template <int D, class V, class Mid = NoMid>
__device__ __forceinline__ void phi_inv_direct_multi(const double (&v)[D],
                                                     const uint32_t (&sgn)[D], double (&z)[D],
                                                     const V& tab, Mid&& mid = Mid{}) {
  bool tail[D];
#pragma unroll
  for (int d = 0; d < D; ++d) z[d] = phi_inv_direct(v[d], tab, &tail[d]);
  mid();
  bool any_tail = false;
#pragma unroll
  for (int d = 0; d < D; ++d) any_tail |= tail[d];
  if (any_tail) {  // one rare region for all D draws
#pragma unroll
    for (int d = 0; d < D; ++d)
      if (tail[d]) z[d] = -phi_inv_lower_tail(v[d]);
  }
#pragma unroll
  for (int d = 0; d < D; ++d) z[d] = flip_sign_mask(z[d], sgn[d]);
}

// `mid` runs between the Newton block and the slow-path fix-ups, in the
// same basic block as the Newton steps (the sampler's software pipeline
// puts the previous batch's legs there, lpmc_level.cuh).
template <int D, bool EXACT_HALF = true, class V = FlatTab, class Mid = NoMid>
__device__ __forceinline__ void phi_inv_stage2(const double (&v)[D], const double (&x0)[D],
                                               uint32_t neg, uint32_t half, double (&z)[D],
                                               const V& mtab, Mid&& mid = Mid{}) {
  bool slow[D];
#pragma unroll
  for (int d = 0; d < D; ++d) z[d] = newton_fast(x0[d], v[d], mtab, &slow[d]);
  mid();
  bool any_slow = false;
#pragma unroll
  for (int d = 0; d < D; ++d) any_slow |= slow[d];
#pragma unroll
  for (int d = 0; d < D; ++d) {
    if (any_slow && slow[d]) z[d] = phi_inv_lower_slow(v[d]);
    const double r = (neg >> d) & 1u ? -z[d] : z[d];
    if constexpr (EXACT_HALF) {
      z[d] = (half >> d) & 1u ? 0.0 : r;
    } else {
      z[d] = r;
    }
  }
}

// exact_inv_cdf for D arbitrary u (diagnostics; the sampler reflects from
// its integer draws, dev::draw_reflect).
// -DLPMC_HALLEY_Z (A/B only): the round-1 fast mode (fp32 guess + Halley step
// on the erfc) instead of the direct table, in every kernel of the build.
template <int D, class V>
__device__ __forceinline__ void phi_inv_multi_direct(const double (&u)[D], double (&z)[D],
                                                     const V& tab) {
  double v[D];
  uint32_t sgn[D];
#pragma unroll
  for (int d = 0; d < D; ++d) {
    v[d] = u[d] > 0.5 ? 1.0 - u[d] : u[d];  // exact (gaussian.hpp:63)
    sgn[d] = u[d] < 0.5 ? 0x80000000u : 0u;  // u == 1/2: +0 (gaussian.hpp:62)
  }
  phi_inv_direct_multi<D>(v, sgn, z, tab);
}
template <int D>
__device__ __forceinline__ void phi_inv_multi(const double (&u)[D], double (&z)[D],
                                              const DirectTab& tab) {
  phi_inv_multi_direct<D>(u, z, tab);
}
template <int D>
__device__ __forceinline__ void phi_inv_multi(const double (&u)[D], double (&z)[D],
                                              const LaneDirectTab& tab) {
  phi_inv_multi_direct<D>(u, z, tab);
}

template <int D>
__device__ __forceinline__ void phi_inv_multi(const double (&u)[D], double (&z)[D],
                                              const FlatTab& mtab) {
#ifndef LPMC_HALLEY_Z
  (void)mtab;  // small kernels: the direct table straight from global memory
  phi_inv_multi_direct<D>(u, z, DirectTab{kDirectTable});
#else
  double v[D], x0[D];
  uint32_t neg = 0, half = 0;
#pragma unroll
  for (int d = 0; d < D; ++d) {
    v[d] = u[d] > 0.5 ? 1.0 - u[d] : u[d];  // exact (gaussian.hpp:63)
    neg |= (u[d] > 0.5 ? 1u : 0u) << d;
    half |= (u[d] == 0.5 ? 1u : 0u) << d;
  }
  phi_inv_stage1<D>(v, x0);
  phi_inv_stage2<D, true>(v, x0, neg, half, z, mtab);
#endif
}

// The same with the reference's formula on libdevice (diagnostics only).
__device__ __forceinline__ double phi_inv_libdevice(double u) {
  const bool upper = u > 0.5;
  const double r = phi_inv_lower_libdevice(upper ? 1.0 - u : u);
  const double z = upper ? -r : r;
  return u == 0.5 ? 0.0 : z;
}
#endif

}  // namespace math
}  // namespace lpmc_b200
