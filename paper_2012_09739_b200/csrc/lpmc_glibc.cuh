// Bit-exact restatement of the glibc 2.39 libm routines behind the
// reference's exact Gaussian (gaussian.hpp:15 std::erfc, :19 std::exp,
// :45 std::log; the reference itself is CPU C++ linked against glibc), so
// that the device's exact inverse CDF can reproduce the reference's Z bit for
// bit (LPMC_EXACT_Z_GLIBC).  The algorithms are glibc's, restated from their
// published structure and its x86-64 build (tools/glibc_constants.py names
// the sources and reads the constants; tests/test_glibc_math.py compares this
// code with the running libm bitwise):
//   exp   ARM optimized-routines exp, N = 128, FMA-contracted build (__exp_fma)
//   log   ARM optimized-routines log, N = 128, FMA-contracted build (__log_fma)
//   erfc  Sun fdlibm s_erf.c with glibc's Estrin-style evaluation, no FMA
// Restated ranges (a superset of what the sampler reaches, u >= 2^-54):
// exp for |x| < 1024, log for normal x outside [1 - 2^-4, 1 + 0x1.09p-4),
// erfc everywhere except the |x| >= 28 underflow branch.  Outside them *ok
// is cleared and the caller falls back.
//
// Plain + - * / sqrt: on the device every kernel is compiled with
// -fmad=false and IEEE division/sqrt, on the host with -ffp-contract=off, so
// each operator is one correctly rounded operation on both; the contracted
// glibc builds are reproduced with explicit fmad().
//
// Upstream notices of the restated algorithms:
//  * erfc -- Sun fdlibm s_erf.c:
//      Copyright (C) 1993 by Sun Microsystems, Inc. All rights reserved.
//      Developed at SunPro, a Sun Microsystems, Inc. business.
//      Permission to use, copy, modify, and distribute this
//      software is freely granted, provided that this notice
//      is preserved.
//    (as distributed in the GNU C Library, sysdeps/ieee754/dbl-64/s_erf.c,
//    GNU LGPL 2.1 or later)
//  * exp, log -- ARM optimized-routines (Copyright (c) 2018 Arm Limited;
//    upstream licence MIT OR Apache-2.0 WITH LLVM-exception), as contributed
//    to the GNU C Library (sysdeps/ieee754/dbl-64/e_exp.c, e_log.c,
//    e_exp_data.c, e_log_data.c; Copyright (C) 2018-2024 Free Software
//    Foundation, Inc., GNU LGPL 2.1 or later).
#pragma once

#include "lpmc_glibc_coef.h"
#include "lpmc_math.cuh"

namespace lpmc_b200 {
namespace glibc {

using math::bits;
using math::fmad;
using math::from_bits;

// Word offsets inside the staged math block (after the fast path's tables).
constexpr int kExpTabOff = math::kGlibcOff;        // 256 words (tail, sbits) x 128
constexpr int kLogTabOff = math::kGlibcOff + 256;  // 256 words (invc, logc) x 128

LPMC_HD double sqrt_rn(double x) {
#ifdef __CUDA_ARCH__
  return __dsqrt_rn(x);
#else
  return std::sqrt(x);
#endif
}

// exp's specialcase (512 <= |x| < 1024): the scale's exponent would leave
// the binary64 range, so it is offset, and a subnormal result is rounded once.
LPMC_HD double exp_special(double tmp, uint64_t sbits, uint64_t ki) {
  if ((ki & 0x80000000ull) == 0) {  // k > 0
    const double scale = from_bits(sbits - (1009ull << 52));
    return fmad(scale, tmp, scale) * 0x1p1009;
  }
  const double scale = from_bits(sbits + (1022ull << 52));
  const double st = scale * tmp;
  double y = scale + st;
  if (y < 1.0) {
    const double hi = y + 1.0;
    double lo = (scale - y) + st;
    lo = ((1.0 - hi) + y) + lo;
    y = (lo + hi) - 1.0;
    if (y == 0.0) y = 0.0;
  }
  return y * 0x1p-1022;
}

// exp (sysdeps/ieee754/dbl-64/e_exp.c, __exp_fma): x = k ln2/N + r,
// exp(x) = 2^(k/N) (1 + tail + r + r^2 (C2 + r C3) + r^4 (C4 + r C5)).
LPMC_HD double exp(double x, const double* mtab, bool* ok) {
  const uint32_t abstop = static_cast<uint32_t>(bits(x) >> 52) & 0x7ffu;
  bool special = false;
  if (abstop - 0x3c9u >= 0x3fu) {
    if (static_cast<int>(abstop) - 0x3c9 < 0) return 1.0 + x;  // |x| < 2^-54
    if (abstop > 0x408u) {                                      // |x| >= 1024, Inf, NaN
      *ok = false;                                              // not restated
      return 0.0;
    }
    special = true;  // 512 <= |x| < 1024
  }
  double kd = fmad(x, LPMC_GLIBC_EXP_INVLN2N, LPMC_GLIBC_EXP_SHIFT);
  const uint64_t ki = bits(kd);
  kd = kd - LPMC_GLIBC_EXP_SHIFT;
  double r = fmad(kd, LPMC_GLIBC_EXP_NEGLN2HIN, x);
  r = fmad(kd, LPMC_GLIBC_EXP_NEGLN2LON, r);
  const int idx = 2 * static_cast<int>(ki & 127u);
  const uint64_t top = ki << 45;
  const double tail = mtab[kExpTabOff + idx];
  const uint64_t sbits = bits(mtab[kExpTabOff + idx + 1]) + top;
  const double p23 = fmad(r, LPMC_GLIBC_EXP_C3, LPMC_GLIBC_EXP_C2);
  const double t0 = r + tail;
  const double r2 = r * r;
  const double p45 = fmad(r, LPMC_GLIBC_EXP_C5, LPMC_GLIBC_EXP_C4);
  const double t1 = fmad(p23, r2, t0);
  const double r4 = r2 * r2;
  const double tmp = fmad(r4, p45, t1);
  if (special) return exp_special(tmp, sbits, ki);
  const double scale = from_bits(sbits);
  return fmad(scale, tmp, scale);
}

// log (sysdeps/ieee754/dbl-64/e_log.c, __log_fma): x = 2^k z, z in
// [OFF, 2 OFF), log(x) = k ln2 + log(c) + log1p(z/c - 1) with c from the
// table subinterval of z.
LPMC_HD double log(double x, const double* mtab, bool* ok) {
  const uint64_t ix = bits(x);
  const uint32_t top = static_cast<uint32_t>(ix >> 48);
  if (ix - 0x3fee000000000000ull <= 0x308ffffffffffull || top - 0x0010u >= 0x7ff0u - 0x0010u) {
    *ok = false;  // near 1, or zero/subnormal/negative/Inf/NaN: not restated
    return 0.0;
  }
  const uint64_t tmp = ix - 0x3fe6000000000000ull;
  const int i = static_cast<int>((tmp >> 45) & 127u);
  const int k = static_cast<int>(static_cast<int64_t>(tmp) >> 52);
  const uint64_t iz = ix - (tmp & 0xfff0000000000000ull);
  const double invc = mtab[kLogTabOff + 2 * i];
  const double logc = mtab[kLogTabOff + 2 * i + 1];
  const double z = from_bits(iz);
  const double r = fmad(z, invc, -1.0);
  const double kd = static_cast<double>(k);
  const double w = fmad(kd, LPMC_GLIBC_LOG_LN2HI, logc);
  const double hi = w + r;
  const double lo = fmad(kd, LPMC_GLIBC_LOG_LN2LO, (w - hi) + r);
  const double r2 = r * r;
  const double p = fmad(fmad(r, LPMC_GLIBC_LOG_A4, LPMC_GLIBC_LOG_A3), r2,
                        fmad(r, LPMC_GLIBC_LOG_A2, LPMC_GLIBC_LOG_A1));
  const double y = fmad(r * r2, p, fmad(r2, LPMC_GLIBC_LOG_A0, lo));
  return y + hi;
}

#define LPMC_E(k, i) LPMC_GLIBC_ERFC_##k##_##i

// erfc (sysdeps/ieee754/dbl-64/s_erf.c) by |x| range; the branches are
// separate functions so the multi-draw sampler path can run the rare ones in
// warp-uniform passes.  Range codes of erfc_range():
enum : int { kErfcTiny = 0, kErfcB1 = 1, kErfcB2 = 2, kErfcB3 = 3, kErfcOut = 4 };

LPMC_HD int erfc_range(double x) {
  const uint32_t ix = static_cast<uint32_t>(bits(x) >> 32) & 0x7fffffffu;
  if (ix < 0x3c700000u) return kErfcTiny;  // |x| < 2^-56
  if (ix < 0x3feb0000u) return kErfcB1;    // |x| < 0.84375
  if (ix < 0x3ff40000u) return kErfcB2;    // |x| < 1.25
  if (ix < 0x403c0000u) return kErfcB3;    // |x| < 28 (x <= -6 included: a constant)
  return kErfcOut;                         // |x| >= 28, Inf, NaN
}

// 2^-56 <= |x| < 0.84375
LPMC_HD double erfc_b1(double x) {
  const int32_t hx = static_cast<int32_t>(bits(x) >> 32);
  const double z = x * x;
  const double z2 = z * z;
  const double z4 = z2 * z2;
  const double r = ((LPMC_E(R1, 0) * z - LPMC_E(R1, 1)) * z2 + (LPMC_E(R1, 2) * z + LPMC_E(R1, 3))) +
                   LPMC_E(R1, 4) * z4;
  const double s = (LPMC_E(S1, 3) * z + LPMC_E(S1, 4)) * z4 +
                   ((LPMC_E(S1, 0) * z + LPMC_E(S1, 1)) * z2 + (LPMC_E(S1, 2) * z + 1.0));
  const double xy = (r / s) * x;
  if (hx < 0x3fd00000) return 1.0 - (xy + x);  // x < 1/4
  return 0.5 - ((x - 0.5) + xy);
}

// 0.84375 <= |x| < 1.25
LPMC_HD double erfc_b2(double x) {
  const uint64_t bx = bits(x);
  const double s = from_bits(bx & 0x7fffffffffffffffull) - 1.0;
  const double s2 = s * s;
  const double s4 = s2 * s2;
  const double s6 = s2 * s4;
  const double P = (((LPMC_E(P2, 0) * s - LPMC_E(P2, 1)) * s2 + (LPMC_E(P2, 2) * s - LPMC_E(P2, 3))) +
                    (LPMC_E(P2, 4) * s - LPMC_E(P2, 5)) * s4) +
                   LPMC_E(P2, 6) * s6;
  const double Q = ((LPMC_E(Q2, 3) * s + LPMC_E(Q2, 4)) * s4 +
                    ((LPMC_E(Q2, 0) * s + LPMC_E(Q2, 1)) * s2 + (LPMC_E(Q2, 2) * s + 1.0))) +
                   LPMC_E(Q2, 5) * s6;
  const double pq = P / Q;
  if (static_cast<int64_t>(bx) >= 0) return LPMC_E(ERX, 1) - pq;  // (1 - erx) - P/Q
  return 1.0 + (pq + LPMC_E(ERX, 0));
}

// 1.25 <= |x| < 28
LPMC_HD double erfc_b3(double x, const double* mtab, bool* ok) {
  const uint64_t bx = bits(x);
  const int32_t hx = static_cast<int32_t>(bx >> 32);
  const uint32_t ix = static_cast<uint32_t>(hx) & 0x7fffffffu;
  const double ax = from_bits(bx & 0x7fffffffffffffffull);
  const double s = 1.0 / (x * x);
  const double s2 = s * s;
  const double s4 = s2 * s2;
  const double s6 = s2 * s4;
  double R, S;
  if (ix < 0x4006db6du) {  // |x| < 1/0.35
    R = (((LPMC_E(R3, 0) * s - LPMC_E(R3, 1)) * s2 + (LPMC_E(R3, 2) * s - LPMC_E(R3, 3))) +
         (LPMC_E(R3, 4) * s - LPMC_E(R3, 5)) * s4) +
        (LPMC_E(R3, 6) * s - LPMC_E(R3, 7)) * s6;
    S = ((LPMC_E(S3, 5) * s + LPMC_E(S3, 6)) * s6 +
         (((LPMC_E(S3, 0) * s + LPMC_E(S3, 1)) * s2 + (1.0 + LPMC_E(S3, 2) * s)) +
          (LPMC_E(S3, 3) * s + LPMC_E(S3, 4)) * s4)) +
        (s4 * s4) * LPMC_E(S3, 7);
  } else {
    if (hx < 0 && ix >= 0x40180000u) return 2.0 - 1e-300;  // x <= -6
    R = (((LPMC_E(R4, 0) * s - LPMC_E(R4, 1)) * s2 + (LPMC_E(R4, 2) * s - LPMC_E(R4, 3))) +
         (LPMC_E(R4, 4) * s - LPMC_E(R4, 5)) * s4) +
        LPMC_E(R4, 6) * s6;
    S = (((LPMC_E(S4, 0) * s + LPMC_E(S4, 1)) * s2 + (1.0 + LPMC_E(S4, 2) * s)) +
         (LPMC_E(S4, 3) * s + LPMC_E(S4, 4)) * s4) +
        (LPMC_E(S4, 5) * s + LPMC_E(S4, 6)) * s6;
  }
  const double z = from_bits(bits(ax) & 0xffffffff00000000ull);  // SET_LOW_WORD(z, 0)
  const double e1 = glibc::exp((-z) * z - LPMC_E(C5625, 0), mtab, ok);
  const double rs = R / S;
  const double e2 = glibc::exp((z - ax) * (z + ax) + rs, mtab, ok);
  const double r = e2 * e1;
  if (hx > 0) return r / ax;
  return 2.0 - r / ax;
}

LPMC_HD double erfc(double x, const double* mtab, bool* ok) {
  const int32_t hx = static_cast<int32_t>(bits(x) >> 32);
  switch (erfc_range(x)) {
    case kErfcTiny: return 1.0 - x;
    case kErfcB1: return erfc_b1(x);
    case kErfcB2: return erfc_b2(x);
    case kErfcB3: return erfc_b3(x, mtab, ok);
    default: break;
  }
  if ((static_cast<uint32_t>(hx) & 0x7fffffffu) >= 0x7ff00000u)  // Inf, NaN
    return static_cast<double>((static_cast<uint32_t>(hx) >> 31) << 1) + 1.0 / x;
  *ok = false;  // |x| >= 28: underflow branch, not restated
  return hx > 0 ? 0.0 : 2.0;
}
#undef LPMC_E

// Acklam's rational (gaussian.hpp:41-50) with plain (unfused) arithmetic and
// IEEE division, as the reference's build evaluates it.
LPMC_HD double acklam_central(double u) {  // u >= 0.02425
  const double q = u - 0.5;
  const double r = q * q;
  return (((((-3.969683028665376e+01 * r + 2.209460984245205e+02) * r + -2.759285104469687e+02) * r +
            1.383577518672690e+02) * r + -3.066479806614716e+01) * r + 2.506628277459239e+00) * q /
         (((((-5.447609879822406e+01 * r + 1.615858368580409e+02) * r + -1.556989798598866e+02) * r +
            6.680131188771972e+01) * r + -1.328068155288572e+01) * r + 1.0);
}

LPMC_HD double acklam_tail(double u, const double* mtab, bool* ok) {  // u < 0.02425
  const double q = sqrt_rn(-2.0 * glibc::log(u, mtab, ok));
  return (((((-7.784894002430293e-03 * q + -3.223964580411365e-01) * q + -2.400758277161838e+00) * q +
            -2.549732539343734e+00) * q + 4.374664141464968e+00) * q + 2.938163982698783e+00) /
         ((((7.784695709041462e-03 * q + 3.224671290700398e-01) * q + 2.445134137142996e+00) * q +
           3.754408661907416e+00) * q + 1.0);
}

// The Newton step (gaussian.hpp:52-53) given erfc(-x * (1/sqrt 2)).
LPMC_HD double newton(double x, double u, double erfc_t, const double* mtab, bool* ok) {
  const double err = 0.5 * erfc_t - u;
  return x - err / (0.3989422804014326779 * glibc::exp(-0.5 * x * x, mtab, ok));
}

LPMC_HD double erfc_arg(double x) { return -x * 0.7071067811865475244; }  // gaussian.hpp:15

// The reference's inv_cdf_lower (gaussian.hpp:26-55) for u in (0, 1/2].
LPMC_HD double inv_cdf_lower(double u, const double* mtab, bool* ok) {
  const double x = u < 0.02425 ? acklam_tail(u, mtab, ok) : acklam_central(u);
  return newton(x, u, glibc::erfc(erfc_arg(x), mtab, ok), mtab, ok);
}

// exact_inv_cdf (gaussian.hpp:59-65) in glibc mode; u in (0, 1).
LPMC_HD double inv_cdf(double u, const double* mtab, bool* ok) {
  if (u == 0.5) return 0.0;
  if (u > 0.5) return -inv_cdf_lower(1.0 - u, mtab, ok);
  return inv_cdf_lower(u, mtab, ok);
}

#ifdef __CUDACC__
// Scalar entry, out of line: the fallback of the multi-draw path and the
// diagnostics.  Outside the restated ranges (u == 1, which the sampler
// reports as a failure anyway; u < ~1e-300) the libdevice formula.
static __device__ __noinline__ double exact_z(double u, const double* mtab) {
  bool ok = u > 0.0 && u < 1.0;
  const double z = ok ? inv_cdf(u, mtab, &ok) : 0.0;
  return ok ? z : math::phi_inv_libdevice(u);
}

// D draws of one thread, warp-cooperatively (every active lane must call):
// Acklam's central rational and erfc's first range (|t| < 0.84375, about 77 %
// of draws) branch-free for all draws; Acklam's tail (4.9 %) and erfc's
// second (15 %) and third (7.7 %) ranges in warp-uniform passes that give
// each lane one pending draw per pass, so a warp pays for a rare range about
// once per batch instead of once per draw slot.  Bitwise the scalar path.
template <int D>
__device__ __forceinline__ void inv_cdf_multi(const double (&u)[D], double (&z)[D],
                                              const double* mtab) {
  const unsigned mask = __activemask();
  double v[D], x[D], e[D];
  uint32_t neg = 0, pend = 0, slow = 0;
#pragma unroll
  for (int d = 0; d < D; ++d) {
    neg |= (u[d] > 0.5 ? 1u : 0u) << d;
    v[d] = u[d] > 0.5 ? 1.0 - u[d] : u[d];
    x[d] = acklam_central(v[d]);
    pend |= (v[d] < 0.02425 ? 1u : 0u) << d;
    slow |= (u[d] > 0.0 && u[d] < 1.0 ? 0u : 1u) << d;
  }
  while (__any_sync(mask, pend != 0u)) {  // Acklam's tail
    double vs = 0.01;
#pragma unroll
    for (int d = D - 1; d >= 0; --d)
      if (pend & (1u << d)) vs = v[d];
    bool okt = true;
    const double xt = pend ? acklam_tail(vs, mtab, &okt) : 0.0;
    const uint32_t low = pend & (0u - pend);
#pragma unroll
    for (int d = 0; d < D; ++d)
      if (low == (1u << d)) {
        x[d] = xt;
        slow |= okt ? 0u : low;
      }
    pend &= pend - 1u;
  }
  uint32_t p2 = 0, p3 = 0;
#pragma unroll
  for (int d = 0; d < D; ++d) {
    const double t = erfc_arg(x[d]);
    const int rg = erfc_range(t);
    e[d] = rg == kErfcTiny ? 1.0 - t : erfc_b1(t);
    p2 |= (rg == kErfcB2 ? 1u : 0u) << d;
    p3 |= (rg == kErfcB3 ? 1u : 0u) << d;
    slow |= (rg == kErfcOut ? 1u : 0u) << d;
  }
  while (__any_sync(mask, p2 != 0u)) {  // 0.84375 <= t < 1.25
    double ts = 1.0;
#pragma unroll
    for (int d = D - 1; d >= 0; --d)
      if (p2 & (1u << d)) ts = erfc_arg(x[d]);
    const double et = erfc_b2(ts);
    const uint32_t low = p2 & (0u - p2);
#pragma unroll
    for (int d = 0; d < D; ++d)
      if (low == (1u << d)) e[d] = et;
    p2 &= p2 - 1u;
  }
  while (__any_sync(mask, p3 != 0u)) {  // 1.25 <= t < 28
    double ts = 2.0;
#pragma unroll
    for (int d = D - 1; d >= 0; --d)
      if (p3 & (1u << d)) ts = erfc_arg(x[d]);
    bool okt = true;
    const double et = erfc_b3(ts, mtab, &okt);
    const uint32_t low = p3 & (0u - p3);
#pragma unroll
    for (int d = 0; d < D; ++d)
      if (low == (1u << d)) {
        e[d] = et;
        slow |= okt ? 0u : low;
      }
    p3 &= p3 - 1u;
  }
#pragma unroll
  for (int d = 0; d < D; ++d) {
    bool okn = true;
    const double r = newton(x[d], v[d], e[d], mtab, &okn);
    slow |= okn ? 0u : 1u << d;
    z[d] = (neg >> d) & 1u ? -r : r;
    z[d] = u[d] == 0.5 ? 0.0 : z[d];
  }
  if (slow != 0u) {  // outside the restated ranges: never for the sampler's u >= 2^-54
#pragma unroll
    for (int d = 0; d < D; ++d)
      if ((slow >> d) & 1u) z[d] = exact_z(u[d], mtab);
  }
}
#endif

}  // namespace glibc
}  // namespace lpmc_b200
