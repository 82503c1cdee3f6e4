// The coupled level sampler: simulate_coupled (sde.hpp:211-284) for batches
// of 256 paths (one path per thread, two for the IEEE-half2 legs), each
// reduced to per-batch central moments by the threads that simulated it.
// Instances that draw exact Gaussians in the fast mode are persistent: one
// 768-thread CTA per SM, three 256-path groups looping over batches on their
// own named barriers, the direct inverse-CDF table in eight lane-private
// shared-memory copies (lpmc_math.cuh); the others run one batch per CTA.
//
// Hot loop per coarse step (two fine draws), software-pipelined across
// batches:
//   legs of the previous batch -> RNG for the next batch -> reflection of
//   both draws (three exact FP64 subtractions, no compares or selects) ->
//   exact Gaussians (direct table, one rare out-of-line tail call) ->
//   approximate Gaussians (reversed dyadic table copy) -> rounding into the
//   bar precision.
// State stays in registers.  Failure bookkeeping in the hot loop is a
// running minimum over the draws' low words (a superset of the u == 1 and
// u == 1/2 draws) and the range guards of the folded / native arithmetics;
// non-finite values are absorbing, so a non-finite end state <=> a
// non-finite operation somewhere.  Only a path that may have failed or left
// a guard is replayed (noinline, CHECKED, in the reference's own operation
// order) to find its values and its first failing step in the reference's
// serial order.
#pragma once

#include <cstdio>
#include <type_traits>

#include "lpmc_device.cuh"
#include "lpmc_glibc.cuh"

namespace lpmc_b200 {
namespace dev {

template <int NP>
struct PathEnd {
  double hf[NP], hc[NP], bf[NP], bc[NP];
  uint64_t fk[NP];   // CHECKED: first failure (n << 3 | stage), kNoFail if none
  bool suspect[NP];  // lean: the path may have failed
  bool range_bad;    // native bar legs left the exact range
};

__device__ __forceinline__ void note_fail(uint64_t& fk, bool bad, uint64_t n, uint32_t stage) {
  if (bad) {
    const uint64_t ord = (n << 3) | stage;
    fk = ord < fk ? ord : fk;
  }
}

// Uniforms of H draws x NP paths (draw-major), with their u == 1 bits (top)
// and u == 1/2 bits (half), read off the integer draws.
template <int D>
struct Uniforms {
  double u[D];
  uint32_t top, half;
};

// EXACT = false (the unchecked hot loop, which only needs to know that a
// path must be replayed): the path is flagged (lomin, below) when any of its
// draws has a low word of 0 or 0xffffffff, a superset of both
// special draws (kHalfDraw's low word is 0, kTopDraw's 0xffffffff) that costs
// two integer operations per draw instead of two 64-bit compares and their
// selects.  A false positive (probability 2^-31 per draw) only sends the path
// to the exact replay, which recomputes the same values.  -DLPMC_EXACT_SPECIAL
// restores the exact tests everywhere (A/B only).
// lomin[p] (EXACT = false): the running minimum over all draws of path p of
// (low word + 1) mod 2^32 -- <= 1 at the end of the path iff some draw's low
// word was 0xffffffff or 0: one fused add-min per draw.
template <int NP, int H, bool EXACT_ARG = true>
__device__ __forceinline__ void draw_uniforms(uint64_t (&kc)[NP], Uniforms<H * NP>& U,
                                              uint32_t (&lomin)[NP]) {
#ifdef LPMC_EXACT_SPECIAL
  constexpr bool EXACT = true;
#else
  constexpr bool EXACT = EXACT_ARG;
#endif
  U.top = 0u;
  U.half = 0u;
#pragma unroll
  for (int h = 0; h < H; ++h)
#pragma unroll
    for (int p = 0; p < NP; ++p) {
      const uint64_t b = next_draw(kc[p]);
      const int d = h * NP + p;
      U.u[d] = uniform_of(b);
      if constexpr (EXACT) {
        U.top |= (b == kTopDraw ? 1u : 0u) << d;
        U.half |= (b == kHalfDraw ? 1u : 0u) << d;
      } else {
        lomin[p] = min(lomin[p], static_cast<uint32_t>(b) + 1u);
      }
    }
}

// H draws per path starting at fine index n0 from pre-drawn uniforms `cur`:
// exact Gaussians (hat legs, or bar legs without a table) and R(approx)
// packed for the bar legs (sde.hpp:256-258).  With PREFETCH the uniforms of
// the next batch are drawn between the Acklam stage and the Newton stage, so
// the integer RNG interleaves with FP64 work instead of forming its own
// phase (software pipelining across batches).
// The fast mode's staged tables: the flat layout (math::FlatTab);
// -DLPMC_LANE_TABLES selects the conflict-free lane-private layout
// (math::LaneTab; same values).  Measured A/B (DESIGN.md section 8,
// profiles/r02_ab_summary.md): the lane layout halves the shared-memory
// wavefronts but leaves fp32 levels within 0.3 % and slows the emulated-fp16
// kernel by 3 % (the 8x table copies shrink L1 under the replay call's
// stack), so the flat layout stays the default.
#if !defined(LPMC_HALLEY_Z)
// The direct table (math::phi_inv_direct).  The fused level kernel is
// persistent where it draws exact Gaussians in the fast mode: one CTA per SM,
// kGroups groups of kBatch / NP threads, each group looping over batches, and
// eight lane-private copies of the table (144 KB) staged once per CTA -- the
// gathers are then free of bank conflicts (math::LaneDirectTab).  With one
// flat copy per 256-thread CTA the shared-memory crossbar bound the kernel:
// fp16 and fp32 legs ran at the same 1.68e11 path-steps/s
// (gpurun_out/r02g), 55 wavefronts per warp-step against 37 issue cycles.
// -DLPMC_FLAT_DIRECT keeps that one-batch-per-CTA form (A/B).  The
// warp-per-path kernel stages the flat table.
#ifndef LPMC_FLAT_DIRECT
#define LPMC_PERSISTENT 1
using FastTab = math::LaneDirectTab;
constexpr int kFastWords = math::kLaneDirectWords;
__device__ __forceinline__ void stage_fast(double* s) {
  for (int i = threadIdx.x; i < kFastWords; i += blockDim.x)
    s[i] = math::kDirectTable[math::lane_direct_source(i)];
}
// per-thread view (copy = lane % 8); the shared-space address goes through a
// volatile move so that ptxas keeps it in a register instead of re-deriving
// it (S2R SR_TID, S2UR SR_CgaCtaId, ULEA, ...) in every loop iteration
__device__ __forceinline__ FastTab fast_tab(const double* s) {
  const double* t = s + 2 * static_cast<int>(threadIdx.x & (math::kLaneCopies - 1));
  uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(t)), pinned;
  asm volatile("mov.u32 %0, %1;" : "=r"(pinned) : "r"(a));
  return FastTab{t, pinned};
}
#else
using FastTab = math::DirectTab;
constexpr int kFastWords = math::kDirectWords;
__device__ __forceinline__ void stage_fast(double* s) {
  for (int i = threadIdx.x; i < kFastWords; i += blockDim.x) s[i] = math::kDirectTable[i];
}
__device__ __forceinline__ FastTab fast_tab(const double* s) { return FastTab{s}; }
#endif
using WppTab = math::DirectTab;
constexpr int kWppFastWords = math::kDirectWords;
__device__ __forceinline__ void stage_wpp(double* s) {
  for (int i = threadIdx.x; i < kWppFastWords; i += blockDim.x) s[i] = math::kDirectTable[i];
}
__device__ __forceinline__ WppTab wpp_tab(const double* s) { return WppTab{s}; }
#elif !defined(LPMC_LANE_TABLES)
using FastTab = math::FlatTab;
constexpr int kFastWords = kFastMathWords;
__device__ __forceinline__ void stage_fast(double* s) { stage_math(s, kFastMathWords); }
__device__ __forceinline__ FastTab fast_tab(const double* s) { return FastTab{s}; }
#else
using FastTab = math::LaneTab;
constexpr int kFastWords = kLaneWords;
__device__ __forceinline__ void stage_fast(double* s) { stage_lane(s); }
__device__ __forceinline__ FastTab fast_tab(const double* s) { return math::lane_tab(s); }
#endif
#ifdef LPMC_HALLEY_Z
using WppTab = FastTab;
constexpr int kWppFastWords = kFastWords;
__device__ __forceinline__ void stage_wpp(double* s) { stage_fast(s); }
__device__ __forceinline__ WppTab wpp_tab(const double* s) { return fast_tab(s); }
#endif

// Exact-Gaussian mode of a level instance (values of LPMC_EXACT_Z_*).
enum : int { kZFast = 0, kZGlibc = 1 };

// Shared-space address of p, computed once: the volatile move keeps ptxas
// from re-deriving it (S2R SR_CgaCtaId, LEA, ...) inside the hot loop.
__device__ __forceinline__ uint32_t pinned_saddr(const void* p) {
  uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(p)), out;
  asm volatile("mov.u32 %0, %1;" : "=r"(out) : "r"(a));
  return out;
}

// Instances whose unchecked pass reads the reversed (and, for the native
// binary16 arithmetic, pre-scaled) copy of the dyadic table (approx_inv_up).
template <int TAB, bool DUMP, int ZM>
__host__ __device__ constexpr bool run_copy() {
#ifdef LPMC_HALLEY_Z
  return false;
#else
  return TAB == kTabDyadicLinear && !DUMP && ZM != kZGlibc;
#endif
}

template <class Arith, int TAB, bool NEED_EXACT, bool BAR, bool CHECKED, bool DUMP, int H,
          bool PREFETCH, int ZM, class Mid = math::NoMid>
__device__ __forceinline__ void gen_draws(const LevelArgs& A, const TableView& tab,
                                          const double* s_math, const FastTab& lt,
                                          const Arith& ar,
                                          uint64_t (&kc)[Arith::NP], bool (&u1)[Arith::NP],
                                          uint32_t (&lomin)[Arith::NP],
                                          uint64_t (&fk)[Arith::NP],
                                          const uint64_t (&local)[Arith::NP],
                                          const bool (&valid)[Arith::NP], uint64_t n0,
                                          const Uniforms<H * Arith::NP>& cur,
                                          Uniforms<H * Arith::NP>& next,
                                          double (&z)[H][Arith::NP],
                                          typename Arith::T (&zb)[H], Mid&& mid = Mid{}) {
  constexpr int NP = Arith::NP;
  constexpr int D = H * NP;
  const double(&u)[D] = cur.u;
#pragma unroll
  for (int h = 0; h < H; ++h)
#pragma unroll
    for (int p = 0; p < NP; ++p) {
      const uint32_t bit = 1u << (h * NP + p);
      if constexpr (CHECKED) {
        note_fail(fk[p], (cur.top & bit) != 0u, n0 + h, kStageDraw);
      } else {  // u == 1 or u == 1/2: the path is replayed exactly
#ifdef LPMC_EXACT_SPECIAL
        u1[p] |= ((cur.top | cur.half) & bit) != 0u;
#else
        (void)bit;  // flagged through lomin (draw_uniforms)
#endif
      }
    }
  double zz[D];
  double up[D];      // reflected draws of the approximate transform (fast exact mode)
  uint32_t sgn[D];   // common sign mask of both transforms (fast exact mode)
  // unchecked production instances with a dyadic-linear table evaluate it
  // from the reflected draw and the kernel's reversed table copy
  constexpr bool kShared = run_copy<TAB, DUMP, ZM>() && !CHECKED
#ifdef LPMC_HALLEY_Z
                           && false
#endif
      ;
  if constexpr (NEED_EXACT && ZM == kZGlibc) {
    if constexpr (PREFETCH) draw_uniforms<NP, H, CHECKED>(kc, next, lomin);
    glibc::inv_cdf_multi<D>(u, zz, s_math);
    mid();
  } else if constexpr (NEED_EXACT) {
    double v[D], x0[D];
    uint32_t neg = 0;
#if !defined(LPMC_HALLEY_Z)
    // Reflection without compares or selects: q = u - 1/2 is exact (u is an
    // odd multiple of 2^-54 below 1/2 and a multiple of 2^-53 above, so the
    // difference has at most 53 bits), v = 1/2 - |q| = min(u, 1 - u) exactly
    // (gaussian.hpp:63), and the approximate transform's reflected draw
    // u > 1/2 ? u : fl(1 - u) (invcdf_approx.hpp:47-49) is fl(1 - v) in both
    // half-planes (exact above 1/2, the reference's own rounding below).  The
    // sign bit of q is the common sign mask of both transforms (the direct
    // table holds the upper half, like the approximate transform); u == 1/2
    // gives q = +0, hence v = up = 1/2, mask 0 and the reference's +0.
    // Three FP64 operations and two LOP3 instead of a subtraction, a compare,
    // four selects of register halves and a mask select.
#pragma unroll
    for (int d = 0; d < D; ++d) {
      const double q = __dsub_rn(u[d], 0.5);
      sgn[d] = static_cast<uint32_t>(__double2hiint(q)) & 0x80000000u;
      v[d] = __dsub_rn(0.5, fabs(q));
      up[d] = __dsub_rn(1.0, v[d]);
    }
    (void)neg;
#else
#pragma unroll
    for (int d = 0; d < D; ++d) {
      const bool ng = u[d] > 0.5;
      v[d] = ng ? 1.0 - u[d] : u[d];  // exact (gaussian.hpp:63)
      neg |= (ng ? 1u : 0u) << d;
    }
#endif
#if !defined(LPMC_HALLEY_Z)
    (void)x0;
    if constexpr (CHECKED) {
      // the rare exact replay (also the warp-per-path kernel's, which stages
      // the flat layout): the same table straight from global memory
      const math::DirectTab gt{math::kDirectTable};
      if constexpr (PREFETCH) draw_uniforms<NP, H, CHECKED>(kc, next, lomin);
      math::phi_inv_direct_multi<D>(v, sgn, zz, gt, mid);
    } else {
#if defined(LPMC_DIRECT_MID_FIRST)  // legs, then the RNG, then the polynomials
      mid();
      if constexpr (PREFETCH) draw_uniforms<NP, H, CHECKED>(kc, next, lomin);
      math::phi_inv_direct_multi<D>(v, sgn, zz, lt);
#else  // the previous batch's legs in the polynomials' basic block
      if constexpr (PREFETCH) draw_uniforms<NP, H, CHECKED>(kc, next, lomin);
      math::phi_inv_direct_multi<D>(v, sgn, zz, lt, mid);
#endif
    }
#elif !defined(LPMC_MID_LATE)  // the previous batch's legs run beside the fp32 initial guesses
    mid();
    math::phi_inv_stage1<D>(v, x0);
    if constexpr (PREFETCH) draw_uniforms<NP, H, CHECKED>(kc, next, lomin);
    math::phi_inv_stage2<D, CHECKED>(v, x0, neg, cur.half, zz, lt);
#else
    math::phi_inv_stage1<D>(v, x0);
    if constexpr (PREFETCH) draw_uniforms<NP, H, CHECKED>(kc, next, lomin);
    math::phi_inv_stage2<D, CHECKED>(v, x0, neg, cur.half, zz, lt, mid);
#endif
  } else {
    if constexpr (PREFETCH) draw_uniforms<NP, H, CHECKED>(kc, next, lomin);
    mid();
#pragma unroll
    for (int d = 0; d < D; ++d) zz[d] = 0.0;
    if constexpr (kShared) {  // the reflection of the exact branch above (same comments)
#pragma unroll
      for (int d = 0; d < D; ++d) {
        const double q = __dsub_rn(u[d], 0.5);
        sgn[d] = static_cast<uint32_t>(__double2hiint(q)) & 0x80000000u;
        up[d] = __dsub_rn(1.0, __dsub_rn(0.5, fabs(q)));
      }
    }
  }
#pragma unroll
  for (int h = 0; h < H; ++h) {
    double zl[NP];
#pragma unroll
    for (int p = 0; p < NP; ++p) {
      z[h][p] = zz[h * NP + p];
      if constexpr (DUMP) {
        if (A.z_out != nullptr && valid[p]) {
          LPMC_DCHECK(local[p] < A.n_paths && n0 + h < (1ull << A.level));
          A.z_out[local[p] * (1ull << A.level) + n0 + h] = z[h][p];
        }
      }
      if constexpr (kShared) {
        zl[p] = approx_inv_up(tab, up[h * NP + p], sgn[h * NP + p]);
      } else if constexpr (TAB != kTabNone) {
        // lower = !(u > 1/2): one half-plane test for both transforms (at
        // u == 1/2 both selections of 1 - u and u coincide and the result is
        // the exact 0 of EXACT_HALF / the replay)
        zl[p] = approx_inv<CHECKED, TAB>(tab, u[h * NP + p], !(u[h * NP + p] > 0.5));
      } else {
        zl[p] = z[h][p];
      }
    }
    if constexpr (BAR) {
      if constexpr (Arith::kScaled && TAB == kTabNone) {
        zb[h] = ar.lift_exact(zl);  // exact Gaussians: scaled here (tables are pre-scaled)
      } else {
        zb[h] = ar.lift(zl);
      }
    }
  }
}

// Per-step leg updates in the reference's operation order, shared by the
// fused level kernel (simulate) and the warp-per-path kernel (wpp_kernel).
// State lives in the caller's locals (passed by reference: after inlining
// the same registers as the caller's own code).
// em_step (sde.hpp:60-68), carrier legs
template <int NP, bool CHECKED>
__device__ __forceinline__ void step_hat(const LevelArgs& A, double (&x)[NP], double dt,
                                         const double (&dw_or_z)[NP], bool fine,
                                         uint64_t (&fk)[NP], uint64_t n, uint32_t stage) {
#pragma unroll
  for (int p = 0; p < NP; ++p) {
    const double xp = x[p];
    const double drift = __dmul_rn(__dmul_rn(A.mu, xp), dt);
    // fine: (b sqrt_dt) z (sde.hpp:65); coarse: b dW (:77)
    const double diff = fine ? __dmul_rn(__dmul_rn(__dmul_rn(A.sigma, xp), A.sdtf), dw_or_z[p])
                             : __dmul_rn(__dmul_rn(A.sigma, xp), dw_or_z[p]);
    x[p] = __dadd_rn(xp, __dadd_rn(drift, diff));
    if constexpr (CHECKED) note_fail(fk[p], nonfinite64(x[p]), n, stage);
  }
}

// The carrier legs with power-of-two steps folded into the model constants
// (LevelArgs::bar_pow2 also proves the carrier's dt, 2dt, sqrt(dt) powers of
// two and mu, sigma, their products inside [2^-200, 2^200]):
//   drift  R(R(mu x) dt)         = R(x (mu dt))
//   fine   R(R(R(sigma x) s) z)  = R(R(x (sigma s)) z)
//   coarse dW = R(R(s z0) + R(s z1)) = s R(z0 + z1),
//          R(R(sigma x) dW)      = R(R(x (sigma s)) R(z0 + z1))
// bitwise while every intermediate is normal or zero, which RangeF64 proves
// once per coarse step (|x| in [2^-300, 2^300] there; two fine steps move |x|
// by factors in [2^-53, 2^11] or to exactly 0, where both forms give 0).  A
// path that leaves the range is replayed in the reference's own form
// (replay_checked).  Two fewer FP64 operations per fine step, three per coarse
// step -- and an FP64 instruction costs two issue slots on sm_100a.
// zs = z (fine) or R(z0 + z1) (coarse).
template <int NP>
__device__ __forceinline__ void step_hat_pw(double (&x)[NP], double mu_dt, double sg_sdt,
                                            const double (&zs)[NP]) {
#pragma unroll
  for (int p = 0; p < NP; ++p) {
    const double xp = x[p];
    const double drift = __dmul_rn(xp, mu_dt);
    const double diff = __dmul_rn(__dmul_rn(xp, sg_sdt), zs[p]);
    x[p] = __dadd_rn(xp, __dadd_rn(drift, diff));
  }
}

// em_step / em_step_kahan and the _dw forms (sde.hpp:60-116), bar precision
template <class Arith, bool KAHAN, bool CHECKED>
__device__ __forceinline__ void step_bar(const Arith& ar, typename Arith::Range& range,
                                         typename Arith::T& x, typename Arith::T& cmp,
                                         typename Arith::T mu_l, typename Arith::T sg_l,
                                         typename Arith::T dt_l, typename Arith::T sdt_l,
                                         typename Arith::T zb_or_dw, bool fine,
                                         uint64_t (&fk)[Arith::NP], uint64_t n, uint32_t stage) {
  using T = typename Arith::T;
  const T xp = x;
  T drift, diff;
  if constexpr (Arith::kPair) {
    // the same products pairwise: (mu x, sigma x), then (. dt, . sqrt_dt)
    // (fine) or (. 2dt, . dW) (coarse); bitwise the scalar form below
    const uint64_t ab = ar.mul2(pack2(mu_l, sg_l), pack2(xp, xp));
    if (fine) {
      const uint64_t cd = ar.mul2(ab, pack2(dt_l, sdt_l));
      drift = lo2(cd);
      diff = ar.mul(hi2(cd), zb_or_dw);
    } else {
      const uint64_t cd = ar.mul2(ab, pack2(dt_l, zb_or_dw));
      drift = lo2(cd);
      diff = hi2(cd);
    }
  } else {
    drift = ar.mul(ar.mul(mu_l, xp), dt_l);
    diff = fine ? ar.mul(ar.mul(ar.mul(sg_l, xp), sdt_l), zb_or_dw)
                : ar.mul(ar.mul(sg_l, xp), zb_or_dw);
  }
  const T inc = ar.add(drift, diff);
  if constexpr (KAHAN) {  // kahan_accumulate (sde.hpp:85-92)
    const T y = ar.sub(inc, cmp);
    const T s = ar.add(xp, y);
    cmp = ar.sub(ar.sub(s, xp), y);
    x = s;
  } else {
    x = ar.add(xp, inc);
  }
  range.track(x);
  if constexpr (CHECKED) {
    const uint32_t m = ar.bad(x);
#pragma unroll
    for (int p = 0; p < Arith::NP; ++p) note_fail(fk[p], (m >> p) & 1u, n, stage);
  }
}

// The bar-leg step with power-of-two steps folded into the model constants
// (LevelArgs::bar_pow2; native fp32 arithmetics only).  With dt = 2^-l,
// sqrt(dt) = 2^(-l/2) and mu, sigma, x, z already on the target grid:
//   drift  R(R(mu x) dt)          = R(x (mu dt))
//   fine   R(R(R(sigma x) s) z)   = R(R(x (sigma s)) z)
//   coarse dW = R(s z0 + s z1)    = s R(z0 + z1),
//          R(R(sigma x) dW)       = R(R(x (sigma s)) R(z0 + z1))
// because scaling by a power of two commutes with rounding while every
// intermediate stays normal -- which the native range guard guarantees (states
// in [2^-32, 2^33), constants in [2^-20, 2^20], dt >= 2^-40; a run that leaves
// the range is re-run in the exact binary64 emulation).  Two fewer roundings
// per fine step and 1.5 per coarse step; no failure can occur inside the
// guard, so the failure semantics are unchanged (the checked replay keeps the
// reference's own form).  zs = z (fine) or R(z0 + z1) (coarse).
template <class Arith, bool KAHAN>
__device__ __forceinline__ void step_bar_pw(const Arith& ar, typename Arith::Range& range,
                                            typename Arith::T& x, typename Arith::T& cmp,
                                            typename Arith::T mu_dt, typename Arith::T sg_sdt,
                                            typename Arith::T zs) {
  using T = typename Arith::T;
  const T xp = x;
  const T drift = ar.mul(xp, mu_dt);
  const T diff = ar.mul(ar.mul(xp, sg_sdt), zs);
  const T inc = ar.add(drift, diff);
  if constexpr (KAHAN) {  // kahan_accumulate (sde.hpp:85-92)
    const T y = ar.sub(inc, cmp);
    const T s = ar.add(xp, y);
    cmp = ar.sub(ar.sub(s, xp), y);
    x = s;
  } else {
    x = ar.add(xp, inc);
  }
  // the binary64 (carrier) legs are checked once per coarse step, like the
  // hat legs (RangeF64's argument); the native fp32 / bfloat16 legs on every
  // update
  if constexpr (!Arith::kRangeReplays) range.track(x);
}

// One coarse step of both bar legs with packed fp32 pairs (Arith::kPair):
// fine step n (zb0) and the coarse step (dW = sqrt_dt zb0 + sqrt_dt zb1) as
// (fine, coarse) pairs -- the two legs are independent, so evaluating them
// side by side changes no value -- then fine step n + 1 (zb1) alone.  Every
// pair operation is the reference's operation on each half (sde.hpp:60-116):
// fine diff (b sqrt_dt) z, coarse diff b dW, the coarse half multiplied by
// an exact 1 where the fine half takes its z.
template <class Arith, bool KAHAN>
__device__ __forceinline__ void step_bar_joint(const Arith& ar, typename Arith::Range& range,
                                               float& xf, float& xc, float& cf, float& cc,
                                               float mu_l, float sg_l, float dtf_l, float sdt_l,
                                               float dtc_l, float zb0, float zb1,
                                               uint64_t (&fk)[1], uint64_t n) {
  const uint64_t p = ar.mul2(pack2(zb0, zb1), pack2(sdt_l, sdt_l));
  const float dw = ar.add(lo2(p), hi2(p));  // sde.hpp:261-264
  const uint64_t X = pack2(xf, xc);
  const uint64_t a = ar.mul2(pack2(mu_l, mu_l), X);
  const uint64_t b = ar.mul2(pack2(sg_l, sg_l), X);
  const uint64_t drift = ar.mul2(a, pack2(dtf_l, dtc_l));
  const uint64_t e = ar.mul2(b, pack2(sdt_l, dw));
  const uint64_t diff = ar.mul2(e, pack2(zb0, ar.one()));
  const uint64_t inc = ar.add2(drift, diff);
  uint64_t Xn;
  if constexpr (KAHAN) {  // kahan_accumulate (sde.hpp:85-92) on both legs
    const uint64_t y = ar.sub2(inc, pack2(cf, cc));
    Xn = ar.add2(X, y);
    const uint64_t c = ar.sub2(ar.sub2(Xn, X), y);
    cf = lo2(c);
    cc = hi2(c);
  } else {
    Xn = ar.add2(X, inc);
  }
  xf = lo2(Xn);
  xc = hi2(Xn);
  range.track(xf);
  range.track(xc);
  step_bar<Arith, KAHAN, false>(ar, range, xf, cf, mu_l, sg_l, dtf_l, sdt_l, zb1, true, fk, n + 1,
                                kStageBarFine);
}

// Does the stream of path `local` hold a draw with u == 1 (b = 2^53 - 1) or
// u == 1/2 (b = 2^52) among this level's 2^level draws?  Out of line: runs
// only for the paths the low-word prefilter flagged.
static __device__ __noinline__ bool has_special_draw(const LevelArgs& A, uint64_t local) {
  uint64_t kc = path_key(A.seed_key, A.path_base + local) + A.counter0 * kCounterStep;
  const uint64_t n = 1ull << A.level;
  bool found = false;
  for (uint64_t i = 0; i < n; ++i) {
    const uint64_t b = next_draw(kc);
    found |= b == kTopDraw || b == kHalfDraw;
  }
  return found;
}

// iterations of a loop over `left` coarse steps, `g` per iteration, capped
// so that they fit 32 bits (the caller loops again)
__device__ __forceinline__ uint32_t trip_count(uint64_t left, int g) {
  const uint64_t t = (left + static_cast<uint64_t>(g - 1)) / static_cast<uint64_t>(g);
  return t > 0x40000000ull ? 0x40000000u : static_cast<uint32_t>(t);
}

template <class Arith, bool KAHAN, int LEGS, int TAB, bool CHECKED, bool DUMP, int ZM,
          bool PW = false>
__device__ __forceinline__ void simulate(const LevelArgs& A, const TableView& tab,
                                         const double* s_math,
                                         const uint64_t (&local)[Arith::NP],
                                         const bool (&valid)[Arith::NP],
                                         PathEnd<Arith::NP>& R) {
  using T = typename Arith::T;
  constexpr int NP = Arith::NP;
  constexpr bool kFineOnly = LEGS == 4;  // simulate_two_way (sde.hpp:162-196)
  constexpr bool kHat = (LEGS & 1) != 0 || kFineOnly;
  constexpr bool kBar = (LEGS & 2) != 0 || kFineOnly;
  constexpr bool kNeedExact = kHat || TAB == kTabNone;

  const Arith ar(A);
  // the fast mode's table view, once per path batch (its shared-space address
  // is pinned in a register, fast_tab)
  FastTab lt{};
  if constexpr (kNeedExact && ZM == kZFast) lt = fast_tab(s_math);
  typename Arith::Range range;
  // The carrier arithmetic needs its guard only where steps are folded
  // (step_bar_pw); its unfolded steps track into an object nobody reads.
  typename Arith::Range range_unread;
  typename Arith::Range& unfolded_range =
      (Arith::kRangeReplays && !Arith::kScaled) ? range_unread : range;
  uint64_t kc[NP];
  bool u1[NP];
  uint32_t lomin[NP];
  uint64_t fk[NP];
  double xhf[NP], xhc[NP];
#pragma unroll
  for (int p = 0; p < NP; ++p) {
    kc[p] = path_key(A.seed_key, A.path_base + local[p]) + A.counter0 * kCounterStep;
    u1[p] = false;
    lomin[p] = 0xffffffffu;
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

  constexpr bool kJoint = Arith::kPair && kBar && !kFineOnly && !CHECKED && !PW;
  constexpr bool kPw = PW && Arith::kPow2 && !CHECKED;
  const T mu_dtf = kPw ? ar.c(A.mu_dtf_l, 0) : T{};
  const T mu_dtc = kPw ? ar.c(A.mu_dtc_l, 0) : T{};
  const T sg_sdt = kPw ? ar.c(A.sg_sdt_l, 0) : T{};
  RangeF64 hrange[NP];
  const double h_mu_dtf = kPw ? A.hat_mu_dtf : 0.0, h_mu_dtc = kPw ? A.hat_mu_dtc : 0.0;
  const double h_sg_sdt = kPw ? A.hat_sg_sdt : 0.0;
  auto hat_fine = [&](const double (&z)[NP], uint64_t n) {
    if constexpr (kPw) {
      step_hat_pw<NP>(xhf, h_mu_dtf, h_sg_sdt, z);
    } else {
      step_hat<NP, CHECKED>(A, xhf, A.dtf, z, true, fk, n, kStageHatFine);
    }
  };
  auto bar_fine = [&](T zb, uint64_t n) {
    if constexpr (Arith::kScaled) {  // native binary16 with static scales: xbf = (fine, coarse)
      ar.template fine<KAHAN>(xbf, cmpf, zb, range);  // cmpf = (comp_fine, comp_coarse) / P2
    } else if constexpr (kPw) {
      step_bar_pw<Arith, KAHAN>(ar, range, xbf, cmpf, mu_dtf, sg_sdt, zb);
    } else {
      step_bar<Arith, KAHAN, CHECKED>(ar, unfolded_range, xbf, cmpf, mu_l, sg_l, dtf_l, sdtf_l, zb, true,
                                      fk, n, kStageBarFine);
    }
  };
  // coarse legs: dW = sqrt_dt z0 + sqrt_dt z1 in each precision (sde.hpp:259-264)
  auto coarse = [&](const double (&z0)[NP], const double (&z1)[NP], T zb0, T zb1, uint64_t n) {
    if constexpr (kHat && !kFineOnly && kPw) {
      double zs[NP];
#pragma unroll
      for (int p = 0; p < NP; ++p) zs[p] = __dadd_rn(z0[p], z1[p]);
      step_hat_pw<NP>(xhc, h_mu_dtc, h_sg_sdt, zs);
#pragma unroll
      for (int p = 0; p < NP; ++p) hrange[p].track(xhc[p]);
    } else if constexpr (kHat && !kFineOnly) {
      double dw[NP];
#pragma unroll
      for (int p = 0; p < NP; ++p)
        dw[p] = __dadd_rn(__dmul_rn(A.sdtf, z0[p]), __dmul_rn(A.sdtf, z1[p]));
      step_hat<NP, CHECKED>(A, xhc, A.dtc, dw, false, fk, n, kStageHatCoarse);
    }
    if constexpr (kHat && kPw) {  // once per coarse step (see RangeF64)
#pragma unroll
      for (int p = 0; p < NP; ++p) hrange[p].track(xhf[p]);
    }
    if constexpr (kBar && kPw && Arith::kRangeReplays && !Arith::kScaled) {
      range.track(xbf);  // folded binary64 bar legs: the same guard, the same cadence
      if constexpr (!kFineOnly) range.track(xbc);
    }
    if constexpr (kBar && !kFineOnly && Arith::kScaled) {
      // both bar legs were stepped as one pair in coarse_step below
    } else if constexpr (kBar && !kFineOnly && kPw) {
      step_bar_pw<Arith, KAHAN>(ar, range, xbc, cmpc, mu_dtc, sg_sdt, ar.add(zb0, zb1));
    } else if constexpr (kBar && !kFineOnly && !kJoint) {
      T dw;
      if constexpr (Arith::kPair) {
        const uint64_t p = ar.mul2(pack2(zb0, zb1), pack2(sdtf_l, sdtf_l));
        dw = ar.add(lo2(p), hi2(p));
      } else {
        dw = ar.add(ar.mul(sdtf_l, zb0), ar.mul(sdtf_l, zb1));
      }
      step_bar<Arith, KAHAN, CHECKED>(ar, unfolded_range, xbc, cmpc, mu_l, sg_l, dtc_l, sdtf_l, dw, false,
                                      fk, n, kStageBarCoarse);
    }
  };

  // all legs of one coarse step (fine n, fine n + 1, coarse) in the
  // reference's order; the unchecked instances with packed fp32 pairs step
  // the two bar legs side by side (step_bar_joint; the same values)
  auto coarse_step = [&](const double (&z0)[NP], const double (&z1)[NP], T zb0, T zb1,
                         uint64_t n) {
    if constexpr (kJoint) {
      if constexpr (kHat) {
        hat_fine(z0, n);
        hat_fine(z1, n + 1);
        coarse(z0, z1, zb0, zb1, n + 1);  // the hat leg only (kJoint: bar below)
      }
      step_bar_joint<Arith, KAHAN>(ar, range, xbf, xbc, cmpf, cmpc, mu_l, sg_l, dtf_l, sdtf_l,
                                   dtc_l, zb0, zb1, fk, n);
    } else if constexpr (Arith::kScaled && kBar && !kFineOnly) {
      if constexpr (kHat) hat_fine(z0, n);
      if constexpr (kHat) hat_fine(z1, n + 1);
      coarse(z0, z1, zb0, zb1, n + 1);  // the hat leg only
      ar.template coarse_step<KAHAN>(xbf, cmpf, zb0, zb1, range);
    } else {
      if constexpr (kHat) hat_fine(z0, n);
      if constexpr (kBar) bar_fine(zb0, n);
      if constexpr (kHat) hat_fine(z1, n + 1);
      if constexpr (kBar) bar_fine(zb1, n + 1);
      coarse(z0, z1, zb0, zb1, n + 1);
    }
  };

  // The draws of G coarse steps are generated together (independent chains
  // to hide FP64 latency, one tail pass per batch); the legs consume them in
  // the reference's order (sde.hpp:251-277), one batch later, inside the
  // next batch's Newton block (software pipeline below).  G = 1 with the
  // pipeline at 3 CTAs x 256 threads (85 registers) measured fastest
  // (32.1 -> 28.9 ms at level 10 against G = 2, no
  // pipeline, 4 CTAs).
  // Bar-only and glibc-mode instances keep two coarse steps per batch and no
  // pipeline (their measured optimum).
#if defined(LPMC_NO_PIPE_LEGS)
  constexpr bool kPipe = false;
#elif defined(LPMC_GLIBC_PIPE)
  constexpr bool kPipe = kNeedExact;
#else
  constexpr bool kPipe = kNeedExact && ZM == kZFast;
#endif
#ifndef LPMC_GLIBC_G
#define LPMC_GLIBC_G 2
#endif
#ifdef LPMC_COARSE_PER_BATCH
  constexpr int G = NP == 1 ? LPMC_COARSE_PER_BATCH : 1;
#else
  constexpr int G = NP == 1 ? (ZM == kZGlibc ? LPMC_GLIBC_G : kPipe ? 1 : 2) : 1;
#endif
  if (A.level == 0) {  // sde.hpp:237-249: one draw, fine legs only, coarse := 0
    double z[1][NP];
    T zb[1];
    Uniforms<NP> cur, unused;
    draw_uniforms<NP, 1, CHECKED>(kc, cur, lomin);
    gen_draws<Arith, TAB, kNeedExact, kBar, CHECKED, DUMP, 1, false, ZM>(
        A, tab, s_math, lt, ar, kc, u1, lomin, fk, local, valid, 0, cur, unused, z, zb);
    if constexpr (kHat) hat_fine(z[0], 0);
    if constexpr (kBar) bar_fine(zb[0], 0);
  } else {
    const uint64_t halves = 1ull << (A.level - 1);
    if (halves >= G) {
      // the batch after the last is drawn too (never consumed, its u == 1
      // bits never recorded): the price of a branch-free pipeline
      Uniforms<2 * G * NP> cur;
      draw_uniforms<NP, 2 * G, CHECKED>(kc, cur, lomin);
      if constexpr (kPipe) {
      // software pipeline: the legs of batch i run inside the Newton block of
      // batch i + 1 (one basic block: FP64/shared-load and FP32/integer work
      // interleave); values and failure ordinals are unchanged.
      double zp[2 * G][NP];
      T zbp[2 * G];
      {
        Uniforms<2 * G * NP> next;
        gen_draws<Arith, TAB, kNeedExact, kBar, CHECKED, DUMP, 2 * G, true, ZM>(
            A, tab, s_math, lt, ar, kc, u1, lomin, fk, local, valid, 0, cur, next, zp, zbp);
        cur = next;
      }
      auto legs = [&](const double (&zl)[2 * G][NP], const T (&zbl)[2 * G], uint64_t m0) {
#pragma unroll
        for (int g = 0; g < G; ++g) {
          const uint64_t n = 2 * (m0 + g);
          coarse_step(zl[2 * g], zl[2 * g + 1], zbl[2 * g], zbl[2 * g + 1], n);
        }
      };
      // 32-bit trip counter (m itself is only read by the checked and dump
      // instances): two loop instructions instead of six
      for (uint64_t m0 = G; m0 < halves;) {
      const uint32_t trips = trip_count(halves - m0, G);
      for (uint32_t it = 0; it < trips; ++it) {
        const uint64_t m = m0 + static_cast<uint64_t>(it) * G;  // dead in production instances
        double z[2 * G][NP];
        T zb[2 * G];
        Uniforms<2 * G * NP> next;
        gen_draws<Arith, TAB, kNeedExact, kBar, CHECKED, DUMP, 2 * G, true, ZM>(
            A, tab, s_math, lt, ar, kc, u1, lomin, fk, local, valid, 2 * m, cur, next, z, zb,
            [&]() { legs(zp, zbp, m - G); });
        cur = next;
#pragma unroll
        for (int i = 0; i < 2 * G; ++i) {
          zbp[i] = zb[i];
#pragma unroll
          for (int p = 0; p < NP; ++p) zp[i][p] = z[i][p];
        }
      }
      m0 += static_cast<uint64_t>(trips) * G;
      }
      legs(zp, zbp, halves - G);
      } else {
      for (uint64_t m0 = 0; m0 < halves;) {
      const uint32_t trips = trip_count(halves - m0, G);
      for (uint32_t it = 0; it < trips; ++it) {
        const uint64_t m = m0 + static_cast<uint64_t>(it) * G;  // dead in production instances
        double z[2 * G][NP];
        T zb[2 * G];
        Uniforms<2 * G * NP> next;
        gen_draws<Arith, TAB, kNeedExact, kBar, CHECKED, DUMP, 2 * G, true, ZM>(
            A, tab, s_math, lt, ar, kc, u1, lomin, fk, local, valid, 2 * m, cur, next, z, zb);
        cur = next;
#pragma unroll
        for (int g = 0; g < G; ++g) {
          const uint64_t n = 2 * (m + g);
          coarse_step(z[2 * g], z[2 * g + 1], zb[2 * g], zb[2 * g + 1], n);
        }
      }
      m0 += static_cast<uint64_t>(trips) * G;
      }
      }
    } else {  // fewer coarse steps than one batch: one coarse step at a time
      for (uint64_t m = 0; m < halves; ++m) {
        double z[2][NP];
        T zb[2];
        Uniforms<2 * NP> cur, unused;
        draw_uniforms<NP, 2, CHECKED>(kc, cur, lomin);
        gen_draws<Arith, TAB, kNeedExact, kBar, CHECKED, DUMP, 2, false, ZM>(
            A, tab, s_math, lt, ar, kc, u1, lomin, fk, local, valid, 2 * m, cur, unused, z, zb);
        coarse_step(z[0], z[1], zb[0], zb[1], 2 * m);
      }
    }
  }

  constexpr bool kCoarse = !kFineOnly;
  if constexpr (Arith::kScaled) xbc = xbf;  // one pair (fine, coarse): lane 1 is the coarse leg
  const uint32_t bad_f = kBar ? ar.bad(xbf) : 0u;
  const uint32_t bad_c = (kBar && kCoarse && A.level > 0) ? ar.bad(xbc) : 0u;
#pragma unroll
  for (int p = 0; p < NP; ++p) {
    R.hf[p] = kHat ? xhf[p] : 0.0;
    R.hc[p] = (kHat && kCoarse && A.level > 0) ? xhc[p] : 0.0;
    R.bf[p] = kBar ? ar.get(xbf, p) : 0.0;
    R.bc[p] = (kBar && kCoarse && A.level > 0) ? ar.get(xbc, Arith::kScaled ? 1 : p) : 0.0;
    R.fk[p] = fk[p];
    const bool hat_bad = kHat && (nonfinite64(R.hf[p]) || nonfinite64(R.hc[p]));
    const bool hat_range = kHat && kPw && A.level > 0 && hrange[p].bad();
    // native binary16: a path outside the guard is replayed in the emulation
    const bool bar_range = Arith::kRangeReplays && kBar && range.bad();
    // the low-word prefilter fired (2^-31 per draw): regenerate the path's
    // draws (RNG only, ~1/20 of a checked replay) and replay only if one of
    // them really is u == 1 or u == 1/2 -- at level 16 and above the filter's
    // false positives would otherwise cost whole-group replays
    bool special = false;
    if constexpr (!CHECKED) {
      if (lomin[p] <= 1u) special = has_special_draw(A, local[p]);
    }
    R.suspect[p] = u1[p] || special || hat_bad || hat_range || bar_range ||
                   ((bad_f >> p) & 1u) || ((bad_c >> p) & 1u);
#ifdef LPMC_TRACE_REPLAY
    if (!CHECKED && R.suspect[p]) {
      if constexpr (Arith::kScaled) {
        printf("suspect path %llu: u1 %d lomin %u hat_bad %d hat_range %d bar_range %d bad %u %u lo %08x hi %08x wmin %04x\n",
               static_cast<unsigned long long>(local[p]), int(u1[p]), lomin[p], int(hat_bad),
               int(hat_range), int(bar_range), bad_f, bad_c,
               *reinterpret_cast<const uint32_t*>(&range.lo),
               *reinterpret_cast<const uint32_t*>(&range.hi),
               static_cast<unsigned>(__half_as_ushort(range.wmin)));
      }
    }
#endif
  }
  R.range_bad = Arith::kRangeReplays ? false : range.bad();
}

// Exact replay of this thread's paths (only for suspects: a u == 1 or
// u == 1/2 draw, or a non-finite end state): exact transforms and the first
// failure in the reference's serial order.
template <class Arith, bool KAHAN, int LEGS, int TAB, int ZM>
__device__ __noinline__ void replay_checked(const LevelArgs& A, TableView tab,
                                            const double* s_math,
                                            const uint64_t (&local)[Arith::NP],
                                            const bool (&valid)[Arith::NP],
                                            PathEnd<Arith::NP>& R) {
  simulate<Arith, KAHAN, LEGS, TAB, true, false, ZM>(A, tab, s_math, local, valid, R);
}

// 256 threads x 3 CTAs per SM (85 registers) for one path per thread when
// the instance computes exact Gaussians in the fast mode (pipelined legs),
// x 4 CTAs (64 registers) for bar-only and glibc-mode instances; the half2
// instances (two paths, four draws per coarse step) get 128 threads (170 /
// 128 registers) so they do not spill.
#ifndef LPMC_LEVEL_MIN_CTAS
#define LPMC_LEVEL_MIN_CTAS 3
#endif
#ifndef LPMC_BAR_MIN_CTAS
#define LPMC_BAR_MIN_CTAS 4
#endif
#ifndef LPMC_GLIBC_MIN_CTAS
#define LPMC_GLIBC_MIN_CTAS 4
#endif
template <int LEGS, int TAB, int ZM>
__host__ __device__ constexpr int level_min_ctas() {
  const bool exact = (LEGS & 1) != 0 || LEGS == 4 || TAB == kTabNone;
  return ZM == kZGlibc ? LPMC_GLIBC_MIN_CTAS : exact ? LPMC_LEVEL_MIN_CTAS : LPMC_BAR_MIN_CTAS;
}

// Persistent instances: those that draw exact Gaussians in the fast mode.
// kGroups batches in flight per CTA, one CTA per SM (the lane-private table
// fills most of its shared memory); group g of CTA c runs batches
// c + g gridDim.x, then every kGroups gridDim.x-th.
constexpr int kGroups = 3;
template <int LEGS, int TAB, int ZM>
__host__ __device__ constexpr bool level_persistent() {
#ifdef LPMC_PERSISTENT
  return ZM == kZFast && ((LEGS & 1) != 0 || LEGS == 4 || TAB == kTabNone);
#else
  return false;
#endif
}
template <class Arith, int LEGS, int TAB, int ZM>
__host__ __device__ constexpr int level_threads() {
  return (level_persistent<LEGS, TAB, ZM>() ? kGroups : 1) * (kBatch / Arith::NP);
}
template <int LEGS, int TAB, int ZM>
__host__ __device__ constexpr int level_ctas() {
  return level_persistent<LEGS, TAB, ZM>() ? 1 : level_min_ctas<LEGS, TAB, ZM>();
}

template <class Arith, bool KAHAN, int LEGS, int TAB, bool DUMP, int ZM, bool PW = false>
__global__ void __launch_bounds__(level_threads<Arith, LEGS, TAB, ZM>(), level_ctas<LEGS, TAB, ZM>())
    level_kernel(const __grid_constant__ LevelArgs A) {
  constexpr int NP = Arith::NP;
  constexpr bool kFineOnly = LEGS == 4;
  constexpr bool kHat = (LEGS & 1) != 0 || kFineOnly;
  constexpr bool kBar = (LEGS & 2) != 0 || kFineOnly;
  constexpr bool kNeedExact = kHat || TAB == kTabNone;
  constexpr bool kPersist = level_persistent<LEGS, TAB, ZM>();
  constexpr int kG = kPersist ? kGroups : 1;
  constexpr int kGroupThreads = kBatch / NP;

  // dynamic shared memory: [the lane-private direct table (persistent
  // instances)] [the approximation table]; static: the flat fast-mode or
  // glibc-mode tables of the one-batch-per-CTA instances
  extern __shared__ __align__(16) double s_dyn[];
  constexpr int kStaged = ZM == kZGlibc ? kMathWords : kFastWords;
  __shared__ __align__(16) double s_static[(kNeedExact && !kPersist) ? kStaged : 2];
  const double* s_math = kPersist ? s_dyn : s_static;
  // [direct table (persistent)] [reversed copy (run_copy instances)] [the table]:
  // the unchecked pass's copy sits at a compile-time offset
  double* s_run = s_dyn + (kPersist ? kFastWords : 0);
  double* s_table = s_run + (run_copy<TAB, DUMP, ZM>() ? kRunCopyWords : 0);
  if constexpr (kNeedExact) {
    if constexpr (ZM == kZGlibc) {
      stage_math(s_static, kStaged);
    } else {
      stage_fast(kPersist ? s_dyn : s_static);
    }
  }
  TableView tab{};      // the reference's table (the replay's, for scaled arithmetics)
  TableView tab_run{};  // the table the unchecked pass evaluates
  if constexpr (TAB != kTabNone) {
    for (int i = threadIdx.x; i < A.table_words; i += blockDim.x) s_table[i] = A.table[i];
    tab = TableView{s_table, A.table_stride, A.K, A.degree, A.dyadic, A.table_simple, A.tail};
    tab_run = tab;
    static_assert(!Arith::kScaled || TAB == kTabDyadicLinear,
                  "scaled arithmetics: dyadic-linear tables");
    if constexpr (run_copy<TAB, DUMP, ZM>()) {
      // the unchecked pass's copy: records reversed (approx_inv_up) and, for
      // the native binary16 arithmetic, c0, c1 (and the tail records' value)
      // scaled by 2^kz -- exact, and the scaled polynomial value is the value
      // scaled
      double* s2 = s_run;
      for (int i = threadIdx.x; i < kRunCopyWords; i += blockDim.x) {
        const int w = i % kDyadicRecord;
        double val = A.table[run_copy_source(i / kDyadicRecord) * kDyadicRecord + w];
        if constexpr (Arith::kScaled) {
          if (w >= 2) val *= A.hs_zscale;
        }
        s2[i] = val;
      }
      tab_run = TableView{s2, A.table_stride, A.K, A.degree, A.dyadic, A.table_simple,
                          Arith::kScaled ? A.tail * A.hs_zscale : A.tail,
                          pinned_saddr(s2)};
    }
  }
  __syncthreads();

  const int grp = kPersist ? static_cast<int>(threadIdx.x) / kGroupThreads : 0;
  const int tid = kPersist ? static_cast<int>(threadIdx.x) - grp * kGroupThreads
                           : static_cast<int>(threadIdx.x);
  const uint64_t stride = kPersist ? static_cast<uint64_t>(kG) * gridDim.x : A.n_batches;
  for (uint64_t slot_b = blockIdx.x + static_cast<uint64_t>(grp) * gridDim.x; slot_b < A.n_batches;
       slot_b += stride) {
  const uint64_t batch = A.batch0 + slot_b;
  const uint64_t first = batch * kBatch;
  const uint64_t left = A.n_paths - first;
  const int count = left < kBatch ? static_cast<int>(left) : kBatch;
  uint64_t local[NP];
  bool valid[NP];
#pragma unroll
  for (int p = 0; p < NP; ++p) {
    const int slot = tid + p * kGroupThreads;
    local[p] = first + slot;
    valid[p] = slot < count;
  }

  PathEnd<NP> R;
  simulate<Arith, KAHAN, LEGS, TAB, false, DUMP, ZM, PW>(A, tab_run, s_math, local, valid, R);

  bool any_suspect = false;
#pragma unroll
  for (int p = 0; p < NP; ++p) any_suspect |= valid[p] && R.suspect[p];
  if (any_suspect) {  // rare: exact values and first failure (serial order)
#ifdef LPMC_TRACE_REPLAY  // debugging only: which paths are replayed
    printf("replay path %llu batch %llu\n", static_cast<unsigned long long>(local[0]),
           static_cast<unsigned long long>(slot_b));
#endif
    const bool range_bad = R.range_bad;  // (false for the arithmetics whose guards replay)
    replay_checked<typename Arith::Replay, KAHAN, LEGS, TAB, ZM>(A, tab, s_math, local, valid, R);
    R.range_bad |= range_bad;
#pragma unroll
    for (int p = 0; p < NP; ++p) {
      if (!valid[p] || R.fk[p] == kNoFail) continue;
      const uint64_t n = R.fk[p] >> 3;
      const uint32_t stage = static_cast<uint32_t>(R.fk[p] & 7u);
      uint32_t kind = stage == kStageDraw ? kKindU1 : kKindNonFinite;
      if (Arith::kIeee && (stage == kStageBarFine || stage == kStageBarCoarse)) kind = kKindState;
      atomicMin(A.err_key, err_key_of(local[p], kind, n, A.err_step_bits));
    }
  }
  if (R.range_bad) atomicOr(A.range_flag, 1u);

  // terminal values -> payoff -> per-path differences (mlmc.hpp:86-90)
  double dh[NP], db[NP];
#pragma unroll
  for (int p = 0; p < NP; ++p) {
    if constexpr (DUMP) {
      if (A.path_out != nullptr && valid[p]) {
        LPMC_DCHECK(local[p] < A.n_paths);
        double* o = A.path_out + 4 * local[p];
        o[0] = R.hf[p];
        o[1] = R.hc[p];
        o[2] = R.bf[p];
        o[3] = R.bc[p];
      }
    }
    double pf_h = R.hf[p], pc_h = R.hc[p], pf_b = R.bf[p], pc_b = R.bc[p];
    if (A.payoff == 1) {
      pf_h = fmax(__dsub_rn(R.hf[p], A.strike), 0.0);
      pf_b = fmax(__dsub_rn(R.bf[p], A.strike), 0.0);
      pc_h = (!kFineOnly && A.level > 0) ? fmax(__dsub_rn(R.hc[p], A.strike), 0.0) : 0.0;
      pc_b = (!kFineOnly && A.level > 0) ? fmax(__dsub_rn(R.bc[p], A.strike), 0.0) : 0.0;
    }
    dh[p] = kHat ? __dsub_rn(pf_h, pc_h) : 0.0;
    db[p] = kBar ? __dsub_rn(pf_b, pc_b) : 0.0;
  }
  if (A.path_diff != nullptr) {
#pragma unroll
    for (int p = 0; p < NP; ++p)
      if (valid[p]) {
        const uint64_t r = local[p] - A.batch0 * kBatch;  // slice-relative
        LPMC_DCHECK(local[p] < A.n_paths && r < A.n_batches * kBatch);
        A.path_diff[2 * r + 0] = dh[p];
        A.path_diff[2 * r + 1] = db[p];
      }
  }
  LPMC_DCHECK(slot_b < A.n_batches && count >= 1 && count <= kBatch);
  if (A.batch_acc != nullptr)
    batch_moments<NP, kG>(dh, db, valid, count, A.batch_acc + 15 * slot_b, tid, grp);
  }
}

// -------------------------------------------------- warp per path ---------
// The schedule for runs too small to fill the GPU (few paths of many steps:
// the deep levels of the two-way experiment, the estimator's pilot pass).
// The fused kernel then runs one lone warp per SM sub-partition and each
// path's 2^level steps back to back at dependency latency.  Here one warp
// owns one path: its 32 lanes draw 32 consecutive fine steps in parallel
// (counter-based stream: draw n of a path is mix64(mix64(key + n c3)),
// uniform.hpp:38-41), exact and approximate Gaussians by the fused kernel's
// own device functions (same values), then every lane steps the legs through
// those 32 draws (warp-uniform, values broadcast by shuffles), the same
// step functions as the fused kernel in the reference's order.  A path with
// a u == 1 or u == 1/2 draw or a non-finite end is replayed exactly
// (replay_checked, all lanes).  Lane 0 writes the path's (d_hat, d_bar) to
// path_diff; the batch reduction is the fused kernel's (path_batch_kernel
// runs batch_moments on them; or the sequential order), so the moments are
// bitwise the fused schedule's.  NP == 1 arithmetics only.
constexpr int kWppThreads = 256;  // 8 paths per CTA

template <class Arith, bool KAHAN, int LEGS, int TAB, int ZM>
__global__ void __launch_bounds__(kWppThreads) wpp_kernel(const __grid_constant__ LevelArgs A) {
  static_assert(Arith::NP == 1, "warp-per-path runs one path per warp");
  using T = typename Arith::T;
  constexpr bool kFineOnly = LEGS == 4;
  constexpr bool kHat = (LEGS & 1) != 0 || kFineOnly;
  constexpr bool kBar = (LEGS & 2) != 0 || kFineOnly;
  constexpr bool kNeedExact = kHat || TAB == kTabNone;

  extern __shared__ __align__(16) double s_table[];
  // glibc mode: the flat tables incl. glibc's; fast mode: the lane layout
  constexpr int kStaged = ZM == kZGlibc ? kMathWords : kWppFastWords;
  __shared__ __align__(16) double s_math[kNeedExact ? kStaged : 2];
  if constexpr (kNeedExact) {
    if constexpr (ZM == kZGlibc) {
      stage_math(s_math, kStaged);
    } else {
      stage_wpp(s_math);
    }
  }
  TableView tab{};
  if constexpr (TAB != kTabNone) {
    for (int i = threadIdx.x; i < A.table_words; i += blockDim.x) s_table[i] = A.table[i];
    tab = TableView{s_table, A.table_stride, A.K, A.degree, A.dyadic, A.table_simple, A.tail};
  }
  __syncthreads();

  const int lane = threadIdx.x & 31;
  const uint64_t local1[1] = {A.batch0 * kBatch + blockIdx.x * (kWppThreads / 32) + (threadIdx.x >> 5)};
  const uint64_t local = local1[0];
  if (local >= A.n_paths) return;  // the whole warp
  const bool valid[1] = {true};
  const unsigned full = 0xffffffffu;

  const Arith ar(A);
  typename Arith::Range range;
  uint64_t fk[1] = {kNoFail};
  double xhf[1] = {A.x0}, xhc[1] = {A.x0};
  const T mu_l = ar.c(A.mu_l, A.h_mu), sg_l = ar.c(A.sigma_l, A.h_sigma);
  const T dtf_l = ar.c(A.dtf_l, A.h_dtf), sdtf_l = ar.c(A.sdtf_l, A.h_sdtf);
  const T dtc_l = ar.c(A.dtc_l, A.h_dtc);
  T xbf = ar.c(A.x0_l, A.h_x0);
  T xbc = xbf;
  T cmpf = ar.zero(), cmpc = ar.zero();

  const uint64_t key = path_key(A.seed_key, A.path_base + local);
  const uint64_t n_fine = 1ull << A.level;  // level >= 1 (the host runs level 0 fused)
  bool special = false;
  for (uint64_t n0 = 0; n0 < n_fine; n0 += 32) {
    uint64_t kc = key + (A.counter0 + n0 + static_cast<uint64_t>(lane)) * kCounterStep;
    const uint64_t b = next_draw(kc);
    const double u[1] = {uniform_of(b)};
    const bool live = n0 + lane < n_fine;
    special |= __any_sync(full, live && (b == kTopDraw || b == kHalfDraw));
    double z[1] = {0.0};
    if constexpr (kNeedExact) {
      if constexpr (ZM == kZGlibc) {
        glibc::inv_cdf_multi<1>(u, z, s_math);
      } else {
        math::phi_inv_multi<1>(u, z, wpp_tab(s_math));
      }
    }
    T zb = ar.zero();
    if constexpr (kBar) {
      double zl[1];
      if constexpr (TAB != kTabNone) {
        zl[0] = approx_inv<false, TAB>(tab, u[0]);
      } else {
        zl[0] = z[0];
      }
      zb = ar.lift(zl);
    }
    const int steps = n_fine - n0 < 32 ? static_cast<int>(n_fine - n0) : 32;
    for (int s = 0; s < steps; s += 2) {
      const double z0[1] = {__shfl_sync(full, z[0], s)};
      const double z1[1] = {__shfl_sync(full, z[0], s + 1)};
      const T zb0 = __shfl_sync(full, zb, s);
      const T zb1 = __shfl_sync(full, zb, s + 1);
      const uint64_t n = n0 + s;
      if constexpr (kHat) step_hat<1, false>(A, xhf, A.dtf, z0, true, fk, n, kStageHatFine);
      if constexpr (kBar)
        step_bar<Arith, KAHAN, false>(ar, range, xbf, cmpf, mu_l, sg_l, dtf_l, sdtf_l, zb0, true,
                                      fk, n, kStageBarFine);
      if constexpr (kHat) step_hat<1, false>(A, xhf, A.dtf, z1, true, fk, n + 1, kStageHatFine);
      if constexpr (kBar)
        step_bar<Arith, KAHAN, false>(ar, range, xbf, cmpf, mu_l, sg_l, dtf_l, sdtf_l, zb1, true,
                                      fk, n + 1, kStageBarFine);
      if constexpr (kHat && !kFineOnly) {  // em_step_dw (sde.hpp:72-80)
        const double dw[1] = {__dadd_rn(__dmul_rn(A.sdtf, z0[0]), __dmul_rn(A.sdtf, z1[0]))};
        step_hat<1, false>(A, xhc, A.dtc, dw, false, fk, n + 1, kStageHatCoarse);
      }
      if constexpr (kBar && !kFineOnly) {
        const T dw = ar.add(ar.mul(sdtf_l, zb0), ar.mul(sdtf_l, zb1));
        step_bar<Arith, KAHAN, false>(ar, range, xbc, cmpc, mu_l, sg_l, dtc_l, sdtf_l, dw, false,
                                      fk, n + 1, kStageBarCoarse);
      }
    }
  }

  PathEnd<1> R;
  R.hf[0] = kHat ? xhf[0] : 0.0;
  R.hc[0] = (kHat && !kFineOnly) ? xhc[0] : 0.0;
  R.bf[0] = kBar ? ar.get(xbf, 0) : 0.0;
  R.bc[0] = (kBar && !kFineOnly) ? ar.get(xbc, 0) : 0.0;
  R.fk[0] = kNoFail;
  const bool hat_bad = kHat && (nonfinite64(R.hf[0]) || nonfinite64(R.hc[0]));
  const bool bar_bad = kBar && (ar.bad(xbf) != 0u || (!kFineOnly && ar.bad(xbc) != 0u));
  R.range_bad = range.bad();
  if (special || hat_bad || bar_bad) {  // rare: exact values and first failure (all lanes)
    const bool range_bad = R.range_bad;
    replay_checked<Arith, KAHAN, LEGS, TAB, ZM>(A, tab, s_math, local1, valid, R);
    R.range_bad |= range_bad;
    if (lane == 0 && R.fk[0] != kNoFail) {
      const uint64_t n = R.fk[0] >> 3;
      const uint32_t stage = static_cast<uint32_t>(R.fk[0] & 7u);
      const uint32_t kind = stage == kStageDraw ? kKindU1 : kKindNonFinite;
      atomicMin(A.err_key, err_key_of(local, kind, n, A.err_step_bits));
    }
  }
  if (lane != 0) return;
  if (R.range_bad) atomicOr(A.range_flag, 1u);
  if (A.path_out != nullptr) {
    double* o = A.path_out + 4 * local;
    o[0] = R.hf[0];
    o[1] = R.hc[0];
    o[2] = R.bf[0];
    o[3] = R.bc[0];
  }
  // terminal values -> payoff -> per-path differences (mlmc.hpp:86-90)
  double pf_h = R.hf[0], pc_h = R.hc[0], pf_b = R.bf[0], pc_b = R.bc[0];
  if (A.payoff == 1) {
    pf_h = fmax(__dsub_rn(R.hf[0], A.strike), 0.0);
    pf_b = fmax(__dsub_rn(R.bf[0], A.strike), 0.0);
    pc_h = !kFineOnly ? fmax(__dsub_rn(R.hc[0], A.strike), 0.0) : 0.0;
    pc_b = !kFineOnly ? fmax(__dsub_rn(R.bc[0], A.strike), 0.0) : 0.0;
  }
  if (A.path_diff != nullptr) {
    const uint64_t r = local - A.batch0 * kBatch;  // slice-relative
    A.path_diff[2 * r + 0] = kHat ? __dsub_rn(pf_h, pc_h) : 0.0;
    A.path_diff[2 * r + 1] = kBar ? __dsub_rn(pf_b, pc_b) : 0.0;
  }
}

// ------------------------------------------------------- per-arith glue ----
constexpr int kMaxTableK = 1024;
constexpr int kMaxDynSmem = (kTableRows * kMaxTableK + 1) * 8;  // + 1 / step_w

// Instances with power-of-two step folding (step_bar_pw): production
// (non-dump) fast-mode launches of the native fp32 arithmetics with bar legs.
template <class Arith, int LEGS, bool DUMP, int ZM>
constexpr bool has_pw() {
  // hat-only launches (LEGS == 1) exist for the carrier arithmetic only
  return Arith::kPow2 && !DUMP && ZM == kZFast && (LEGS != 1 || Arith::kRangeReplays);
}

// SMs of the current device (cached per device ordinal).
inline cudaError_t sm_count(int* out) {
  static int cache[64] = {};
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev >= 0 && dev < 64 && cache[dev] > 0) {
    *out = cache[dev];
    return cudaSuccess;
  }
  e = cudaDeviceGetAttribute(out, cudaDevAttrMultiProcessorCount, dev);
  if (e == cudaSuccess && dev >= 0 && dev < 64) cache[dev] = *out;
  return e;
}

template <class Arith, bool KAHAN, int LEGS, int TAB, bool DUMP, int ZM>
cudaError_t launch_one(const LevelArgs& A, cudaStream_t s) {
  constexpr bool kPersist = level_persistent<LEGS, TAB, ZM>();
  constexpr int kThreads = level_threads<Arith, LEGS, TAB, ZM>();
  const size_t smem = (TAB != kTabNone ? static_cast<size_t>(A.table_words) * sizeof(double) : 0) +
                      (run_copy<TAB, DUMP, ZM>() ? kRunCopyWords * sizeof(double) : 0) +
                      (kPersist ? static_cast<size_t>(kFastWords) * sizeof(double) : 0);
  unsigned grid = static_cast<unsigned>(A.n_batches);
  if constexpr (kPersist) {  // one CTA per SM, each group looping over batches
    int sms = 0;
    const cudaError_t e = sm_count(&sms);
    if (e != cudaSuccess) return e;
    grid = A.n_batches < static_cast<uint64_t>(sms) ? grid : static_cast<unsigned>(sms);
  }
  if constexpr (has_pw<Arith, LEGS, DUMP, ZM>()) {
    if (A.bar_pow2) {
      level_kernel<Arith, KAHAN, LEGS, TAB, DUMP, ZM, true><<<grid, kThreads, smem, s>>>(A);
      return cudaGetLastError();
    }
  }
  level_kernel<Arith, KAHAN, LEGS, TAB, DUMP, ZM><<<grid, kThreads, smem, s>>>(A);
  return cudaGetLastError();
}

// Table kind: none (exact Gaussians for the bar legs), a dyadic linear table
// with the signed-zero fix-up proved unnecessary (every BASELINE config; no
// per-draw branches), or any other table.
// Exact-Gaussian mode: glibc instances exist only where exact Gaussians are
// drawn (hat legs, or bar legs without a table).
template <class Arith, bool KAHAN, int LEGS, bool DUMP>
cudaError_t pick_approx(const LevelArgs& A, cudaStream_t s) {
  const bool glibc = A.exact_z == kZGlibc;  // == LPMC_EXACT_Z_GLIBC
  if (A.table == nullptr)
    return glibc ? launch_one<Arith, KAHAN, LEGS, kTabNone, DUMP, kZGlibc>(A, s)
                 : launch_one<Arith, KAHAN, LEGS, kTabNone, DUMP, kZFast>(A, s);
  if constexpr (LEGS != 2) {
    if (glibc) {
      if (A.dyadic && A.table_simple && A.degree == 1)
        return launch_one<Arith, KAHAN, LEGS, kTabDyadicLinear, DUMP, kZGlibc>(A, s);
      return launch_one<Arith, KAHAN, LEGS, kTabGeneric, DUMP, kZGlibc>(A, s);
    }
  }
  if (A.dyadic && A.table_simple && A.degree == 1)
    return launch_one<Arith, KAHAN, LEGS, kTabDyadicLinear, DUMP, kZFast>(A, s);
  return launch_one<Arith, KAHAN, LEGS, kTabGeneric, DUMP, kZFast>(A, s);
}

template <class Arith, bool KAHAN, bool DUMP>
cudaError_t pick_legs(const LevelArgs& A, cudaStream_t s) {
  if (A.legs == 2) return pick_approx<Arith, KAHAN, 2, DUMP>(A, s);
  if (A.legs == 4) return pick_approx<Arith, KAHAN, 4, DUMP>(A, s);
  return pick_approx<Arith, KAHAN, 3, DUMP>(A, s);
}

// Launch the path kernel of one bar arithmetic (legs 2 / 3 / 4 = fine only).
template <class Arith>
cudaError_t launch_level(const LevelArgs& A, bool kahan, bool dump, cudaStream_t s) {
  if (dump) return kahan ? pick_legs<Arith, true, true>(A, s) : pick_legs<Arith, false, true>(A, s);
  return kahan ? pick_legs<Arith, true, false>(A, s) : pick_legs<Arith, false, false>(A, s);
}

template <class Arith, bool KAHAN, int LEGS, bool DUMP, int ZM>
cudaError_t configure_tabs() {
  // persistent instances add the lane-private direct table
  constexpr int kGen = kMaxDynSmem + (level_persistent<LEGS, kTabGeneric, ZM>() ? kFastWords * 8 : 0);
  constexpr int kDyn = kMaxDynSmem + (level_persistent<LEGS, kTabDyadicLinear, ZM>() ? kFastWords * 8 : 0) +
                       kRunCopyWords * 8;
  cudaError_t e = cudaFuncSetAttribute(level_kernel<Arith, KAHAN, LEGS, kTabGeneric, DUMP, ZM>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, kGen);
  if (e != cudaSuccess) return e;
  if constexpr (level_persistent<LEGS, kTabNone, ZM>()) {  // no table: the direct table alone
    e = cudaFuncSetAttribute(level_kernel<Arith, KAHAN, LEGS, kTabNone, DUMP, ZM>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, kFastWords * 8);
    if (e != cudaSuccess) return e;
    if constexpr (has_pw<Arith, LEGS, DUMP, ZM>()) {
      e = cudaFuncSetAttribute(level_kernel<Arith, KAHAN, LEGS, kTabNone, DUMP, ZM, true>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, kFastWords * 8);
      if (e != cudaSuccess) return e;
    }
  }
  e = cudaFuncSetAttribute(level_kernel<Arith, KAHAN, LEGS, kTabDyadicLinear, DUMP, ZM>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, kDyn);
  if constexpr (has_pw<Arith, LEGS, DUMP, ZM>()) {
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(level_kernel<Arith, KAHAN, LEGS, kTabGeneric, DUMP, ZM, true>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, kGen);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(level_kernel<Arith, KAHAN, LEGS, kTabDyadicLinear, DUMP, ZM, true>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, kDyn);
  }
  return e;
}

template <class Arith, bool KAHAN, int LEGS, bool DUMP>
cudaError_t configure_one() {
  const cudaError_t e = configure_tabs<Arith, KAHAN, LEGS, DUMP, kZFast>();
  if constexpr (LEGS == 2) {
    return e;  // bar legs with a table draw no exact Gaussians: no glibc instance
  } else {
    if (e != cudaSuccess) return e;
    return configure_tabs<Arith, KAHAN, LEGS, DUMP, kZGlibc>();
  }
}

// The carrier's hat-only instances (LEGS == 1, no table).
template <class Arith, bool DUMP>
cudaError_t configure_hat_only() {
  if constexpr (level_persistent<1, kTabNone, kZFast>()) {
    cudaError_t e = cudaFuncSetAttribute(level_kernel<Arith, false, 1, kTabNone, DUMP, kZFast>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         kFastWords * 8);
    if constexpr (has_pw<Arith, 1, DUMP, kZFast>()) {
      if (e == cudaSuccess)
        e = cudaFuncSetAttribute(level_kernel<Arith, false, 1, kTabNone, DUMP, kZFast, true>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, kFastWords * 8);
    }
    return e;
  } else {
    return cudaSuccess;
  }
}

template <class Arith>
cudaError_t configure_level() {
  cudaError_t e = cudaSuccess;
  auto acc = [&](cudaError_t x) {
    if (e == cudaSuccess) e = x;
  };
  acc(configure_one<Arith, false, 4, false>());
  acc(configure_one<Arith, true, 4, false>());
  acc(configure_one<Arith, false, 4, true>());
  acc(configure_one<Arith, true, 4, true>());
  acc(configure_one<Arith, false, 2, false>());
  acc(configure_one<Arith, true, 2, false>());
  acc(configure_one<Arith, false, 3, false>());
  acc(configure_one<Arith, true, 3, false>());
  acc(configure_one<Arith, false, 2, true>());
  acc(configure_one<Arith, true, 2, true>());
  acc(configure_one<Arith, false, 3, true>());
  acc(configure_one<Arith, true, 3, true>());
  return e;
}

// Warp-per-path dispatch (same table-kind / exact-mode selection).
template <class Arith, bool KAHAN, int LEGS, int TAB, int ZM>
cudaError_t launch_wpp_one(const LevelArgs& A, cudaStream_t s) {
  const size_t smem = TAB != kTabNone ? static_cast<size_t>(A.table_words) * sizeof(double) : 0;
  const uint64_t paths = (A.batch0 + A.n_batches) * kBatch < A.n_paths
                             ? A.n_batches * kBatch
                             : A.n_paths - A.batch0 * kBatch;
  const unsigned blocks = static_cast<unsigned>((paths + kWppThreads / 32 - 1) / (kWppThreads / 32));
  wpp_kernel<Arith, KAHAN, LEGS, TAB, ZM><<<blocks, kWppThreads, smem, s>>>(A);
  return cudaGetLastError();
}

template <class Arith, bool KAHAN, int LEGS>
cudaError_t pick_approx_wpp(const LevelArgs& A, cudaStream_t s) {
  const bool glibc = A.exact_z == kZGlibc;
  if (A.table == nullptr)
    return glibc ? launch_wpp_one<Arith, KAHAN, LEGS, kTabNone, kZGlibc>(A, s)
                 : launch_wpp_one<Arith, KAHAN, LEGS, kTabNone, kZFast>(A, s);
  if constexpr (LEGS != 2) {
    if (glibc) {
      if (A.dyadic && A.table_simple && A.degree == 1)
        return launch_wpp_one<Arith, KAHAN, LEGS, kTabDyadicLinear, kZGlibc>(A, s);
      return launch_wpp_one<Arith, KAHAN, LEGS, kTabGeneric, kZGlibc>(A, s);
    }
  }
  if (A.dyadic && A.table_simple && A.degree == 1)
    return launch_wpp_one<Arith, KAHAN, LEGS, kTabDyadicLinear, kZFast>(A, s);
  return launch_wpp_one<Arith, KAHAN, LEGS, kTabGeneric, kZFast>(A, s);
}

template <class Arith>
cudaError_t launch_level_wpp(const LevelArgs& A, bool kahan, cudaStream_t s) {
  auto legs = [&](auto k) -> cudaError_t {
    constexpr bool K = decltype(k)::value;
    if constexpr (std::is_same_v<Arith, ArithCarrier>) {  // hat-only runs use the carrier
      if (A.legs == 1) return pick_approx_wpp<Arith, K, 1>(A, s);
    }
    if (A.legs == 2) return pick_approx_wpp<Arith, K, 2>(A, s);
    if (A.legs == 4) return pick_approx_wpp<Arith, K, 4>(A, s);
    return pick_approx_wpp<Arith, K, 3>(A, s);
  };
  return kahan ? legs(std::true_type{}) : legs(std::false_type{});
}

template <class Arith, bool KAHAN, int LEGS, int ZM>
cudaError_t configure_wpp_tabs() {
  cudaError_t e = cudaFuncSetAttribute(wpp_kernel<Arith, KAHAN, LEGS, kTabGeneric, ZM>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxDynSmem);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(wpp_kernel<Arith, KAHAN, LEGS, kTabDyadicLinear, ZM>,
                              cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxDynSmem);
}

template <class Arith>
cudaError_t configure_wpp() {
  cudaError_t e = cudaSuccess;
  auto acc = [&](cudaError_t x) {
    if (e == cudaSuccess) e = x;
  };
  if constexpr (std::is_same_v<Arith, ArithCarrier>) {
    acc(configure_wpp_tabs<Arith, false, 1, kZFast>());
    acc(configure_wpp_tabs<Arith, true, 1, kZFast>());
    acc(configure_wpp_tabs<Arith, false, 1, kZGlibc>());
    acc(configure_wpp_tabs<Arith, true, 1, kZGlibc>());
  }
  acc(configure_wpp_tabs<Arith, false, 2, kZFast>());
  acc(configure_wpp_tabs<Arith, true, 2, kZFast>());
  acc(configure_wpp_tabs<Arith, false, 3, kZFast>());
  acc(configure_wpp_tabs<Arith, true, 3, kZFast>());
  acc(configure_wpp_tabs<Arith, false, 4, kZFast>());
  acc(configure_wpp_tabs<Arith, true, 4, kZFast>());
  acc(configure_wpp_tabs<Arith, false, 3, kZGlibc>());
  acc(configure_wpp_tabs<Arith, true, 3, kZGlibc>());
  acc(configure_wpp_tabs<Arith, false, 4, kZGlibc>());
  acc(configure_wpp_tabs<Arith, true, 4, kZGlibc>());
  return e;
}

}  // namespace dev
}  // namespace lpmc_b200
