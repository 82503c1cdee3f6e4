/*
 * TEST INFRASTRUCTURE ONLY — CPU oracle (see lpmc_oracle.h).
 *
 * Restates the reference algorithm with the reference's exact operation
 * order so that, compiled with -O2 -ffp-contract=off against the same glibc,
 * it reproduces the reference bit for bit (checked in tests/ against
 * oracle/_ref and tests/golden/).  Never linked into the product.
 */
#define _GNU_SOURCE
#include "lpmc_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* ---- counter RNG: uniform.hpp:13-41 ------------------------------------- */

uint64_t orc_mix64(uint64_t z) { /* uniform.hpp:13-20 */
  z = (z ^ (z >> 33)) * 0xff51afd7ed558ccdULL;
  z = (z ^ (z >> 33)) * 0xc4ceb9fe1a85ec53ULL;
  return z ^ (z >> 33);
}

uint64_t orc_stream_word(uint64_t seed, uint64_t path, uint64_t ctr) { /* uniform.hpp:22-27 */
  const uint64_t k0 = orc_mix64(seed + 0x9e3779b97f4a7c15ULL);
  const uint64_t k1 = orc_mix64(k0 ^ orc_mix64(path + 0xbf58476d1ce4e5b9ULL));
  return orc_mix64(orc_mix64(k1 + ctr * 0x94d049bb133111ebULL));
}

double orc_uniform(uint64_t seed, uint64_t path, uint64_t ctr) { /* uniform.hpp:38-41 */
  const uint64_t w = orc_stream_word(seed, path, ctr);
  return (double)(w >> 11) * 0x1p-53 + 0x1p-54;
}

/* ---- exact inverse CDF: gaussian.hpp:14-65 (Acklam + one Newton step) --- */

static const double kA[6] = {-3.969683028665376e+01, 2.209460984245205e+02,
                             -2.759285104469687e+02, 1.383577518672690e+02,
                             -3.066479806614716e+01, 2.506628277459239e+00};
static const double kB[5] = {-5.447609879822406e+01, 1.615858368580409e+02,
                             -1.556989798598866e+02, 6.680131188771972e+01,
                             -1.328068155288572e+01};
static const double kC[6] = {-7.784894002430293e-03, -3.223964580411365e-01,
                             -2.400758277161838e+00, -2.549732539343734e+00,
                             4.374664141464968e+00, 2.938163982698783e+00};
static const double kD[4] = {7.784695709041462e-03, 3.224671290700398e-01,
                             2.445134137142996e+00, 3.754408661907416e+00};

static double lower_half(double u) { /* gaussian.hpp:26-55 */
  double x;
  if (u < 0.02425) {
    const double q = sqrt(-2.0 * log(u));
    double num = kC[0];
    for (int i = 1; i < 6; ++i) num = num * q + kC[i];
    double den = kD[0];
    for (int i = 1; i < 4; ++i) den = den * q + kD[i];
    den = den * q + 1.0;
    x = num / den;
  } else {
    const double q = u - 0.5;
    const double r = q * q;
    double num = kA[0];
    for (int i = 1; i < 6; ++i) num = num * r + kA[i];
    double den = kB[0];
    for (int i = 1; i < 5; ++i) den = den * r + kB[i];
    den = den * r + 1.0;
    x = num * q / den;
  }
  /* normal_cdf (gaussian.hpp:14-16) and normal_pdf (:18-20) inline */
  const double resid = 0.5 * erfc(-x * 0.7071067811865475244) - u;
  const double dens = 0.3989422804014326779 * exp(-0.5 * x * x);
  return x - resid / dens;
}

int orc_exact_inv_cdf(double u, double* z) { /* gaussian.hpp:59-65 */
  if (!(u > 0.0 && u < 1.0)) return ORC_FAIL_U1;
  if (u == 0.5) {
    *z = 0.0;
  } else if (u > 0.5) {
    *z = -lower_half(1.0 - u);
  } else {
    *z = lower_half(u);
  }
  return ORC_OK;
}

/* ---- emulated rounding: softfloat.hpp:69-80 ------------------------------ */

int orc_round(double x, int m, double* out) {
  if (!isfinite(x)) return ORC_FAIL_NONFINITE;
  if (x == 0.0 || m >= 52) {
    *out = x;
    return ORC_OK;
  }
  int e;
  const double f = frexp(x, &e);
  *out = ldexp(nearbyint(ldexp(f, m + 1)), e - (m + 1));
  return ORC_OK;
}

double orc_to_half(double x) { return (double)(_Float16)x; }

/* ---- approximate inverse CDF: invcdf_approx.hpp:44-145 ------------------- */

/* gauss_legendre (quadrature.hpp:17-41), same iteration and op order. */
static void gl_rule(int n, double* nodes, double* weights) {
  for (int i = 0; i < n; ++i) {
    double x = cos(M_PI * (i + 0.75) / (n + 0.5));
    double dp = 0.0;
    for (int it = 0; it < 100; ++it) {
      double pm = 1.0, pk = x;
      for (int k = 2; k <= n; ++k) {
        const double nxt = ((2.0 * k - 1.0) * x * pk - (k - 1.0) * pm) / k;
        pm = pk;
        pk = nxt;
      }
      dp = n * (x * pk - pm) / (x * x - 1.0);
      const double step = pk / dp;
      x -= step;
      if (fabs(step) < 1e-15) break;
    }
    nodes[i] = x;
    weights[i] = 2.0 / ((1.0 - x * x) * dp * dp);
  }
}

int orc_table_build(int kind, int K, double* bp, double* coeff, double* w_max, double* step_w,
                    double* tail) {
  if (K < 2 || (K & (K - 1)) != 0) return ORC_BAD_ARG; /* invcdf_approx.hpp:102-103 */
  double nodes[32], weights[32];
  gl_rule(32, nodes, weights);
  const double wm = fmin((double)(K + 1), 45.0); /* :108 */
  const double sw = (wm - 1.0) / K;               /* :109 */
  double lo = 0.5;
  for (int j = 0; j < K; ++j) {
    const double w_hi = 1.0 + (j + 1) * sw;
    const double hi = 1.0 - exp2(-w_hi);
    bp[j] = hi;
    double c0 = 0.0, c1 = 0.0, c2 = 0.0, c3 = 0.0;
    for (int i = 0; i < 32; ++i) { /* :125-137 */
      const double t = nodes[i];
      const double u = 0.5 * (lo + hi) + 0.5 * (hi - lo) * t;
      double z;
      orc_exact_inv_cdf(u, &z);
      const double f = weights[i] * z;
      const double p2 = 1.5 * t * t - 0.5;
      const double p3 = t * (2.5 * t * t - 1.5);
      c0 += 0.5 * f;
      if (kind != 2) c1 += 1.5 * f * t; /* constant:K keeps the degree-0 term only */
      if (kind == 1) {
        c2 += 2.5 * f * p2;
        c3 += 3.5 * f * p3;
      }
    }
    coeff[4 * j + 0] = c0;
    coeff[4 * j + 1] = c1;
    coeff[4 * j + 2] = c2;
    coeff[4 * j + 3] = c3;
    lo = hi;
  }
  const double* last = coeff + 4 * (K - 1); /* :141-143 */
  *tail = last[0] + last[1] + last[2] + last[3];
  *w_max = wm;
  *step_w = sw;
  return ORC_OK;
}

static double upper_eval(const orc_table* t, double u) { /* invcdf_approx.hpp:74-90 */
  const double w = -log2(1.0 - u);
  if (w >= t->w_max) return t->tail;
  int j = (int)((w - 1.0) / t->step_w);
  if (j < 0) j = 0;
  if (j >= t->K) j = t->K - 1;
  const double a = j == 0 ? 0.5 : t->bp[j - 1];
  const double b = t->bp[j];
  double s = 2.0 * (u - a) / (b - a) - 1.0;
  if (s < -1.0) s = -1.0;
  if (s > 1.0) s = 1.0;
  const double* c = t->coeff + 4 * j;
  const double p2 = 1.5 * s * s - 0.5;
  const double p3 = s * (2.5 * s * s - 1.5);
  return c[0] + c[1] * s + c[2] * p2 + c[3] * p3;
}

int orc_approx_eval(const orc_table* t, double u, double* z) { /* invcdf_approx.hpp:44-50 */
  if (!(u > 0.0 && u < 1.0)) return ORC_FAIL_U1;
  if (u == 0.5) {
    *z = 0.0;
  } else if (u < 0.5) {
    *z = -upper_eval(t, 1.0 - u);
  } else {
    *z = upper_eval(t, u);
  }
  return ORC_OK;
}

/* ---- coupled paths: sde.hpp:60-116, 202-284 ------------------------------ */

/* One low-precision ("bar") leg family: emulated RNE (m < 52), carrier
 * (m >= 52) or IEEE binary16 (ieee).  fail is sticky. */
typedef struct leg_ops {
  int m;
  int ieee;
  int fail;
} leg_ops;

static double op_round(leg_ops* o, double v) {
  if (o->fail) return v;
  if (o->ieee) return (double)(_Float16)v;
  double r;
  if (orc_round(v, o->m, &r) != ORC_OK) {
    o->fail = 1;
    return v;
  }
  return r;
}
/* fp_add / fp_sub / fp_mul (softfloat.hpp:95-111).  For IEEE half the
 * binary64 op is exact or innocuously double-rounded (53 >= 2*11+2). */
static double o_add(leg_ops* o, double a, double b) { return op_round(o, a + b); }
static double o_sub(leg_ops* o, double a, double b) { return op_round(o, a - b); }
static double o_mul(leg_ops* o, double a, double b) { return op_round(o, a * b); }

typedef struct kahan_t {
  double sum, comp;
} kahan_t;

/* em_step / em_step_dw (sde.hpp:60-80) with make_gbm lambdas (:35-40). */
static double inc_fine(leg_ops* o, double mu, double sg, double x, double dt, double sdt,
                       double z) {
  const double a = o_mul(o, mu, x);
  const double b = o_mul(o, sg, x);
  const double drift = o_mul(o, a, dt);
  const double diff = o_mul(o, o_mul(o, b, sdt), z);
  return o_add(o, drift, diff);
}
static double inc_coarse(leg_ops* o, double mu, double sg, double x, double dt, double dw) {
  const double a = o_mul(o, mu, x);
  const double b = o_mul(o, sg, x);
  const double drift = o_mul(o, a, dt);
  const double diff = o_mul(o, b, dw);
  return o_add(o, drift, diff);
}
/* kahan_accumulate (sde.hpp:85-92) or the plain outer add (:67, :79). */
static double accumulate(leg_ops* o, int kahan, kahan_t* k, double x, double inc) {
  if (!kahan) return o_add(o, x, inc);
  const double y = o_sub(o, inc, k->comp);
  const double s = o_add(o, k->sum, y);
  k->comp = o_sub(o, o_sub(o, s, k->sum), y);
  k->sum = s;
  return s;
}

static double payoff(const orc_config* c, double v) {
  if (c->payoff == 1) return fmax(v - c->strike, 0.0);
  return v;
}

/* simulate_coupled (sde.hpp:211-284).  Returns a failure kind; *fail_step
 * gets the fine step index of the first failure (coarse: 2m+1). */
int orc_simulate_coupled(const orc_config* c, uint64_t path, double* out4, double* z_out,
                         uint64_t* fail_step) {
  return orc_simulate_coupled_z(c, path, NULL, out4, z_out, fail_step);
}

/* As orc_simulate_coupled, but z_in (optional, 2^l values) replaces the exact
 * Gaussians: replays the legs on the device's own Z bit for bit. */
int orc_simulate_coupled_z(const orc_config* c, uint64_t path, const double* z_in, double* out4,
                           double* z_out, uint64_t* fail_step) {
  if (c->level < 0) return ORC_BAD_ARG;
  const uint64_t n_fine = (uint64_t)1 << c->level;
  const double dtf = ldexp(c->horizon, -c->level);
  const double sdtf = sqrt(dtf);
  const double dtc = 2.0 * dtf;
  leg_ops lo = {c->mantissa_bits, c->ieee_half, 0};
  leg_ops hi = {52, 0, 0};
  /* constants rounded once (sde.hpp:222-224; make_gbm :36,:39) */
  const double dtf_l = op_round(&lo, dtf);
  const double sdtf_l = op_round(&lo, sdtf);
  const double dtc_l = op_round(&lo, dtc);
  const double mu_l = op_round(&lo, c->mu);
  const double sg_l = op_round(&lo, c->sigma);
  double xb_f = op_round(&lo, c->x0);
  if (lo.fail || !isfinite(c->mu) || !isfinite(c->sigma)) {
    *fail_step = 0;
    return ORC_FAIL_NONFINITE;
  }
  double xh_f = c->x0, xh_c = c->x0, xb_c = xb_f;
  kahan_t kf = {xb_f, 0.0}, kc = {xb_c, 0.0};

  const uint64_t key0 = orc_mix64(c->seed + 0x9e3779b97f4a7c15ULL);
  const uint64_t key = orc_mix64(key0 ^ orc_mix64(path + 0xbf58476d1ce4e5b9ULL));
  uint64_t ctr = 0;

#define ORC_DRAW(Z, ZB, N)                                                              \
  do {                                                                                 \
    const uint64_t w_ = orc_mix64(orc_mix64(key + ctr * 0x94d049bb133111ebULL));       \
    ++ctr;                                                                             \
    const double u_ = (double)(w_ >> 11) * 0x1p-53 + 0x1p-54;                          \
    if (orc_exact_inv_cdf(u_, &(Z)) != ORC_OK) {                                       \
      *fail_step = (N);                                                                \
      return ORC_FAIL_U1;                                                              \
    }                                                                                  \
    if (z_in) (Z) = z_in[N];                                                           \
    if (z_out) z_out[N] = (Z);                                                         \
    double a_ = (Z);                                                                   \
    if (c->table) orc_approx_eval(c->table, u_, &a_);                                  \
    (ZB) = op_round(&lo, a_);                                                          \
  } while (0)

#define ORC_CHECK(N)                                                   \
  do {                                                                 \
    if (hi.fail || (!lo.ieee && lo.fail)) {                            \
      *fail_step = (N);                                                \
      return ORC_FAIL_NONFINITE;                                       \
    }                                                                  \
  } while (0)
#define ORC_CHECK_STATE(X, N)                                          \
  do {                                                                 \
    if (lo.ieee && !isfinite(X)) {                                     \
      *fail_step = (N);                                                \
      return ORC_FAIL_STATE;                                           \
    }                                                                  \
  } while (0)

  if (c->level == 0) { /* sde.hpp:237-249 */
    double z, zb;
    ORC_DRAW(z, zb, 0);
    xh_f = accumulate(&hi, 0, NULL, xh_f, inc_fine(&hi, c->mu, c->sigma, xh_f, dtf, sdtf, z));
    ORC_CHECK(0);
    xb_f = accumulate(&lo, c->kahan, &kf, xb_f, inc_fine(&lo, mu_l, sg_l, xb_f, dtf_l, sdtf_l, zb));
    ORC_CHECK(0);
    ORC_CHECK_STATE(xb_f, 0);
    out4[0] = xh_f;
    out4[1] = 0.0;
    out4[2] = xb_f;
    out4[3] = 0.0;
    return ORC_OK;
  }
  for (uint64_t m = 0; m < n_fine / 2; ++m) { /* sde.hpp:251-277 */
    double dwh[2], dwb[2];
    for (int half = 0; half < 2; ++half) {
      const uint64_t n = 2 * m + half;
      double z, zb;
      ORC_DRAW(z, zb, n);
      dwh[half] = sdtf * z;
      dwb[half] = o_mul(&lo, sdtf_l, zb);
      xh_f = accumulate(&hi, 0, NULL, xh_f, inc_fine(&hi, c->mu, c->sigma, xh_f, dtf, sdtf, z));
      ORC_CHECK(n);
      xb_f = accumulate(&lo, c->kahan, &kf, xb_f,
                        inc_fine(&lo, mu_l, sg_l, xb_f, dtf_l, sdtf_l, zb));
      ORC_CHECK(n);
      ORC_CHECK_STATE(xb_f, n);
    }
    const double dwc_h = dwh[0] + dwh[1];
    const double dwc_b = o_add(&lo, dwb[0], dwb[1]);
    xh_c = accumulate(&hi, 0, NULL, xh_c, inc_coarse(&hi, c->mu, c->sigma, xh_c, dtc, dwc_h));
    ORC_CHECK(2 * m + 1);
    xb_c = accumulate(&lo, c->kahan, &kc, xb_c, inc_coarse(&lo, mu_l, sg_l, xb_c, dtc_l, dwc_b));
    ORC_CHECK(2 * m + 1);
    ORC_CHECK_STATE(xb_c, 2 * m + 1);
  }
#undef ORC_DRAW
#undef ORC_CHECK
#undef ORC_CHECK_STATE
  out4[0] = xh_f;
  out4[1] = xh_c;
  out4[2] = xb_f;
  out4[3] = xb_c;
  return ORC_OK;
}

/* ---- moments: stats.hpp:15-54 -------------------------------------------- */

void orc_moments_add(orc_moments* a, double x) {
  const uint64_t before = a->n;
  a->n += 1;
  const double dn = (double)a->n;
  const double delta = x - a->mean;
  const double dl = delta / dn;
  const double dl2 = dl * dl;
  const double t1 = delta * dl * (double)before;
  a->mean += dl;
  a->m4 += t1 * dl2 * (dn * dn - 3.0 * dn + 3.0) + 6.0 * dl2 * a->m2 - 4.0 * dl * a->m3;
  a->m3 += t1 * dl * (dn - 2.0) - 3.0 * dl * a->m2;
  a->m2 += t1;
}

void orc_moments_merge(orc_moments* a, const orc_moments* b) {
  if (b->n == 0) return;
  if (a->n == 0) {
    *a = *b;
    return;
  }
  const double na = (double)a->n, nb = (double)b->n;
  const double n = na + nb;
  const double d = b->mean - a->mean;
  const double d2 = d * d;
  const double m2 = a->m2 + b->m2 + d2 * na * nb / n;
  const double m3 = a->m3 + b->m3 + d2 * d * na * nb * (na - nb) / (n * n) +
                    3.0 * d * (na * b->m2 - nb * a->m2) / n;
  const double m4 = a->m4 + b->m4 + d2 * d2 * na * nb * (na * na - na * nb + nb * nb) / (n * n * n) +
                    6.0 * d2 * (na * na * b->m2 + nb * nb * a->m2) / (n * n) +
                    4.0 * d * (na * b->m3 - nb * a->m3) / n;
  a->mean += d * nb / n;
  a->m2 = m2;
  a->m3 = m3;
  a->m4 = m4;
  a->n += b->n;
}

/* ---- reference-order level run: mlmc.hpp:67-111 -------------------------- */

typedef struct seq_job {
  const orc_config* c;
  uint64_t n, base, n_batches;
  int threads, tid;
  orc_moments* batches; /* 3 per batch */
  int* fail;            /* per batch */
  uint64_t* fstep;      /* per batch */
  uint64_t* fpath;      /* per batch (local index) */
} seq_job;

static void diffs(const orc_config* c, const double* r, double* dh, double* db) {
  const double pc_h = c->level == 0 ? 0.0 : payoff(c, r[1]);
  const double pc_b = c->level == 0 ? 0.0 : payoff(c, r[3]);
  *dh = payoff(c, r[0]) - pc_h;
  *db = payoff(c, r[2]) - pc_b;
}

static void* seq_worker(void* arg) {
  seq_job* j = (seq_job*)arg;
  for (uint64_t bi = (uint64_t)j->tid; bi < j->n_batches; bi += (uint64_t)j->threads) {
    orc_moments* acc = j->batches + 3 * bi;
    memset(acc, 0, 3 * sizeof(orc_moments));
    j->fail[bi] = 0;
    const uint64_t end = (bi + 1) * 256 < j->n ? (bi + 1) * 256 : j->n;
    for (uint64_t i = bi * 256; i < end; ++i) {
      double r[4];
      uint64_t st = 0;
      const int f = orc_simulate_coupled(j->c, j->base + i, r, NULL, &st);
      if (f != ORC_OK) {
        j->fail[bi] = f;
        j->fstep[bi] = st;
        j->fpath[bi] = i;
        break;
      }
      double dh, db;
      diffs(j->c, r, &dh, &db);
      if (j->c->legs & 1) orc_moments_add(&acc[0], dh);
      if (j->c->legs & 2) orc_moments_add(&acc[1], db);
      if ((j->c->legs & 3) == 3) orc_moments_add(&acc[2], dh - db);
    }
  }
  return NULL;
}

int orc_run_sequential(const orc_config* c, uint64_t n, uint64_t path_base, int threads,
                       orc_moments* out3, uint64_t* fail_path, uint64_t* fail_step) {
  memset(out3, 0, 3 * sizeof(orc_moments));
  if (n == 0) return ORC_OK;
  if (c->level < 0) return ORC_BAD_ARG;
  const uint64_t nb = (n + 255) / 256;
  orc_moments* batches = (orc_moments*)calloc(3 * nb, sizeof(orc_moments));
  int* fail = (int*)calloc(nb, sizeof(int));
  uint64_t* fstep = (uint64_t*)calloc(nb, sizeof(uint64_t));
  uint64_t* fpath = (uint64_t*)calloc(nb, sizeof(uint64_t));
  if (threads < 1) threads = 1;
  if ((uint64_t)threads > nb) threads = (int)nb;
  seq_job* jobs = (seq_job*)calloc((size_t)threads, sizeof(seq_job));
  pthread_t* th = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
  for (int t = 0; t < threads; ++t) {
    jobs[t] = (seq_job){c, n, path_base, nb, threads, t, batches, fail, fstep, fpath};
    if (threads == 1) {
      seq_worker(&jobs[t]);
    } else {
      pthread_create(&th[t], NULL, seq_worker, &jobs[t]);
    }
  }
  if (threads > 1)
    for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
  int rc = ORC_OK;
  for (uint64_t b = 0; b < nb; ++b) {
    if (fail[b]) {
      rc = fail[b];
      *fail_path = path_base + fpath[b];
      *fail_step = fstep[b];
      break;
    }
    for (int k = 0; k < 3; ++k) orc_moments_merge(&out3[k], &batches[3 * b + k]);
  }
  free(batches);
  free(fail);
  free(fstep);
  free(fpath);
  free(jobs);
  free(th);
  return rc;
}

/* ---- restated device reduction tree (paper_2012_09739_b200/csrc) -------- */

/* xor-butterfly over 32 lanes (warp shuffle), result in every lane. */
static double butterfly32(double* v, int first_k) {
  double tmp[32];
  for (int k = first_k; k >= 1; k >>= 1) {
    for (int l = 0; l < 32; ++l) tmp[l] = v[l] + v[l ^ k];
    memcpy(v, tmp, sizeof tmp);
  }
  return v[0];
}

/* batch of c <= 256 values -> {c, mean, S2, S3, S4} */
static void batch_acc(const double* x, int c, orc_moments* out) {
  double grp[8];
  double lanes[32];
  for (int g = 0; g < 8; ++g) {
    for (int l = 0; l < 32; ++l) {
      const int s = 32 * g + l;
      lanes[l] = s < c ? x[s] : 0.0;
    }
    grp[g] = butterfly32(lanes, 16);
  }
  for (int l = 0; l < 32; ++l) lanes[l] = l < 8 ? grp[l] : 0.0;
  const double s1 = butterfly32(lanes, 4);
  const double mean = s1 / (double)c;
  double sums[3];
  for (int p = 0; p < 3; ++p) {
    for (int g = 0; g < 8; ++g) {
      for (int l = 0; l < 32; ++l) {
        const int s = 32 * g + l;
        const double d = s < c ? x[s] - mean : 0.0;
        const double d2 = d * d;
        lanes[l] = p == 0 ? d2 : (p == 1 ? d2 * d : d2 * d2);
      }
      grp[g] = butterfly32(lanes, 16);
    }
    for (int l = 0; l < 32; ++l) lanes[l] = l < 8 ? grp[l] : 0.0;
    sums[p] = butterfly32(lanes, 4);
  }
  out->n = (uint64_t)c;
  out->mean = mean;
  out->m2 = sums[0];
  out->m3 = sums[1];
  out->m4 = sums[2];
}

void orc_tree_from_values(const double* d_hat, const double* d_bar, uint64_t n, unsigned legs,
                          orc_moments* out3) {
  memset(out3, 0, 3 * sizeof(orc_moments));
  const uint64_t n_batches = (n + 255) / 256;
  const uint64_t n_chunks = (n_batches + 1023) / 1024;
  orc_moments* slots = (orc_moments*)malloc(3 * 1024 * sizeof(orc_moments));
  double* four = (double*)malloc(256 * sizeof(double));
  for (uint64_t ch = 0; ch < n_chunks; ++ch) {
    memset(slots, 0, 3 * 1024 * sizeof(orc_moments));
    for (uint64_t bl = 0; bl < 1024; ++bl) {
      const uint64_t b = ch * 1024 + bl;
      if (b >= n_batches) break;
      const uint64_t p0 = b * 256;
      const int c = (int)(n - p0 < 256 ? n - p0 : 256);
      for (int i = 0; i < c; ++i) four[i] = d_hat[p0 + i] - d_bar[p0 + i];
      batch_acc(d_hat + p0, c, &slots[0 * 1024 + bl]);
      batch_acc(d_bar + p0, c, &slots[1 * 1024 + bl]);
      batch_acc(four, c, &slots[2 * 1024 + bl]);
    }
    for (int k = 0; k < 3; ++k) {
      orc_moments* s = slots + k * 1024;
      for (int width = 512; width >= 1; width >>= 1) {
        for (int i = 0; i < width; ++i) {
          orc_moments a = s[2 * i];
          orc_moments_merge(&a, &s[2 * i + 1]);
          s[i] = a;
        }
      }
      orc_moments_merge(&out3[k], &s[0]);
    }
  }
  if (!(legs & 1)) memset(&out3[0], 0, sizeof(orc_moments));
  if (!(legs & 2)) memset(&out3[1], 0, sizeof(orc_moments));
  if ((legs & 3) != 3) memset(&out3[2], 0, sizeof(orc_moments));
  free(slots);
  free(four);
}

int orc_run_tree(const orc_config* c, uint64_t n, uint64_t path_base, orc_moments* out3,
                 uint64_t* fail_path, uint64_t* fail_step) {
  memset(out3, 0, 3 * sizeof(orc_moments));
  if (n == 0) return ORC_OK;
  double* dh = (double*)malloc(n * sizeof(double));
  double* db = (double*)malloc(n * sizeof(double));
  int rc = ORC_OK;
  for (uint64_t i = 0; i < n; ++i) {
    double r[4];
    uint64_t st = 0;
    const int f = orc_simulate_coupled(c, path_base + i, r, NULL, &st);
    if (f != ORC_OK) {
      rc = f;
      *fail_path = path_base + i;
      *fail_step = st;
      break;
    }
    double h = 0.0, b = 0.0;
    diffs(c, r, &h, &b);
    dh[i] = (c->legs & 1) ? h : 0.0;
    db[i] = (c->legs & 2) ? b : 0.0;
  }
  if (rc == ORC_OK) orc_tree_from_values(dh, db, n, c->legs, out3);
  free(dh);
  free(db);
  return rc;
}

/* ---- replay of the carrier ("hat") legs from given Gaussians ------------ */
/* sde.hpp:241, :260-262, :270-272 with z[0..2^l) supplied (e.g. the device's
 * own exact Gaussians), so hat legs can be compared bit for bit even though
 * glibc and libdevice erfc/exp/log differ in the last ulp. */
int orc_replay_hat(const orc_config* c, const double* z, double* out2) {
  if (c->level < 0) return ORC_BAD_ARG;
  const uint64_t n_fine = (uint64_t)1 << c->level;
  const double dtf = ldexp(c->horizon, -c->level);
  const double sdtf = sqrt(dtf);
  const double dtc = 2.0 * dtf;
  leg_ops hi = {52, 0, 0};
  double xf = c->x0, xc = c->x0;
  if (c->level == 0) {
    xf = accumulate(&hi, 0, NULL, xf, inc_fine(&hi, c->mu, c->sigma, xf, dtf, sdtf, z[0]));
    out2[0] = xf;
    out2[1] = 0.0;
    return hi.fail ? ORC_FAIL_NONFINITE : ORC_OK;
  }
  for (uint64_t m = 0; m < n_fine / 2; ++m) {
    const double z0 = z[2 * m], z1 = z[2 * m + 1];
    xf = accumulate(&hi, 0, NULL, xf, inc_fine(&hi, c->mu, c->sigma, xf, dtf, sdtf, z0));
    xf = accumulate(&hi, 0, NULL, xf, inc_fine(&hi, c->mu, c->sigma, xf, dtf, sdtf, z1));
    const double dwc = sdtf * z0 + sdtf * z1;
    xc = accumulate(&hi, 0, NULL, xc, inc_coarse(&hi, c->mu, c->sigma, xc, dtc, dwc));
  }
  out2[0] = xf;
  out2[1] = xc;
  return hi.fail ? ORC_FAIL_NONFINITE : ORC_OK;
}

/* Reference-order accumulation (mlmc.hpp:78-110) of given per-path diffs. */
void orc_sequential_from_values(const double* d_hat, const double* d_bar, uint64_t n,
                                orc_moments* out3) {
  memset(out3, 0, 3 * sizeof(orc_moments));
  for (uint64_t b0 = 0; b0 < n; b0 += 256) {
    orc_moments acc[3];
    memset(acc, 0, sizeof acc);
    const uint64_t end = b0 + 256 < n ? b0 + 256 : n;
    for (uint64_t i = b0; i < end; ++i) {
      orc_moments_add(&acc[0], d_hat[i]);
      orc_moments_add(&acc[1], d_bar[i]);
      orc_moments_add(&acc[2], d_hat[i] - d_bar[i]);
    }
    for (int k = 0; k < 3; ++k) orc_moments_merge(&out3[k], &acc[k]);
  }
}

/* Per-path differences (mlmc.hpp:86-90, payoff applied) for paths
 * path_base .. path_base+n-1; legs not simulated give 0.  Returns the first
 * failure kind (0 if none). */
int orc_diffs(const orc_config* c, uint64_t path_base, uint64_t n, double* d_hat, double* d_bar) {
  for (uint64_t i = 0; i < n; ++i) {
    double r[4];
    uint64_t st = 0;
    const int f = orc_simulate_coupled(c, path_base + i, r, NULL, &st);
    if (f != ORC_OK) return f;
    double h, b;
    diffs(c, r, &h, &b);
    d_hat[i] = (c->legs & 1) ? h : 0.0;
    d_bar[i] = (c->legs & 2) ? b : 0.0;
  }
  return ORC_OK;
}
