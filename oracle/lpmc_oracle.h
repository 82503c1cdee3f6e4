/*
 * TEST INFRASTRUCTURE ONLY — the CPU oracle for the B200 level sampler.
 *
 * A plain-C restatement of the reference's hot path (/root/reference/proj/
 * include/lpmc/{uniform,gaussian,softfloat,invcdf_approx,sde,stats,mlmc}.hpp),
 * every function citing the reference file:line it follows, plus the
 * extensions the BASELINE configs need and the reference lacks (constant:K
 * tables, call payoff, IEEE-binary16 legs, legs mask) and a restatement of the
 * device library's fixed reduction tree.  Pinned against the unmodified
 * reference (oracle/_ref) and the committed golden vectors (tests/golden/).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * reference legs may load this; the product library never does.
 */
#ifndef LPMC_ORACLE_H_
#define LPMC_ORACLE_H_

#include <stdint.h>

typedef struct orc_table {
  int kind; /* 0 linear, 1 cubic, 2 constant */
  int K;
  double w_max, step_w, tail;
  const double* bp;    /* K */
  const double* coeff; /* 4K */
} orc_table;

typedef struct orc_config {
  double mu, sigma, x0, horizon;
  int level;
  int mantissa_bits;
  int ieee_half;
  const orc_table* table; /* NULL = exact inverse CDF for the bar legs */
  int kahan;
  uint64_t seed;
  unsigned legs; /* 1 hat, 2 bar, 3 all */
  int payoff;    /* 0 terminal, 1 call */
  double strike;
} orc_config;

typedef struct orc_moments {
  uint64_t n;
  double mean, m2, m3, m4;
} orc_moments;

/* failure kinds (same numbering as lpmc_fail_kind) */
enum { ORC_OK = 0, ORC_FAIL_U1 = 1, ORC_FAIL_NONFINITE = 2, ORC_FAIL_STATE = 3, ORC_BAD_ARG = 4 };

uint64_t orc_mix64(uint64_t z);
uint64_t orc_stream_word(uint64_t seed, uint64_t path, uint64_t ctr);
double orc_uniform(uint64_t seed, uint64_t path, uint64_t ctr);
int orc_exact_inv_cdf(double u, double* z);
int orc_round(double x, int m, double* out);
int orc_table_build(int kind, int K, double* bp, double* coeff, double* w_max, double* step_w,
                    double* tail);
int orc_approx_eval(const orc_table* t, double u, double* z);
/* double -> IEEE binary16 -> double (single rounding) */
double orc_to_half(double x);

int orc_simulate_coupled(const orc_config* c, uint64_t path, double* out4, double* z_out,
                         uint64_t* fail_step);
int orc_simulate_coupled_z(const orc_config* c, uint64_t path, const double* z_in, double* out4,
                           double* z_out, uint64_t* fail_step);
void orc_moments_add(orc_moments* a, double x);
void orc_moments_merge(orc_moments* a, const orc_moments* b);

/* Reference-order run (mlmc.hpp:67-111). fail_path = global path index. */
int orc_run_sequential(const orc_config* c, uint64_t n, uint64_t path_base, int threads,
                       orc_moments* out3, uint64_t* fail_path, uint64_t* fail_step);
/* The device library's tree (batches -> chunks -> index-order fold). */
void orc_tree_from_values(const double* d_hat, const double* d_bar, uint64_t n, unsigned legs,
                          orc_moments* out3);
int orc_run_tree(const orc_config* c, uint64_t n, uint64_t path_base, orc_moments* out3,
                 uint64_t* fail_path, uint64_t* fail_step);



int orc_replay_hat(const orc_config* c, const double* z, double* out2);
void orc_sequential_from_values(const double* d_hat, const double* d_bar, uint64_t n,
                                orc_moments* out3);
int orc_diffs(const orc_config* c, uint64_t path_base, uint64_t n, double* d_hat, double* d_bar);
#endif
