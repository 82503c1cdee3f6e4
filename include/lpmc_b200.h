/*
 * lpmc_b200.h — C-ABI of the B200-native MLMC level-correction sampler.
 *
 * This is the drop-in boundary under the reference's level-sampling entry
 * points (reference: /root/reference/proj/include/lpmc/mlmc.hpp).  Plain C
 * types only: pointers, sizes and PODs; no CUDA or C++ types in signatures.
 * The C++ headers in include/lpmc/ (the reference-compatible API) and the
 * Python package paper_2012_09739_b200 both bind to exactly these symbols.
 *
 * Replaced reference interfaces (file:line under /root/reference/proj):
 *   lpmc_run_coupled_paths      <- run_coupled_paths       include/lpmc/mlmc.hpp:67-111
 *   lpmc_estimate_level_stats   <- estimate_level_stats    include/lpmc/mlmc.hpp:113-149
 *   lpmc_simulate_paths         <- simulate_coupled        include/lpmc/sde.hpp:211-284
 *                                  (batched per-path dump, for parity only)
 *   lpmc_invcdf_build           <- InvCdfApprox::build     include/lpmc/invcdf_approx.hpp:101-145
 *   lpmc_invcdf_eval            <- InvCdfApprox::operator() include/lpmc/invcdf_approx.hpp:44-50
 *   lpmc_round_to_precision     <- round_to_precision      include/lpmc/softfloat.hpp:69-80
 *   lpmc_moments_add / _merge   <- MomentAccumulator::add / merge  include/lpmc/stats.hpp:15-54
 *   lpmc_level_partials +       <- the batch loop + index-order merge of
 *   lpmc_fold_partials             run_coupled_paths (mlmc.hpp:74-110), split
 *                                  so paths can be sharded over GPUs/ranks
 *   lpmc_run_coupled_many       <- a loop of run_coupled_paths calls (the
 *                                  callers: mlmc.hpp:254-278,
 *                                  experiments.hpp:126-143, :185-194), run
 *                                  concurrently on one device
 *   lpmc_run_two_way_paths      <- run_batched(simulate_two_way) (experiments.hpp:136-141,
 *                                  sde.hpp:162-196)
 *   lpmc_allocate_samples       <- allocate_samples        include/lpmc/mlmc.hpp:165-195
 *   lpmc_predicted_times        <- predicted_times         include/lpmc/mlmc.hpp:202-213
 *   lpmc_per_level_speedup      <- per_level_speedup       include/lpmc/mlmc.hpp:223-230
 *   lpmc_run_nested_estimator   <- run_nested_estimator    include/lpmc/mlmc.hpp:244-283
 *   lpmc_step_error_probe       <- step_error_probe        include/lpmc/sde.hpp:297-344
 *   lpmc_density_histogram      <- the histogram loop of run_density_report
 *                                  include/lpmc/experiments.hpp:276-285
 * Diagnostics without a reference counterpart: lpmc_bar_arithmetic (which
 * arithmetic a run's low-precision legs use: native fp32 / bfloat16 /
 * binary16, fp32- or binary64-carried rounding -- all bitwise
 * softfloat.hpp:69-111), lpmc_device_math, lpmc_erfc_core,
 * lpmc_phi_inv_direct_core, lpmc_glibc_math, lpmc_measure_pipe_peaks.
 *
 * Error contract: every entry point returns an lpmc_status.  The values map
 * one-to-one onto the exception types the reference throws
 * (std::invalid_argument, std::domain_error, std::runtime_error); the
 * message text in lpmc_error.message is the reference's what() string.
 * LPMC_CUDA_ERROR / LPMC_NO_DEVICE have no reference counterpart: there is no
 * CPU fallback, a device failure is reported, never papered over.
 */
#ifndef LPMC_B200_H_
#define LPMC_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LPMC_B200_ABI_VERSION 3

typedef enum lpmc_status {
  LPMC_OK = 0,
  LPMC_INVALID_ARGUMENT = 1, /* std::invalid_argument */
  LPMC_DOMAIN_ERROR = 2,     /* std::domain_error     */
  LPMC_RUNTIME_ERROR = 3,    /* std::runtime_error    */
  LPMC_CUDA_ERROR = 4,       /* device/driver failure */
  LPMC_NO_DEVICE = 5         /* no usable sm_100 device */
} lpmc_status;

/* Which first failure a path hit (lpmc_error.kind). */
typedef enum lpmc_fail_kind {
  LPMC_FAIL_NONE = 0,
  LPMC_FAIL_UNIFORM_IS_ONE = 1, /* u == 1.0 reached exact_inv_cdf (gaussian.hpp:60-61) */
  LPMC_FAIL_NONFINITE = 2,      /* non-finite operand (softfloat.hpp:70)               */
  LPMC_FAIL_NONFINITE_STATE = 3 /* IEEE-half legs only: non-finite state (sde.hpp:120)  */
} lpmc_fail_kind;

typedef struct lpmc_error {
  int32_t status;      /* lpmc_status */
  int32_t kind;        /* lpmc_fail_kind, for sampler failures */
  uint64_t path_index; /* global path index (path_base + i) of the first failing path */
  uint64_t step;       /* fine step index of the first failure in that path */
  char message[192];   /* reference what() text, or a CUDA error string */
} lpmc_error;

/* GBM dS = mu S dt + sigma S dW on [0, horizon] (make_gbm, sde.hpp:32-44). */
typedef struct lpmc_gbm {
  double mu, sigma, x0, horizon;
} lpmc_gbm;

typedef enum lpmc_approx_kind {
  LPMC_APPROX_LINEAR = 0,  /* InvCdfApprox::Kind::linear */
  LPMC_APPROX_CUBIC = 1,   /* InvCdfApprox::Kind::cubic  */
  LPMC_APPROX_CONSTANT = 2 /* extension (BASELINE config 3): degree-0 Legendre projection */
} lpmc_approx_kind;

/*
 * Host copy of an InvCdfApprox table (invcdf_approx.hpp:92-98).  The device
 * layout is private; the library uploads what it needs per call.
 */
typedef struct lpmc_invcdf_table {
  int32_t kind;           /* lpmc_approx_kind */
  int32_t interval_count; /* K, a power of two >= 2 */
  double w_max;
  double step_w;
  double tail_value;
  const double* breakpoints; /* K ascending interior breakpoints in (1/2, 1) */
  const double* coeff;       /* K x 4 Legendre coefficients, row-major */
} lpmc_invcdf_table;

/*
 * Arithmetic of the low-precision ("bar") legs.  mantissa_bits follows
 * PrecisionSpec (softfloat.hpp:18-64): 1..51 = emulated round-to-nearest-even
 * with an unbounded exponent, >= 52 = the binary64 carrier.  ieee_half = 1
 * selects native IEEE binary16 legs (BASELINE config 3; requires
 * mantissa_bits == 10): subnormals and the 65504 overflow are IEEE, so these
 * legs are pinned against an IEEE restatement, not the emulated reference.
 */
typedef struct lpmc_precision {
  int32_t mantissa_bits;
  int32_t ieee_half;
} lpmc_precision;

enum {
  LPMC_LEGS_HAT = 1, /* carrier legs, exact Gaussians: d_hat only */
  LPMC_LEGS_BAR = 2, /* low-precision legs: d_bar only            */
  LPMC_LEGS_ALL = 3, /* all four legs (the reference always runs these) */
  /*
   * Fine legs only = simulate_two_way (sde.hpp:162-196): the carrier and
   * the low-precision path at the same level, no coarse legs.  The three
   * accumulators then hold x_hat, x_bar and x_hat - x_bar (the two-way
   * experiment's quantity, experiments.hpp:136-141).
   */
  LPMC_LEGS_FINE = 4
};

enum {
  LPMC_PAYOFF_TERMINAL = 0, /* P(S) = S_T (the reference's quantity) */
  LPMC_PAYOFF_CALL = 1      /* extension (config 4): max(S_T - strike, 0) in fp64 */
};

enum {
  LPMC_REDUCE_TREE = 0,      /* fixed two-pass/Pebay tree; GPU-count independent */
  LPMC_REDUCE_SEQUENTIAL = 1 /* the reference's own add/merge order, bitwise */
};

/*
 * Exact Gaussians (gaussian.hpp:14-65: Acklam + one Newton step on glibc's
 * erfc/exp/log).  FAST restates the algorithm for the B200 issue budget (own
 * erfc/exp, MUFU-seeded divisions): Z within a few ulp of the reference's.
 * GLIBC restates the reference's own operation sequence and glibc 2.39's
 * erfc/exp/log bit for bit (lpmc_glibc.cuh): Z, hat legs and moments equal
 * the reference's bitwise, at a lower throughput.
 */
enum {
  LPMC_EXACT_Z_FAST = 0,
  LPMC_EXACT_Z_GLIBC = 1
};

/*
 * Kernel schedule of a run (results are bitwise the same either way).
 * FUSED: one thread per path, 256-path CTAs (throughput).  WARP_PER_PATH:
 * one warp per path, 32 steps' Gaussians drawn in parallel, then the legs
 * stepped by the warp (latency: runs with too few paths to fill the GPU).
 * AUTO picks WARP_PER_PATH for runs of at most 6144 paths at levels >= 5
 * (the fused grid would leave most SMs idle); never for the IEEE half2 legs
 * (two paths per thread).
 */
enum {
  LPMC_SCHEDULE_AUTO = 0,
  LPMC_SCHEDULE_FUSED = 1,
  LPMC_SCHEDULE_WARP_PER_PATH = 2
};

typedef struct lpmc_options {
  uint32_t legs;  /* LPMC_LEGS_*; 0 means LPMC_LEGS_ALL */
  int32_t payoff; /* LPMC_PAYOFF_* */
  double strike;  /* for LPMC_PAYOFF_CALL */
  int32_t reduce; /* LPMC_REDUCE_* */
  int32_t device; /* CUDA ordinal; -1 = current device */
  void* stream;   /* cudaStream_t to launch on; NULL = the library's stream */
  int32_t exact_z; /* LPMC_EXACT_Z_* */
  /*
   * Devices of one process to shard each run over (NULL / n_devices <= 1:
   * the single device above).  Runs split into contiguous 2^18-path chunk
   * ranges, one per listed device (a device may repeat), launched
   * concurrently; the partials are folded in chunk order, so results are
   * bitwise those of one device.  Multi-device calls are synchronous and
   * ignore `stream`.
   */
  const int32_t* devices;
  int32_t n_devices;
  int32_t schedule; /* LPMC_SCHEDULE_* */
  /*
   * First counter of every path's uniform stream (UniformStream(seed, path,
   * counter), uniform.hpp:31-36); 0 everywhere in the reference's own
   * callers (mlmc.hpp:83).  Lets a per-path call resume a stream.
   */
  uint64_t counter;
} lpmc_options;

/* Raw MomentAccumulator state (stats.hpp:84-89). */
typedef struct lpmc_moments {
  uint64_t n;
  double mean, m2, m3, m4;
} lpmc_moments;

/* CostModel (mlmc.hpp:20-34). */
typedef struct lpmc_cost_model {
  double cycles_exact_rng;
  double cycles_approx_rng_single;
  double cycles_approx_rng_half;
  double kahan_overhead_factor;
  double per_step_arithmetic;
} lpmc_cost_model;

/* LevelStats (mlmc.hpp:36-51). */
typedef struct lpmc_level_stats {
  int32_t level;
  double mean_hat, v_hat, v_hat_stderr;
  double mean_bar, v_bar, v_bar_stderr;
  double mean_four, V_bar, V_bar_stderr;
  double c_hat, c_bar, C_bar;
  uint64_t m_hat, m_bar, M_bar;
} lpmc_level_stats;

/* Paths per reduction batch and batches per chunk (the fixed merge tree). */
#define LPMC_BATCH_PATHS 256u
#define LPMC_CHUNK_BATCHES 1024u
#define LPMC_CHUNK_PATHS (LPMC_BATCH_PATHS * LPMC_CHUNK_BATCHES)

/* ---- version / device ---------------------------------------------------- */
int32_t lpmc_abi_version(void);
/* Number of visible sm_100 devices (0 on a CPU-only host). */
int32_t lpmc_device_count(void);
/* Kernel launches issued by this thread since the last reset (bench evidence). */
uint64_t lpmc_launch_count(void);
void lpmc_reset_launch_count(void);
void lpmc_default_options(lpmc_options* opts);
void lpmc_default_cost_model(lpmc_cost_model* cost);

/* ---- host-side numerics (no GPU needed) --------------------------------- */
/* round_to_precision (softfloat.hpp:69-80). */
lpmc_status lpmc_round_to_precision(double x, int32_t mantissa_bits, double* out, lpmc_error* err);
/*
 * InvCdfApprox::build (invcdf_approx.hpp:101-145), same operation order, so
 * the table is bitwise the reference's.  breakpoints: K doubles; coeff: 4K.
 */
lpmc_status lpmc_invcdf_build(int32_t kind, int32_t interval_count, double* breakpoints,
                              double* coeff, double* w_max, double* step_w, double* tail_value,
                              lpmc_error* err);
/* InvCdfApprox::operator() on the host (invcdf_approx.hpp:44-90). */
lpmc_status lpmc_invcdf_eval(const lpmc_invcdf_table* table, double u, double* out,
                             lpmc_error* err);
/* MomentAccumulator::add / merge (stats.hpp:15-54), bitwise. */
void lpmc_moments_add(lpmc_moments* acc, double x);
void lpmc_moments_merge(lpmc_moments* acc, const lpmc_moments* other);
/*
 * Index-order fold of per-chunk partials (3 per chunk: d_hat, d_bar, d_four),
 * the run_coupled_paths merge (mlmc.hpp:108-110).  out: 3 accumulators.
 */
void lpmc_fold_partials(const lpmc_moments* partials, uint64_t n_chunks, lpmc_moments* out);
/* LevelStats from three accumulators + the cost model (mlmc.hpp:125-148). */
void lpmc_level_stats_from_moments(const lpmc_moments* acc3, int32_t level,
                                   const lpmc_precision* prec, int32_t kahan,
                                   const lpmc_cost_model* cost, uint64_t n_paths,
                                   lpmc_level_stats* out);

/* ---- device sampler ------------------------------------------------------ */
/*
 * run_coupled_paths (mlmc.hpp:67-111): n_paths coupled fine/coarse x
 * exact/approx paths at `level`; table == NULL selects the exact inverse CDF
 * for the bar legs.  out: 3 accumulators (d_hat, d_bar, d_four).
 */
lpmc_status lpmc_run_coupled_paths(const lpmc_gbm* model, int32_t level,
                                   const lpmc_precision* prec, const lpmc_invcdf_table* table,
                                   int32_t kahan, uint64_t n_paths, uint64_t seed,
                                   uint64_t path_base, const lpmc_options* opts,
                                   lpmc_moments* out, lpmc_error* err);

/* estimate_level_stats (mlmc.hpp:113-149).  cost may be NULL (defaults). */
lpmc_status lpmc_estimate_level_stats(const lpmc_gbm* model, int32_t level,
                                      const lpmc_precision* prec,
                                      const lpmc_invcdf_table* table, int32_t kahan,
                                      uint64_t n_paths, uint64_t seed,
                                      const lpmc_cost_model* cost, uint64_t path_base,
                                      const lpmc_options* opts, lpmc_level_stats* out,
                                      lpmc_error* err);

/*
 * Shard entry point: chunk accumulators for chunks [chunk_begin, chunk_end)
 * of an n_paths run (chunk c = paths [c*LPMC_CHUNK_PATHS, ...) relative to
 * path_base).  out: 3*(chunk_end-chunk_begin) accumulators, chunk-major.
 * Folding every rank's chunks with lpmc_fold_partials in chunk order gives
 * the same bits as lpmc_run_coupled_paths for any number of ranks.
 */
lpmc_status lpmc_level_partials(const lpmc_gbm* model, int32_t level,
                                const lpmc_precision* prec, const lpmc_invcdf_table* table,
                                int32_t kahan, uint64_t n_paths, uint64_t seed,
                                uint64_t path_base, uint64_t chunk_begin, uint64_t chunk_end,
                                const lpmc_options* opts, lpmc_moments* out, lpmc_error* err);

/*
 * Per-path dump for parity tests: out4 = n x {x_hat_fine, x_hat_coarse,
 * x_bar_fine, x_bar_coarse} as simulate_coupled returns them (sde.hpp:279-283),
 * host memory.  z_out (optional, n x 2^level) receives the exact Gaussians
 * the hat legs consumed, so the CPU can replay those legs bit for bit.
 */
lpmc_status lpmc_simulate_paths(const lpmc_gbm* model, int32_t level, const lpmc_precision* prec,
                                const lpmc_invcdf_table* table, int32_t kahan, uint64_t n_paths,
                                uint64_t seed, uint64_t path_base, const lpmc_options* opts,
                                double* out4, double* z_out, lpmc_error* err);

/*
 * Exact Gaussians / approximate Gaussians for host-provided uniforms, on the
 * device (the kernels' own device functions; parity tests of a2/a3); exact
 * Gaussians in the mode opts->exact_z selects.
 */
lpmc_status lpmc_device_inv_cdf(const double* u, uint64_t n, const lpmc_invcdf_table* table,
                                double* out, const lpmc_options* opts, lpmc_error* err);

/*
 * Measured lane-operation rates of the current B200 (roofline denominators
 * for this non-tensor path): out4 = {fp64 FMA, fp32 FMA, fp16 (per half lane,
 * HFMA2), 64-bit integer multiply-add} operations per second.
 */
lpmc_status lpmc_measure_pipe_peaks(int32_t device, double* out4, lpmc_error* err);

/*
 * Diagnostics of the device math on host-given inputs: op 0 = exact inverse
 * CDF (the sampler's), 1 = approximate inverse CDF (table required), 2 = the
 * reference's Acklam+Newton formula on CUDA libdevice, 3 = erfc core on
 * t in [0, 6.5), 5 = exact inverse CDF in LPMC_EXACT_Z_GLIBC mode.
 */
lpmc_status lpmc_device_math(int32_t op, const double* in, uint64_t n,
                             const lpmc_invcdf_table* table, double* out,
                             const lpmc_options* opts, lpmc_error* err);
/*
 * Which arithmetic the production launch of a run uses for the low-precision
 * legs (a host decision, no device needed): the low byte is 0 carrier
 * (binary64), 1 native fp32, 2 fp32-carried rounding to m+1 bits, 3 binary64
 * with integer rounding, 4 IEEE binary16 pairs; LPMC_ARITH_POW2_FOLDED: power-
 * of-two steps folded into the model constants; LPMC_ARITH_NATIVE_BINARY16:
 * the m = 10 legs run on native binary16 with static scales (paths that leave
 * its guard are replayed in arithmetic 2); LPMC_ARITH_NATIVE_BFLOAT16: the
 * m = 7 legs run on native bfloat16.  All of them are bitwise the
 * reference's softfloat.hpp:69-111 semantics; the choice only affects speed.
 */
#define LPMC_ARITH_POW2_FOLDED 0x100
#define LPMC_ARITH_NATIVE_BINARY16 0x200
#define LPMC_ARITH_NATIVE_BFLOAT16 0x400 /* the m = 7 legs on native bfloat16 */
lpmc_status lpmc_bar_arithmetic(const lpmc_gbm* model, int32_t level, const lpmc_precision* prec,
                                const lpmc_invcdf_table* table, int32_t kahan,
                                const lpmc_options* opts, int32_t* out, lpmc_error* err);
/* Host evaluation of the same erfc core (bitwise equal to op 3). */
double lpmc_erfc_core(double t);
/*
 * Host evaluation of the direct table behind op 0 (the default exact inverse
 * CDF, gaussian.hpp:59-65 to 0.42 eps (v / pdf(z) + |z|)): Phi^-1(v) for
 * v = min(u, 1 - u) in [2^-15, 1/2], bitwise the device's value.
 * *in_table = 0 (and NaN returned) for v outside that range, where the device
 * takes the Halley step on the erfc core instead.
 */
double lpmc_phi_inv_direct_core(double v, int32_t* in_table);
/*
 * Host evaluation of the restated glibc routines behind the reference's exact
 * Gaussian (the LPMC_EXACT_Z_GLIBC device path, same code): op 0 = exp,
 * 1 = log, 2 = erfc, 3 = exact_inv_cdf (gaussian.hpp:59-65).  *ok = 0 where
 * the argument is outside the restated ranges.
 */
double lpmc_glibc_math(int32_t op, double x, int32_t* ok);

/* ---- host scheme utilities of the reference API ----------------------------
 * The reference's header-only helpers around the sampler, computed by the
 * library on the host with the reference's expression trees (bitwise the
 * reference's on the same libm):
 *   lpmc_stream_word / _uniform  <- detail::stream_word, UniformStream::next
 *                                   include/lpmc/uniform.hpp:22-41
 *   lpmc_normal_cdf / _pdf       <- normal_cdf, normal_pdf   gaussian.hpp:14-20
 *   lpmc_exact_inv_cdf           <- exact_inv_cdf            gaussian.hpp:59-65
 *   lpmc_inv_cdf_lower           <- detail::inv_cdf_lower    gaussian.hpp:26-55
 *   lpmc_gauss_legendre          <- gauss_legendre           quadrature.hpp:17-41
 *   lpmc_ulp_spacing             <- ulp_spacing              softfloat.hpp:129-136
 *   lpmc_moment_diagnostics      <- moment_diagnostics       invcdf_approx.hpp:150-185
 */
uint64_t lpmc_stream_word(uint64_t seed, uint64_t path_index, uint64_t counter);
double lpmc_stream_uniform(uint64_t seed, uint64_t path_index, uint64_t counter);
double lpmc_normal_cdf(double x);
double lpmc_normal_pdf(double x);
lpmc_status lpmc_exact_inv_cdf(double u, double* out, lpmc_error* err);
double lpmc_inv_cdf_lower(double u);
/* nodes, weights: n doubles each */
lpmc_status lpmc_gauss_legendre(int32_t n, double* nodes, double* weights, lpmc_error* err);
lpmc_status lpmc_ulp_spacing(double x, int32_t mantissa_bits, double* out, lpmc_error* err);
/* out: E[Z^p], p = 1..p_max (p_max in [1, 8]) */
lpmc_status lpmc_moment_diagnostics(const lpmc_invcdf_table* table, int32_t p_max, double* out,
                                    lpmc_error* err);

/* ---- callers of the level sampler (mlmc.hpp:151-285) --------------------- */
/* One run of a multi-run call. */
typedef struct lpmc_run_desc {
  int32_t level;
  lpmc_precision prec;
  int32_t kahan;
  uint64_t n_paths;
  uint64_t path_base;
} lpmc_run_desc;

/*
 * n_runs run_coupled_paths calls sharing model, table, seed and options,
 * executed concurrently on one device (one stream per run, up to 16 in
 * flight; small levels overlap instead of serialising behind host syncs).
 * out: 3 accumulators per run, run-major.  Results are exactly those of the
 * separate calls; the first failing run in list order is reported, as a
 * serial loop would throw it.  opts->stream, if set, is waited on before
 * the runs start.  Blocking.
 */
lpmc_status lpmc_run_coupled_many(const lpmc_gbm* model, const lpmc_invcdf_table* table,
                                  uint64_t seed, const lpmc_run_desc* runs, uint64_t n_runs,
                                  const lpmc_options* opts, lpmc_moments* out, lpmc_error* err);

/*
 * The multi-run call restricted to one chunk range per run (one process per
 * GPU: rank r passes its contiguous chunk shard of every run).  Chunks are
 * LPMC_CHUNK_PATHS paths; run i covers chunks [chunk_begin[i], chunk_end[i]).
 * out: the raw chunk accumulators, run-major, 3 per chunk (d_hat, d_bar,
 * d_four), i.e. sum_i 3 (chunk_end[i] - chunk_begin[i]) entries; fold the
 * gathered ranges of all ranks with lpmc_fold_partials.  Always the tree
 * reduction.  Same concurrency, failure order and blocking as
 * lpmc_run_coupled_many.
 */
lpmc_status lpmc_run_coupled_many_partials(const lpmc_gbm* model, const lpmc_invcdf_table* table,
                                           uint64_t seed, const lpmc_run_desc* runs,
                                           uint64_t n_runs, const uint64_t* chunk_begin,
                                           const uint64_t* chunk_end, const lpmc_options* opts,
                                           lpmc_moments* out, lpmc_error* err);

/*
 * The two-way sampler: MomentAccumulator of x_hat - x_bar over n_paths
 * simulate_two_way paths (sde.hpp:162-196), batched and merged like
 * run_batched (experiments.hpp:89-112).  out: 1 accumulator.
 */
lpmc_status lpmc_run_two_way_paths(const lpmc_gbm* model, int32_t level,
                                   const lpmc_precision* prec, const lpmc_invcdf_table* table,
                                   int32_t kahan, uint64_t n_paths, uint64_t seed,
                                   uint64_t path_base, const lpmc_options* opts,
                                   lpmc_moments* out, lpmc_error* err);

enum { LPMC_ALLOCATION_STANDARD = 0, LPMC_ALLOCATION_NESTED = 1 }; /* AllocationKind */

/*
 * allocate_samples (mlmc.hpp:165-195), bitwise: primary[n_levels];
 * secondary[n_levels] for the nested kind (may be NULL for standard);
 * *degenerate = every variance was zero.
 */
lpmc_status lpmc_allocate_samples(const lpmc_level_stats* stats, uint64_t n_levels, double eps,
                                  int32_t kind, uint64_t* primary, uint64_t* secondary,
                                  int32_t* degenerate, lpmc_error* err);
/* predicted_times (mlmc.hpp:202-213), bitwise. */
lpmc_status lpmc_predicted_times(const lpmc_level_stats* stats, uint64_t n_levels, double eps,
                                 double* t_hat, double* t_bar, lpmc_error* err);
/* per_level_speedup (mlmc.hpp:223-230), bitwise. */
lpmc_status lpmc_per_level_speedup(const lpmc_level_stats* stats, double* value,
                                   int32_t* cost_ratio_only, lpmc_error* err);

/* EstimatorResult (mlmc.hpp:232-239); the arrays are caller-owned with
 * max_level + 1 entries each (any may be NULL). */
typedef struct lpmc_estimator_result {
  double value; /* theta_bar */
  double eps;
  double t_hat, t_bar;  /* predicted_times of the pilot stats */
  int32_t degenerate;   /* Allocation::degenerate */
  double* level_contributions;
  lpmc_level_stats* pilot_stats;
  uint64_t* primary;   /* Allocation::primary */
  uint64_t* secondary; /* Allocation::secondary */
} lpmc_estimator_result;

/*
 * run_nested_estimator (mlmc.hpp:244-283): pilot estimate_level_stats of
 * pilot_paths per level (path base l << 40), nested allocation, then per
 * level a two-way pass (phase 1, primary[l] paths) and a four-way pass
 * (phase 2, secondary[l]); contribution_l = two_way.d_bar.mean() +
 * (four_way.d_hat.mean() - four_way.d_bar.mean()).  Each pass runs all its
 * levels concurrently (lpmc_run_coupled_many).  cost may be NULL.
 */
lpmc_status lpmc_run_nested_estimator(const lpmc_gbm* model, int32_t max_level,
                                      const lpmc_precision* prec,
                                      const lpmc_invcdf_table* table, int32_t kahan, double eps,
                                      uint64_t seed, const lpmc_cost_model* cost,
                                      uint64_t pilot_paths, const lpmc_options* opts,
                                      lpmc_estimator_result* out, lpmc_error* err);

/*
 * The histogram of run_density_report (experiments.hpp:276-285): the draws
 * 0..n_samples-1 of UniformStream(seed, 0) through the table (NULL = exact
 * inverse CDF), binned as b = (int)((z + z_max) / bin_width) clamped to
 * [0, n_bins).  bins: n_bins counts, exact (integer adds).  A draw that
 * rounds to u == 1 fails as the reference's transform throws (error.step =
 * the draw index).
 */
lpmc_status lpmc_density_histogram(const lpmc_invcdf_table* table, uint64_t seed,
                                   uint64_t n_samples, double z_max, double bin_width,
                                   int32_t n_bins, uint64_t* bins, const lpmc_options* opts,
                                   lpmc_error* err);

/* StepErrorStats (sde.hpp:289-295). */
typedef struct lpmc_step_error_stats {
  double mean_eta, mean_abs_eta, mean_eta_prime, mean_abs_eta_prime;
  uint64_t samples;
} lpmc_step_error_stats;

/*
 * step_error_probe (sde.hpp:297-344): per-step rounding residuals eta (outer
 * add) and eta' (inner sum) along the low-precision paths 0, 1, ... of
 * `seed` at `level`, n_samples steps in total (the last path truncated).
 * One path per device thread; the means differ from the reference's single
 * sequential sum only by summation order.  ieee_half is not supported.
 */
lpmc_status lpmc_step_error_probe(const lpmc_gbm* model, int32_t level,
                                  const lpmc_precision* prec, const lpmc_invcdf_table* table,
                                  uint64_t n_samples, uint64_t seed, const lpmc_options* opts,
                                  lpmc_step_error_stats* out, lpmc_error* err);

/* ---- plans: device-resident repeated launches (bench / sweeps) ---------- */
typedef struct lpmc_plan lpmc_plan;

lpmc_status lpmc_plan_create(const lpmc_gbm* model, int32_t level, const lpmc_precision* prec,
                             const lpmc_invcdf_table* table, int32_t kahan, uint64_t n_paths,
                             uint64_t seed, uint64_t path_base, const lpmc_options* opts,
                             lpmc_plan** plan, lpmc_error* err);
/* A plan over chunks [chunk_begin, chunk_end) only (one rank's shard). */
lpmc_status lpmc_plan_create_range(const lpmc_gbm* model, int32_t level,
                                   const lpmc_precision* prec, const lpmc_invcdf_table* table,
                                   int32_t kahan, uint64_t n_paths, uint64_t seed,
                                   uint64_t path_base, uint64_t chunk_begin, uint64_t chunk_end,
                                   const lpmc_options* opts, lpmc_plan** plan, lpmc_error* err);
/* Enqueue the level's kernels on `stream` (NULL = plan's stream); no sync. */
lpmc_status lpmc_plan_launch(lpmc_plan* plan, void* stream, lpmc_error* err);
/* Wait, copy the partials back, fold, and map device failures to errors. */
lpmc_status lpmc_plan_collect(lpmc_plan* plan, lpmc_moments* out, lpmc_error* err);
/* Wait and copy back the raw chunk partials (3 per chunk, chunk-major),
 * unfolded, for a cross-rank gather. */
lpmc_status lpmc_plan_collect_partials(lpmc_plan* plan, lpmc_moments* out, lpmc_error* err);
/* Number of chunks the plan covers. */
uint64_t lpmc_plan_chunk_count(const lpmc_plan* plan);
/* Number of kernels one lpmc_plan_launch enqueues. */
int32_t lpmc_plan_kernels_per_launch(const lpmc_plan* plan);
void lpmc_plan_destroy(lpmc_plan* plan);

#ifdef __cplusplus
} /* extern "C" */
#endif

#endif /* LPMC_B200_H_ */
