/*
 * asyrk_cuda.h — the drop-in C ABI of the B200-native AsyRK hot path.
 *
 * Plain C: pointers, sizes and PODs only (no C++, no torch types); no
 * function throws. Every entry point returns an asyrk_status whose values are
 * the reference's ErrorCode ordinals + 1 (ref/include/asyrk/error.hpp:8-33),
 * so a host wrapper can rethrow asyrk::Error{code, asyrk_last_error()}
 * exactly as the reference does. Device failures map to the closest
 * reference code (see ASYRK_E_* below and DESIGN.md §Errors).
 *
 * Entry points and the reference interface each one replaces:
 *   asyrk_solve_parallel     solve_parallel          ref/include/asyrk/parallel.hpp:52-54
 *                                                    (pybind: ref/bindings/module.cpp:173-200,297-303)
 *   asyrk_rk_solve           rk_solve                ref/include/asyrk/kaczmarz.hpp:108-109
 *                                                    (pybind: ref/bindings/module.cpp:156-171,292-296)
 *   asyrk_sweep_threads      sweep_threads           ref/include/asyrk/parallel.hpp:73-75
 *   asyrk_residuals          residuals               ref/include/asyrk/csr.hpp:89-90
 *   asyrk_power_iteration_lambda_max
 *                            power_iteration_lambda_max  ref/include/asyrk/stats.hpp:46-47
 *   asyrk_compute_stats      compute_stats           ref/include/asyrk/stats.hpp:42 (the
 *                                                    structural fields; ref/src/stats.cpp:52-130;
 *                                                    the dense spectrum: include/asyrk_dense.h)
 *   asyrk_simulate           simulate                ref/include/asyrk/delay_sim.hpp:61-71
 *   asyrk_monte_carlo_ratios monte_carlo_ratios      ref/include/asyrk/delay_sim.hpp:81-88
 *   asyrk_rate_fit           rate_fit                ref/include/asyrk/delay_sim.hpp:95
 *   asyrk_system_*           (new) device-resident CSR + b handle: the
 *                            "device-CSR cache" the reference has no
 *                            equivalent of (SURVEY.md §8b "Ownership").
 *   asyrk_mrhs_*             (new) multi-right-hand-side AsyRK (config 5);
 *                            the reference is single-RHS.
 *
 * Threading: calls are synchronous and blocking (the caller's thread is the
 * coordinator, as in ref/src/parallel.cpp:388-408). A system handle must not
 * be used by two threads at once.
 */
#ifndef ASYRK_CUDA_H
#define ASYRK_CUDA_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ASYRK_ABI_VERSION 2

/* ErrorCode ordinal + 1 (ref/include/asyrk/error.hpp:8-33). */
typedef enum {
    ASYRK_OK = 0,
    ASYRK_E_IndexOutOfRange = 1,
    ASYRK_E_DuplicateEntry = 2,
    ASYRK_E_ZeroRow = 3,
    ASYRK_E_ZeroColumn = 4,
    ASYRK_E_NotNormalized = 5,
    ASYRK_E_DimensionMismatch = 6,
    ASYRK_E_PowerIterationDiverged = 7,
    ASYRK_E_NonFinite = 8,
    ASYRK_E_ComponentNotInSupport = 9,
    ASYRK_E_Inconsistent = 10,
    ASYRK_E_TooLarge = 11,             /* also: device out of memory, index width overflow */
    ASYRK_E_InvalidRho = 12,
    ASYRK_E_MissingStats = 13,
    ASYRK_E_StepTooLarge = 14,
    ASYRK_E_ZeroLambdaMin = 15,
    ASYRK_E_InvalidGamma = 16,
    ASYRK_E_NonPositiveData = 17,
    ASYRK_E_InsufficientData = 18,
    ASYRK_E_NonPositiveSigma = 19,
    ASYRK_E_SigmaUnavailable = 20,
    ASYRK_E_InfeasibleSpec = 21,
    ASYRK_E_ThreadSpawnFailure = 22,   /* also: kernel launch failure / no CUDA device */
    ASYRK_E_IoError = 23,
    ASYRK_E_InvalidArgument = 24,
} asyrk_status;

/* Message of the last failing call on this thread ("" if none). */
const char* asyrk_last_error(void);
int asyrk_abi_version(void);
/* Select the CUDA device for this host thread (one process per GPU). */
asyrk_status asyrk_set_device(int32_t device);

/* Host CSR, the reference CsrMatrix fields (ref/include/asyrk/csr.hpp:69-75).
 * row_norm are the reference's cached norms (csr.cpp:53-61, recomputed by
 * normalize_rows csr.cpp:130-134); they enter the projection coefficient
 * gamma*res/(nrm*nrm) and so must be passed, not assumed to be 1. */
typedef struct {
    int64_t m, n, nnz;
    const int64_t* row_ptr;  /* m+1 */
    const int64_t* col_idx;  /* nnz, strictly increasing within a row */
    const double* values;    /* nnz */
    const double* row_norm;  /* m */
    int32_t normalized;      /* CsrMatrix::is_normalized() */
} asyrk_csr_view;

/* UpdateVariant (kaczmarz.hpp:20) */
enum { ASYRK_SINGLE_COMPONENT = 0, ASYRK_FULL_ROW = 1 };
/* ParSampling (parallel.hpp:14-17) + device extension: norm_proportional
 * (alias table over ||a_i||^2, only Sampling in rk_solve upstream). */
enum { ASYRK_WITH_REPLACEMENT = 0, ASYRK_SLICE_SHUFFLE = 1, ASYRK_NORM_PROPORTIONAL = 2 };
/* Sampling (kaczmarz.hpp:89-93) */
enum { ASYRK_RK_UNIFORM = 0, ASYRK_RK_NORM_PROPORTIONAL = 1, ASYRK_RK_SHUFFLE = 2 };
/* Device precision of the async path (values / x). fp64 is the reference's. */
enum { ASYRK_F64 = 0, ASYRK_F32 = 1, ASYRK_F32_VALUES_F64_X = 2 };

/* RunConfig (parallel.hpp:19-31) plus device extensions. threads maps to
 * concurrent warp-workers; threads == 1 is the deterministic path that
 * consumes the reference's mt19937_64 row sequence. */
typedef struct {
    int64_t threads;
    double gamma;
    int64_t epochs;
    double target_r_sq;
    int32_t variant;           /* ASYRK_FULL_ROW | ASYRK_SINGLE_COMPONENT */
    int32_t sampling;          /* ASYRK_SLICE_SHUFFLE (reference default) | ... */
    uint64_t seed;
    int64_t snapshot_interval;
    const double* x_star;      /* host, n entries, or NULL (dist_sq disabled) */
    /* --- device extensions (zero = reference behaviour) --- */
    int32_t precision;         /* ASYRK_F64 ... */
    int32_t allow_unnormalized; /* 1: async/norm_proportional on raw rows (config 4) */
    int32_t record_every_boundary; /* async: 1 = a record at every snapshot boundary; 0 = the
                                      boundaries the host-driven monitor schedule picks (
                                      the reference coordinator likewise records only the boundaries
                                      it catches), always including the stopping one */
    int32_t det_reassociate;   /* threads == 1: 0 = the reference's floating-point order (bitwise,
                                  default); 1 = the same row sequence with a warp-tree dot product,
                                  the precomputed reciprocal and a fused update (iterates within
                                  1e-12 relative of the reference) */
} asyrk_run_config;

/* RkConfig (kaczmarz.hpp:95-103) */
typedef struct {
    int64_t max_epochs;
    double target_r_sq;
    uint64_t seed;
    int32_t sampling;          /* ASYRK_RK_* */
    const double* x_star;
    /* --- device extension (zero = reference behaviour) --- */
    int32_t det_reassociate;   /* as asyrk_run_config::det_reassociate */
} asyrk_rk_config;

/* Trace (trace.hpp:11-37), caller-allocated. count receives the number of
 * records produced; at most cap are written. dist_sq entries are -1 when
 * x_star is NULL. final_x (n entries) may be NULL. */
typedef struct {
    int64_t cap;
    int64_t count;
    int64_t* epoch_index;
    double* r_sq;
    double* grad_sq;
    double* dist_sq;
    double* wall_seconds;
    int64_t* updates_applied;
    double* final_x;
} asyrk_trace_out;

/* InstrumentReport (parallel.hpp:36-42). */
typedef struct {
    int64_t row_updates;
    int64_t increments;
    double max_abs_error;
    double tolerance;
    int32_t consistent;
} asyrk_instrument_out;

/* Device-side timing of the last solve on a system (CUDA events on the
 * launching stream). */
typedef struct {
    double solve_ms;           /* first to last kernel of the solve */
    double worker_ms;          /* sum over projection-kernel launches */
    double monitor_ms;         /* sum over residual-monitor launches */
    int64_t worker_launches;
    int64_t monitor_launches;
    int64_t kernel_launches;   /* all kernels this library launched */
    int64_t projections;       /* row projections applied */
    int32_t resident_warps;    /* concurrent worker warps actually resident */
    int32_t warps;             /* worker warps launched */
} asyrk_solve_stats;

/* ---- one-shot entry points: host buffers in, host buffers out ---------- */

/* solve_parallel (parallel.hpp:52-54). instrument may be NULL. */
asyrk_status asyrk_solve_parallel(const asyrk_csr_view* A, const double* b, const double* x0,
                                  const asyrk_run_config* cfg, asyrk_trace_out* trace,
                                  asyrk_instrument_out* instrument);

/* rk_solve (kaczmarz.hpp:108-109) — deterministic, bit-identical iterates. */
asyrk_status asyrk_rk_solve(const asyrk_csr_view* A, const double* b, const double* x0,
                            const asyrk_rk_config* cfg, asyrk_trace_out* trace);

/* residuals (csr.hpp:89-90): r_sq, grad_sq in the reference's summation order. */
asyrk_status asyrk_residuals(const asyrk_csr_view* A, const double* x, const double* b, double* r_sq,
                             double* grad_sq);

/* power_iteration_lambda_max (stats.hpp:46-47), same start vector. */
asyrk_status asyrk_power_iteration_lambda_max(const asyrk_csr_view* A, double tol, int64_t max_iters,
                                              double* lambda_max);

/* compute_stats (stats.hpp:42, stats.cpp:52-130) with exact_spectral =
 * false: every field of SystemStats except lambda_min / sigma_r (those come
 * from asyrk_dense_spectrum). mu, nu, delta, alpha, frob_sq, l_max, l_res and
 * theta are bit-identical to the reference; lambda_max is the device power
 * iteration (tol, max_iters = StatsOptions::tol / max_power_iters);
 * max_iters < 0 skips it (lambda_max = 0), for exact_spectral callers that
 * take lambda_max / lambda_min / sigma_r from asyrk_dense_spectrum
 * (include/asyrk_dense.h).
 * Errors: NotNormalized (A not flagged normalized), ZeroColumn (first empty
 * column), PowerIterationDiverged. */
typedef struct asyrk_stats_out {
    int64_t m, n;
    double delta;            /* nnz / (m n) */
    int64_t mu, nu;          /* max row / column nonzero count */
    double alpha;            /* max_{i,t} theta_i |a_it| ||column t|| */
    double lambda_max;       /* power iteration on A^T A */
    double frob_sq;          /* ||A||_F^2, column order */
    double l_max;            /* max diagonal entry of A^T A */
    double l_res;            /* max row norm of A^T A */
    int64_t power_iterations;
    int64_t* theta;          /* optional caller buffer of m per-row counts */
} asyrk_stats_out;
asyrk_status asyrk_compute_stats(const asyrk_csr_view* A, double tol, int64_t max_iters, asyrk_stats_out* out);

/* ---- bounded-delay simulator (delay_sim.hpp, delay_sim.cpp:71-338) -------- *
 * Deterministic replay of the asynchronous recursion with a delay model
 * (DelayModel, delay_sim.hpp:17-31), bit-identical to the reference: trace
 * records, events, history, probes, final_x and Monte-Carlo means.
 * Distances (SimOptions::projector): dist_point = the projector's solution
 * point A^+ b (n entries; SolutionProjector::solution_point, full column
 * rank) adds ||x - dist_point||^2 to every record and enables probe_dist_sq;
 * without it probe_dist_sq fails with InvalidArgument, as the reference does
 * without a SolutionProjector. */
typedef struct {
    double gamma;          /* StepParams::gamma, >= 0 (InvalidGamma) */
    int64_t tau;           /* DelayModel::tau, >= 0 */
    int32_t delay;         /* 0 fixed, 1 uniform_random, 2 max_staleness */
    int32_t variant;       /* 0 single_component, 1 full_row (UpdateVariant) */
    int64_t iterations;    /* >= 1 */
    uint64_t seed;         /* simulate: seed; monte_carlo_ratios: base_seed */
    int64_t probe_every;   /* SimOptions (simulate only) */
    int32_t probe_r_sq;
    int32_t probe_dist_sq; /* needs dist_point: InvalidArgument */
    int64_t max_events;
    const double* dist_point;  /* NULL, or the projector's A^+ b (n) */
} asyrk_sim_config;

/* SimRun (delay_sim.hpp:44-55). Caller buffers with capacities; counts are
 * the reference's sizes (at most cap entries are written). history holds
 * history_rows x n doubles (the last min(tau+1, iterations+1) iterates,
 * oldest first). Events: t = -1 marks full_row (kAllComponents). */
typedef struct {
    asyrk_trace_out trace;
    int64_t ev_cap, ev_count;
    int64_t *ev_j, *ev_i, *ev_t, *ev_k;
    double* ev_step;
    int64_t history_cap, history_rows;
    double* history;
    int64_t probe_cap, probe_count;
    int64_t* probe_iteration;
    double* probe_r_sq;
    double* probe_dist_sq;     /* probe_cap entries when probe_dist_sq (may be NULL otherwise) */
} asyrk_sim_out;

asyrk_status asyrk_simulate(const asyrk_csr_view* A, const double* b, const double* x0, const asyrk_sim_config* cfg,
                            asyrk_sim_out* out);
/* mean_r_sq: iterations + 1 entries; ratios: iterations entries. runs >= 100
 * (InsufficientData); run r uses seed base_seed + r. */
asyrk_status asyrk_monte_carlo_ratios(const asyrk_csr_view* A, const double* b, const double* x0,
                                      const asyrk_sim_config* cfg, int64_t runs, double* mean_r_sq, double* ratios);
/* rate_fit (host arithmetic, delay_sim.cpp:272-338). */
asyrk_status asyrk_rate_fit(const double* y, int64_t count, double stride, double* slope, double* r2);

/* sweep_threads (parallel.hpp:73-75): one solve per entry of thread_list
 * (must contain 1); out arrays have n_threads entries. */
asyrk_status asyrk_sweep_threads(const asyrk_csr_view* A, const double* b, const double* x0,
                                 const asyrk_run_config* cfg, const int64_t* thread_list,
                                 int64_t n_threads, double* wall_seconds, int64_t* epochs,
                                 double* final_r_sq, double* speedup);

/* The host-driven monitor schedule of the async solves (DESIGN.md §5,
 * csrc/schedule.h), host arithmetic: given the records so far (boundaries in
 * snapshot intervals, ascending, and their r_sq), the next boundary to
 * evaluate. every != 0 (record_every_boundary) or target <= 0: the next one.
 * max_gap <= 0: the default (24, or ASYRK_MONITOR_MAX_GAP). Exposed so that
 * multi-rank drivers in any language take the same decisions. */
asyrk_status asyrk_monitor_schedule_next(double target_r_sq, int32_t every, int64_t max_gap,
                                         const int64_t* boundaries, const double* r_sq, int64_t count,
                                         int64_t* next);

/* ---- device-resident system: upload once, solve many times ------------- */
typedef struct asyrk_system asyrk_system;

/* Uploads A (+ b) and packs the device layout (row records, CSC, alias).
 * stream: a cudaStream_t (cudaStreamLegacy = (void*)1 for the legacy default
 * stream) or NULL for a library-owned stream. */
asyrk_status asyrk_system_create(const asyrk_csr_view* A, const double* b, int32_t precision,
                                 void* stream, asyrk_system** out);
asyrk_status asyrk_system_destroy(asyrk_system* sys);
/* x0 NULL means x0 = 0. */
asyrk_status asyrk_system_solve(asyrk_system* sys, const double* x0, const asyrk_run_config* cfg,
                                asyrk_trace_out* trace, asyrk_instrument_out* instrument);
asyrk_status asyrk_system_rk_solve(asyrk_system* sys, const double* x0, const asyrk_rk_config* cfg,
                                   asyrk_trace_out* trace);
asyrk_status asyrk_system_residuals(asyrk_system* sys, const double* x, double* r_sq, double* grad_sq);
/* Replace b (m entries) of a system in place (device re-pack of the record headers). */
asyrk_status asyrk_system_set_rhs(asyrk_system* sys, const double* b);
/* y = A x (m entries) and y = A^T x (n entries), reference summation order
 * (CsrMatrix::multiply / multiply_transpose, ref/src/csr.cpp:72-92). */
asyrk_status asyrk_system_multiply(asyrk_system* sys, const double* x, double* y);
asyrk_status asyrk_system_multiply_transpose(asyrk_system* sys, const double* x, double* y);
asyrk_status asyrk_system_power_iteration(asyrk_system* sys, double tol, int64_t max_iters, double* lambda_max,
                                          int64_t* iterations);
/* Counts and device timings of the last solve on this system; the timings are
 * read from its CUDA events here (not inside the solve call), valid until the
 * next solve. */
asyrk_status asyrk_system_last_stats(const asyrk_system* sys, asyrk_solve_stats* out);
/* simulate / monte_carlo_ratios on a resident fp64 system (b = the system's). */
asyrk_status asyrk_system_simulate(asyrk_system* sys, const double* x0, const asyrk_sim_config* cfg,
                                   asyrk_sim_out* out);
asyrk_status asyrk_system_monte_carlo_ratios(asyrk_system* sys, const double* x0, const asyrk_sim_config* cfg,
                                             int64_t runs, double* mean_r_sq, double* ratios);
/* compute_stats on a resident fp64 system (see asyrk_compute_stats). */
asyrk_status asyrk_system_compute_stats(asyrk_system* sys, double tol, int64_t max_iters, asyrk_stats_out* out);
/* The async workers' own row draws (tests and diagnostics): rows_out[w *
 * per_warp + j] = the row warp w of a `warps`-warp solve with `seed` draws at
 * position j of epoch `epoch` (sampling: with_replacement, slice_shuffle —
 * a permutation of the warp's slice per pass — or norm_proportional through
 * the device alias table, ref kaczmarz.cpp:14-69). */
asyrk_status asyrk_system_sample_rows(asyrk_system* sys, int32_t sampling, uint64_t seed, int64_t warps, int64_t epoch,
                                      int64_t per_warp, int32_t* rows_out);
/* Deterministic multi-RHS rk_solve on a resident fp64 system (SURVEY.md §8c,
 * config 5's parity definition): B is m x k row-major (k right-hand sides), X0
 * (or NULL = zeros), cfg->x_star (or NULL) and X_out are n x k row-major. All
 * columns consume ONE row sequence — the reference rk_solve's
 * (kaczmarz.cpp:128-227) for cfg->seed / sampling — and column j's iterate is
 * bit-identical to rk_solve(A, B[:, j], X0[:, j]) with that seed. A record per
 * epoch: r_sq, grad_sq, dist_sq are the per-column exact values summed in
 * column order; the stop is global (sum r_sq <= target_r_sq, or max_epochs).
 * trace->final_x is not written (X_out holds the iterates). */
asyrk_status asyrk_system_rk_solve_multi(asyrk_system* sys, const double* B, int64_t k, const double* X0,
                                         const asyrk_rk_config* cfg, double* X_out, asyrk_trace_out* trace);
/* Largest number of worker warps that are co-resident for this system. */
asyrk_status asyrk_system_max_resident_warps(const asyrk_system* sys, int32_t precision, int32_t* out);

/* ---- multi-right-hand-side AsyRK (BASELINE config 5) -------------------- *
 * k right-hand sides share A and the row sequence: one row projection
 * updates every RHS column (X n x k row-major fp32, B m x k). A GPU owns the
 * column shard [c0, c1) (a power of two, 2..64 columns). The reference is
 * single-RHS (its solve_parallel, ref/include/asyrk/parallel.hpp:52-54, per
 * column is the oracle: SURVEY.md §8c). Sampling: with_replacement or
 * slice_shuffle (RunConfig::sampling).
 *
 * Residual evaluations follow the host-driven monitor schedule:
 * every boundary while the target is 0 or record_every_boundary is set, else
 * the boundaries a decay fit of the last records picks, always the last one.
 *
 * Multi-GPU protocol (one process per GPU; the collective is the caller's,
 * e.g. NCCL all-reduce on the system's stream):
 *   begin -> [all-reduce(norms, sum)] -> commit ->
 *   loop { stopped? -> step -> if due: [all-reduce(norms, sum)] -> commit }
 *   -> finish
 * norms is a device double[3] = this shard's {||R||_F^2, ||A^T R||_F^2,
 * ||X - X*||_F^2}, valid when due() reports 1 (the step ended at an
 * evaluated boundary); after the all-reduce every rank takes the same global
 * stop decision (r_sq <= target_r_sq) on the device. stopped() waits for the
 * latest commit that recorded and returns its decision (or 1 at the epoch
 * cap), so all ranks leave the loop after the same step. Native drivers of
 * the same loop: asyrk_mrhs_solve (one shard, no collective),
 * asyrk_mrhs_solve_nccl (one shard per process, an NCCL communicator) and
 * asyrk_mrhs_solve_devices (one process, several GPUs, ncclCommInitAll). */
typedef struct asyrk_mrhs asyrk_mrhs;
asyrk_status asyrk_mrhs_create(const asyrk_csr_view* A, const float* B, int64_t k_total, int64_t c0, int64_t c1,
                               void* stream, asyrk_mrhs** out);
asyrk_status asyrk_mrhs_destroy(asyrk_mrhs* h);
/* X0 (n x k_total fp32) and Xstar (n x k_total fp64) may be NULL. */
asyrk_status asyrk_mrhs_begin(asyrk_mrhs* h, const asyrk_run_config* cfg, const float* X0, const double* Xstar);
asyrk_status asyrk_mrhs_norms(asyrk_mrhs* h, double** dev_norms);
/* 1 when the last begin/step ended at an evaluated boundary: all-reduce norms, then commit */
asyrk_status asyrk_mrhs_due(asyrk_mrhs* h, int32_t* due);
/* records the evaluated boundary the last begin/step reached (no-op otherwise; advance is ignored) */
asyrk_status asyrk_mrhs_commit(asyrk_mrhs* h, int32_t advance);
asyrk_status asyrk_mrhs_step(asyrk_mrhs* h);
asyrk_status asyrk_mrhs_stopped(asyrk_mrhs* h, int32_t* stopped);
/* X_out: n x (c1 - c0) fp32, this shard's columns. */
asyrk_status asyrk_mrhs_finish(asyrk_mrhs* h, asyrk_trace_out* trace, float* X_out);
/* single-process convenience: begin + loop + finish (no collective) */
asyrk_status asyrk_mrhs_solve(asyrk_mrhs* h, const asyrk_run_config* cfg, const float* X0, const double* Xstar,
                              asyrk_trace_out* trace, float* X_out);
asyrk_status asyrk_mrhs_last_stats(const asyrk_mrhs* h, asyrk_solve_stats* out);
/* Largest number of co-resident worker warps for this shard's width. */
asyrk_status asyrk_mrhs_max_resident_warps(const asyrk_mrhs* h, int32_t* out);
/* asyrk_microbench_xside_mrhs on this shard's own X (n x kl, re-initialized
 * by every solve; the address and pages the worker uses, as
 * asyrk_system_microbench_xside does for config 2), theta = the rows' length
 * (at most 32). proj_per_s = row projections per second. */
asyrk_status asyrk_mrhs_microbench_xside(asyrk_mrhs* h, int32_t warps, int64_t proj_per_warp, double* proj_per_s,
                                         double* kernel_ms);

/* ---- multi-GPU: NCCL (SURVEY.md §8b "mrhs_shard_solve(..., ncclComm_t)") ----
 * libnccl.so.2 is resolved at run time (the copy already loaded in the
 * process if any, e.g. PyTorch's, else the system library), so the library
 * has no link-time NCCL dependency; these return ThreadSpawnFailure with the
 * reason when NCCL cannot be loaded. Communicators are ncclComm_t passed as
 * void*. The unique id is the opaque 128-byte ncclUniqueId: rank 0 creates it
 * and the launcher broadcasts it (e.g. torch.distributed / MPI). */
#define ASYRK_NCCL_UNIQUE_ID_BYTES 128
asyrk_status asyrk_nccl_available(int32_t* version);
asyrk_status asyrk_nccl_get_unique_id(char* id /* [ASYRK_NCCL_UNIQUE_ID_BYTES] */);
/* on the calling thread's current device */
asyrk_status asyrk_nccl_comm_init_rank(void** comm, int32_t nranks, const char* id, int32_t rank);
asyrk_status asyrk_nccl_comm_destroy(void* comm);
/* One rank's shard of a sharded solve: the whole loop in C++, one
 * ncclAllReduce(sum) of the 3 shard norms per evaluated boundary on the
 * shard's stream. Every rank of comm calls it with the same cfg. */
asyrk_status asyrk_mrhs_solve_nccl(asyrk_mrhs* h, const asyrk_run_config* cfg, void* comm, const float* X0,
                                   const double* Xstar, asyrk_trace_out* trace, float* X_out);
/* One process, ndev GPUs: k_total columns split evenly over devices[], one
 * shard per device, ncclCommInitAll, the same loop with grouped all-reduces.
 * trace: the (global, identical) records; X_out: n x k_total fp32; stats:
 * device 0's solve stats (may be NULL). */
asyrk_status asyrk_mrhs_solve_devices(const asyrk_csr_view* A, const float* B, int64_t k_total, const int32_t* devices,
                                      int32_t ndev, const asyrk_run_config* cfg, const float* X0, const double* Xstar,
                                      asyrk_trace_out* trace, float* X_out, asyrk_solve_stats* stats);

/* ---- measurement ------------------------------------------------------- */
/* x-side roofline R_x: theta random gathers of an n-element
 * x, a warp reduction, theta random red.global.add per "projection", no A
 * stream. mode 0 dependent gather->red, 1 gathers only, 2 reds only; mode + 16
 * keeps 2 rows in flight per warp (the K2 worker's shape). */
asyrk_status asyrk_microbench_xside(int64_t n, int32_t theta, int32_t precision, int32_t warps,
                                    int64_t proj_per_warp, int32_t mode, double* proj_per_s, double* kernel_ms);
/* The multi-RHS x side (config 5): per "projection" theta
 * random rows of an n x kl fp32 X gathered (float4 lanes), a per-column warp
 * reduction, theta red.global.add.v4.f32 back; no A / B stream. At the widths
 * where the row-parallel worker runs (kl 8 / 16 / 32) the pattern is that worker's:
 * a group of kl/4 lanes per row, four gathers in flight, no reduction, and
 * every lane group projects proj_per_warp rows. proj_per_s = row projections
 * per second (x kl for column projections). */
asyrk_status asyrk_microbench_xside_mrhs(int64_t n, int32_t theta, int32_t kl, int32_t warps, int64_t proj_per_warp,
                                         double* proj_per_s, double* kernel_ms);
/* The same on a resident system's own x buffer (address, footprint, its row
 * length as theta, x's precision) on its stream; x is re-initialised by every
 * solve, so the ~1e-30 perturbation it leaves does not matter. */
asyrk_status asyrk_system_microbench_xside(asyrk_system* sys, int32_t warps, int64_t proj_per_warp, int32_t mode,
                                           double* proj_per_s, double* kernel_ms);

#ifdef __cplusplus
}
#endif
#endif /* ASYRK_CUDA_H */
