/* Dense spectrum and least squares — C ABI (SURVEY.md §8f item 4 and the
 * dense oracle it needs).
 *
 *   asyrk_dense_svd     replaces decompose()/spectrum_of() (ref/src/dense.cpp:27-50,
 *                       Eigen BDCSVD) with a one-sided Jacobi SVD on the device
 *                       (paper_1401_4780_b200/csrc/dense.cu)
 *   asyrk_lsq_augment   augment()        (ref/src/lsq.cpp:36-101, lsq.hpp:33-38)
 *   asyrk_lsq_solve     lsq_solve()      (ref/src/lsq.cpp:103-170, lsq.hpp:62-66)
 *                       — the augmented system is solved by the device rk_solve
 *                       (threads <= 1: the reference's own path, bit-identical
 *                       iterates) or by the async warp workers (threads > 1)
 *   asyrk_lsq_optimal_params / asyrk_lsq_critical_ratio  (lsq.cpp:12-34)
 *
 * Status codes and asyrk_last_error() as in asyrk_cuda.h. */
#ifndef ASYRK_DENSE_H
#define ASYRK_DENSE_H

#include "asyrk_cuda.h"
#include "asyrk_io.h"

#ifdef __cplusplus
extern "C" {
#endif

/* SolutionProjector::kDefaultDenseCap (dense.hpp:28) */
#define ASYRK_DENSE_CAP_DEFAULT 4000000
/* largest m*n the device SVD accepts when max_cells = 0 (512 MB of fp64) */
#define ASYRK_DENSE_DEVICE_CAP 67108864

/* Thin SVD of A: sigma (min(m,n) entries, descending); U (m x min(m,n)) and
 * V (n x min(m,n)), column-major, may each be NULL. rank counts singular
 * values above 1e-10 * sigma_max (dense.cpp:12,36-40). sweeps (may be NULL)
 * receives the Jacobi sweeps used. TooLarge when m*n > max_cells
 * (0 = ASYRK_DENSE_DEVICE_CAP). */
asyrk_status asyrk_dense_svd(const asyrk_csr_view* A, int64_t max_cells, double* sigma, double* U, double* V,
                             int32_t* rank, int32_t* sweeps);

/* Spectrum (dense.hpp:15-20) */
typedef struct {
    double lambda_max;  /* sigma_max^2 */
    double lambda_min;  /* sigma_r^2 */
    double sigma_r;     /* smallest singular value above the rank cutoff */
    int32_t rank;
} asyrk_spectrum;
asyrk_status asyrk_dense_spectrum(const asyrk_csr_view* A, asyrk_spectrum* out);

/* dense_min_norm_lstsq (dense.hpp:53-55, dense.cpp:110-117): x = A^+ b
 * (n entries) from the device SVD. */
asyrk_status asyrk_dense_lstsq(const asyrk_csr_view* A, const double* b, double* x);

/* optimal_params (lsq.cpp:12-18): phi = 1, zeta = sigma_r / sqrt(2);
 * NonPositiveSigma unless sigma_r > 0. */
asyrk_status asyrk_lsq_optimal_params(double sigma_r, double* phi, double* zeta);
/* critical_ratio (lsq.cpp:20-34); InvalidArgument on non-positive inputs. */
asyrk_status asyrk_lsq_critical_ratio(double sigma_r, double frob_sq, int64_t m, double zeta, double phi,
                                      double* ratio);

/* augment (lsq.cpp:36-101): the (n+m) x (n+m) normalized augmented system,
 * bit-identical to the reference's a_tilde / b_tilde / row_scales. A must be
 * flagged normalized (NotNormalized), zeta, phi > 0 (InvalidArgument), no
 * empty column (ZeroColumn). b_tilde and row_scales: n+m caller entries. */
asyrk_status asyrk_lsq_augment(const asyrk_csr_view* A, const double* b, double zeta, double phi,
                               asyrk_host_csr** a_tilde, double* b_tilde, double* row_scales);

/* LsqConfig (lsq.hpp:40-50) + the device solver choice */
typedef struct {
    double zeta;            /* 0: the optimal value from sigma_r */
    double phi;             /* 0: the optimal value (1) */
    int32_t has_sigma_r;    /* std::optional<double> sigma_r */
    double sigma_r;         /* used when has_sigma_r; must be > 0 */
    int64_t max_epochs;     /* reference default 5000 */
    double target_r_sq;     /* stop threshold on the augmented residual */
    uint64_t seed;
    int32_t sampling;       /* ASYRK_RK_* (threads <= 1) */
    int64_t threads;        /* <= 1: rk_solve (reference path); > 1: async warp workers */
    double gamma;           /* async step (threads > 1), 0 = 1.0 */
} asyrk_lsq_config;

/* LsqResult (lsq.hpp:52-60). x_ls: n entries; y: m entries (may be NULL);
 * trace: records of the augmented solve (final_x, if given, n+m entries). */
typedef struct {
    double* x_ls;
    double* y;
    double grad_norm;       /* ||A^T (A x_ls - b)|| */
    double zeta, phi, sigma_r;
    asyrk_trace_out trace;
} asyrk_lsq_out;

/* lsq_solve (lsq.cpp:103-170). Without a supplied sigma_r the dense spectrum
 * is used when m*n <= ASYRK_DENSE_CAP_DEFAULT, else SigmaUnavailable. */
asyrk_status asyrk_lsq_solve(const asyrk_csr_view* A, const double* b, const asyrk_lsq_config* cfg,
                             asyrk_lsq_out* out);

#ifdef __cplusplus
}
#endif
#endif /* ASYRK_DENSE_H */
