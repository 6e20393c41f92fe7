/*
 * asyrk_datagen.h — seeded synthetic systems with the BASELINE.json config
 * shapes (fixed nonzeros per row at distinct uniform columns). The
 * reference's gen_sparse_gaussian (ref/src/datagen.cpp:13-137) samples a
 * delta-density grid and cannot produce fixed-theta rows,
 * so the benchmark configs use this generator; instances are plain host CSR
 * arrays that feed both the GPU path and the reference CPU path.
 *
 * Row i draws from its own stream (xoshiro256** seeded by splitmix64 of
 * (seed, i)), so generation is multithreaded and independent of the thread
 * count. Rows are normalized with the reference's normalize_rows semantics
 * (csr.cpp:113-138: divide, then recompute the norm in storage order), then
 * optionally scaled by s_i with log10 s_i ~ U(-scale_decades, scale_decades)
 * (config 4). x* ~ N(0,1) (k columns, row-major n x k) and B = A X* in
 * storage order.
 */
#ifndef ASYRK_DATAGEN_H
#define ASYRK_DATAGEN_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ASYRK_GEN_NORMAL = 0, ASYRK_GEN_UNIFORM = 1 };

/* Caller-allocated outputs: row_ptr[m+1], col_idx[m*theta], values[m*theta],
 * row_norm[m], b[m*k] (row-major m x k), x_star[n*k] (row-major n x k).
 * Returns 0, or an asyrk_status on invalid arguments. *normalized receives 1
 * when every row norm is within 1e-12 of 1. */
int asyrk_generate_fixed_theta(int64_t m, int64_t n, int64_t theta, uint64_t seed, int32_t value_dist,
                               double scale_decades, int64_t k, int32_t threads, int64_t* row_ptr,
                               int64_t* col_idx, double* values, double* row_norm, double* b, double* x_star,
                               int32_t* normalized);

#ifdef __cplusplus
}
#endif
#endif
