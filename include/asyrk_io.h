/* C ABI of the instance I/O (libasyrk_b200.so), for FFI hosts.
 *
 *   entry point                  replaces (reference)
 *   asyrk_read_matrix_market     read_matrix_market   ref/include/asyrk/io.hpp:16
 *   asyrk_write_matrix_market    write_matrix_market  ref/include/asyrk/io.hpp:15
 *   asyrk_read_vector            read_vector          ref/include/asyrk/io.hpp:20
 *   asyrk_write_vector           write_vector         ref/include/asyrk/io.hpp:19
 *   asyrk_read_instance          read_instance        ref/include/asyrk/io.hpp:30
 *   asyrk_write_instance         write_instance       ref/include/asyrk/io.hpp:29
 *   asyrk_read_csr_cache / asyrk_write_csr_cache      (new) binary CSR cache
 *
 * Status codes and asyrk_last_error() as in asyrk_cuda.h (IoError = 23 + 1).
 * Matrices read from files come back as library-owned host CSR handles:
 * query the sizes from asyrk_host_csr_info, copy the arrays out with
 * asyrk_host_csr_copy, release with asyrk_host_csr_free. Vectors come back
 * as library-allocated arrays released with asyrk_free. */
#ifndef ASYRK_IO_H
#define ASYRK_IO_H

#include <stdint.h>

#include "asyrk_cuda.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct asyrk_host_csr asyrk_host_csr;

typedef struct {
    int64_t m, n, nnz;
    int32_t normalized;
} asyrk_host_csr_info;

/* GenSpec echo of meta.json (ref datagen.hpp:11-18) */
typedef struct {
    int64_t m, n;
    double delta;
    uint64_t seed;
    int32_t consistent;
    double noise_level;
    int32_t has_x_star;   /* read: xstar.txt was present */
} asyrk_instance_meta;

asyrk_status asyrk_read_matrix_market(const char* path, asyrk_host_csr** out, asyrk_host_csr_info* info);
asyrk_status asyrk_write_matrix_market(const char* path, const asyrk_csr_view* A);
asyrk_status asyrk_read_csr_cache(const char* path, asyrk_host_csr** out, asyrk_host_csr_info* info);
asyrk_status asyrk_write_csr_cache(const char* path, const asyrk_csr_view* A);
asyrk_status asyrk_host_csr_get_info(const asyrk_host_csr* h, asyrk_host_csr_info* info);
/* row_norm may be NULL */
asyrk_status asyrk_host_csr_copy(const asyrk_host_csr* h, int64_t* row_ptr, int64_t* col_idx, double* values,
                                 double* row_norm);
void asyrk_host_csr_free(asyrk_host_csr* h);

asyrk_status asyrk_read_vector(const char* path, double** out, int64_t* count);
asyrk_status asyrk_write_vector(const char* path, const double* v, int64_t count);
void asyrk_free(void* p);

/* x_star may be NULL (inconsistent instance: no xstar.txt) */
asyrk_status asyrk_write_instance(const char* dir, const asyrk_csr_view* A, const double* b, const double* x_star,
                                  const asyrk_instance_meta* spec);
/* *x_star is NULL when the instance has no planted solution */
asyrk_status asyrk_read_instance(const char* dir, asyrk_host_csr** A, double** b, double** x_star,
                                 asyrk_instance_meta* meta);

#ifdef __cplusplus
}
#endif
#endif
