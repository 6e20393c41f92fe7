/*
 * workload.c — TEST / BENCHMARK INFRASTRUCTURE ONLY. A plain-C restatement of
 * the seeded fixed-theta instance generator (include/asyrk_datagen.h,
 * paper_1401_4780_b200/csrc/host/datagen.cpp) so that bench.py's reference
 * arm (--impl reference) and cpu_baseline leg build the BASELINE config
 * instances without mapping the product library (libasyrk_b200.so) into the
 * reference process. tests/test_oracle.py::test_workload_generator_bitwise
 * pins it bit for bit against the product generator.
 *
 * Same algorithm: per-row xoshiro256** streams seeded through splitmix64 of
 * (seed, row), theta distinct columns by rejection then sorted, N(0,1)
 * (Marsaglia polar) or U(-1,1) values, normalize_rows semantics
 * (ref/src/csr.cpp:113-138: divide by the norm, recompute it in storage
 * order, skip rows within 1e-12 of unit norm), optional log-uniform row scale
 * (config 4), x* ~ N(0,1) (k columns) and B = A X* in storage order
 * (ref/src/csr.cpp:65-70 row_dot). Compiled with -ffp-contract=off like the
 * product's host code, and both call the same libm, so the arrays are
 * bit-identical.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

static uint64_t wl_mix64(uint64_t z) {
    z += 0x9e3779b97f4a7c15ULL;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

typedef struct {
    uint64_t s[4];
} wl_rng;

static void wl_seed(wl_rng* g, uint64_t seed, uint64_t stream) {
    uint64_t z = wl_mix64(seed) ^ wl_mix64(stream + 0x632BE59BD9B4E019ULL);
    for (int k = 0; k < 4; ++k) g->s[k] = z = wl_mix64(z);
}

static uint64_t wl_rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

static uint64_t wl_next(wl_rng* g) {
    uint64_t* s = g->s;
    const uint64_t r = wl_rotl(s[1] * 5, 7) * 9, t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = wl_rotl(s[3], 45);
    return r;
}

static uint64_t wl_below(wl_rng* g, uint64_t n) {
    const uint64_t lim = UINT64_MAX - UINT64_MAX % n;
    for (;;) {
        const uint64_t v = wl_next(g);
        if (v < lim) return v % n;
    }
}

static double wl_unit(wl_rng* g) { return (double)(wl_next(g) >> 11) * 0x1.0p-53; }

static double wl_normal(wl_rng* g) {
    for (;;) {
        const double u = 2.0 * wl_unit(g) - 1.0, v = 2.0 * wl_unit(g) - 1.0, q = u * u + v * v;
        if (q < 1.0 && q != 0.0) return u * sqrt(-2.0 * log(q) / q);
    }
}

typedef struct {
    int64_t m, n, theta, k;
    uint64_t seed;
    int32_t uniform_values;
    double scale_decades;
    int64_t *row_ptr, *col_idx;
    double *values, *row_norm, *b, *x_star;
    char* row_unit;
    int64_t lo, hi;
} wl_job;

static void* wl_xstar_rows(void* p) {
    wl_job* J = (wl_job*)p;
    for (int64_t j = J->lo; j < J->hi; ++j) {
        wl_rng g;
        wl_seed(&g, J->seed ^ 0x5EEDF00DULL, 0x8000000000000000ULL | (uint64_t)j);
        for (int64_t c = 0; c < J->k; ++c) J->x_star[j * J->k + c] = wl_normal(&g);
    }
    return NULL;
}

static void* wl_rows(void* p) {
    wl_job* J = (wl_job*)p;
    const int64_t theta = J->theta;
    int64_t* cols = (int64_t*)malloc((size_t)theta * sizeof(int64_t));
    for (int64_t i = J->lo; i < J->hi; ++i) {
        wl_rng g;
        wl_seed(&g, J->seed, (uint64_t)i);
        for (int64_t t = 0; t < theta;) {
            const int64_t c = (int64_t)wl_below(&g, (uint64_t)J->n);
            int dup = 0;
            for (int64_t u = 0; u < t; ++u)
                if (cols[u] == c) {
                    dup = 1;
                    break;
                }
            if (!dup) cols[t++] = c;
        }
        for (int64_t a = 1; a < theta; ++a) {  // insertion sort (theta is small)
            const int64_t v = cols[a];
            int64_t q = a - 1;
            while (q >= 0 && cols[q] > v) {
                cols[q + 1] = cols[q];
                --q;
            }
            cols[q + 1] = v;
        }
        const int64_t base = i * theta;
        J->row_ptr[i + 1] = base + theta;
        double ss = 0.0;
        for (int64_t t = 0; t < theta; ++t) {
            double v;
            do {
                v = J->uniform_values ? 2.0 * wl_unit(&g) - 1.0 : wl_normal(&g);
            } while (v == 0.0);
            J->col_idx[base + t] = cols[t];
            J->values[base + t] = v;
            ss += v * v;
        }
        double nrm = sqrt(ss);
        if (fabs(nrm - 1.0) > 1e-12) {
            for (int64_t t = 0; t < theta; ++t) J->values[base + t] /= nrm;
            ss = 0.0;
            for (int64_t t = 0; t < theta; ++t) ss += J->values[base + t] * J->values[base + t];
            nrm = sqrt(ss);
        }
        if (J->scale_decades > 0.0) {
            const double s = pow(10.0, J->scale_decades * (2.0 * wl_unit(&g) - 1.0));
            ss = 0.0;
            for (int64_t t = 0; t < theta; ++t) {
                J->values[base + t] *= s;
                ss += J->values[base + t] * J->values[base + t];
            }
            nrm = sqrt(ss);
        }
        J->row_norm[i] = nrm;
        J->row_unit[i] = fabs(nrm - 1.0) <= 1e-12;
        for (int64_t c = 0; c < J->k; ++c) {
            double s = 0.0;
            for (int64_t t = 0; t < theta; ++t) s += J->values[base + t] * J->x_star[J->col_idx[base + t] * J->k + c];
            J->b[i * J->k + c] = s;
        }
    }
    free(cols);
    return NULL;
}

static void wl_parallel(wl_job* proto, int64_t rows, int threads, void* (*fn)(void*)) {
    if (threads <= 0) threads = (int)sysconf(_SC_NPROCESSORS_ONLN);
    if (threads < 1) threads = 1;
    int64_t cap = rows / 1024;
    if (cap < 1) cap = 1;
    if (threads > cap) threads = (int)cap;
    pthread_t* th = (pthread_t*)malloc((size_t)threads * sizeof(pthread_t));
    wl_job* jobs = (wl_job*)malloc((size_t)threads * sizeof(wl_job));
    for (int t = 0; t < threads; ++t) {
        jobs[t] = *proto;
        jobs[t].lo = rows * t / threads;
        jobs[t].hi = rows * (t + 1) / threads;
        pthread_create(&th[t], NULL, fn, &jobs[t]);
    }
    for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
    free(th);
    free(jobs);
}

/* Same contract as asyrk_generate_fixed_theta (include/asyrk_datagen.h). */
int oc_generate_fixed_theta(int64_t m, int64_t n, int64_t theta, uint64_t seed, int32_t value_dist,
                            double scale_decades, int64_t k, int32_t threads, int64_t* row_ptr, int64_t* col_idx,
                            double* values, double* row_norm, double* b, double* x_star, int32_t* normalized) {
    if (m < 1 || n < 1 || theta < 1 || theta > n || k < 1) return 24; /* InvalidArgument */
    wl_job J;
    memset(&J, 0, sizeof(J));
    J.m = m;
    J.n = n;
    J.theta = theta;
    J.k = k;
    J.seed = seed;
    J.uniform_values = value_dist == 1;
    J.scale_decades = scale_decades;
    J.row_ptr = row_ptr;
    J.col_idx = col_idx;
    J.values = values;
    J.row_norm = row_norm;
    J.b = b;
    J.x_star = x_star;
    J.row_unit = (char*)malloc((size_t)m);
    wl_parallel(&J, n, threads, wl_xstar_rows);
    wl_parallel(&J, m, threads, wl_rows);
    row_ptr[0] = 0;
    int32_t all = 1;
    for (int64_t i = 0; i < m; ++i)
        if (!J.row_unit[i]) {
            all = 0;
            break;
        }
    free(J.row_unit);
    if (normalized) *normalized = all;
    return 0;
}
