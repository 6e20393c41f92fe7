/*
 * oracle.c — TEST INFRASTRUCTURE ONLY. A plain-C restatement of the reference
 * AsyRK hot path, used by tests/ (via ctypes, oracle/__init__.py), by
 * __graft_entry__.smoke() as the checker, and by bench.py's cpu_baseline leg.
 * The product (paper_1401_4780_b200/) never links, imports or calls it.
 *
 * Reference: /root/reference/proj ("ref" below). Every function cites the
 * file:line it restates. Arithmetic follows the reference build exactly:
 * x86-64 SSE2 doubles, separate multiply and add (compiled here with
 * -ffp-contract=off), CSR storage order, left-to-right evaluation — so the
 * deterministic paths are bit-identical to the reference (pinned against
 * oracle/_ref and tests/golden/ in tests/test_oracle.py).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

/* ------------------------------------------------------------------ RNG */
/* std::mt19937_64 as specified by the C++ standard [rand.predef]
 * (w=64,n=312,m=156,r=31,a=0xb5026f5aa96619e9,u=29,d=0x5555555555555555,
 * s=17,b=0x71d67fffeda60000,t=37,c=0xfff7eee000000000,l=43,f=6364136223846793005).
 * ref/include/asyrk/rng.hpp:20-22 seeds it with splitmix64(seed ^ stream). */
#define MT_N 312
#define MT_M 156
typedef struct {
    uint64_t mt[MT_N];
    int idx;
} oc_mt64;

void oc_mt_seed(oc_mt64* g, uint64_t seed) {
    g->mt[0] = seed;
    for (int i = 1; i < MT_N; ++i)
        g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
    g->idx = MT_N;
}

static void mt_refill(oc_mt64* g) {
    const uint64_t UPPER = 0xFFFFFFFF80000000ULL, LOWER = 0x7FFFFFFFULL;
    const uint64_t A = 0xB5026F5AA96619E9ULL;
    for (int i = 0; i < MT_N; ++i) {
        uint64_t y = (g->mt[i] & UPPER) | (g->mt[(i + 1) % MT_N] & LOWER);
        uint64_t v = g->mt[(i + MT_M) % MT_N] ^ (y >> 1);
        if (y & 1ULL) v ^= A;
        g->mt[i] = v;
    }
    g->idx = 0;
}

uint64_t oc_mt_next(oc_mt64* g) {
    if (g->idx >= MT_N) mt_refill(g);
    uint64_t x = g->mt[g->idx++];
    x ^= (x >> 29) & 0x5555555555555555ULL;
    x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
    x ^= (x << 37) & 0xFFF7EEE000000000ULL;
    x ^= x >> 43;
    return x;
}

/* ref/include/asyrk/rng.hpp:14-19 */
uint64_t oc_splitmix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}

/* ref/include/asyrk/rng.hpp:20-22 */
void oc_make_stream(oc_mt64* g, uint64_t seed, uint64_t stream) { oc_mt_seed(g, oc_splitmix64(seed ^ stream)); }

/* ref/include/asyrk/rng.hpp:26-33 — rejection, then modulo */
uint64_t oc_uniform_below(oc_mt64* g, uint64_t n) {
    const uint64_t limit = UINT64_MAX - UINT64_MAX % n;
    uint64_t v;
    do {
        v = oc_mt_next(g);
    } while (v >= limit);
    return v % n;
}

/* ref/include/asyrk/rng.hpp:36-38 */
double oc_uniform_unit(oc_mt64* g) { return (double)(oc_mt_next(g) >> 11) * 0x1.0p-53; }

/* ref/include/asyrk/rng.hpp:41-48 (polar Box-Muller) */
double oc_standard_normal(oc_mt64* g) {
    double u, v, s;
    do {
        u = 2.0 * oc_uniform_unit(g) - 1.0;
        v = 2.0 * oc_uniform_unit(g) - 1.0;
        s = u * u + v * v;
    } while (s >= 1.0 || s == 0.0);
    return u * sqrt(-2.0 * log(s) / s);
}

/* ref/include/asyrk/rng.hpp:51-57 (Fisher-Yates from the top) */
void oc_shuffle_i64(int64_t* v, int64_t n, oc_mt64* g) {
    for (int64_t i = n; i > 1; --i) {
        int64_t j = (int64_t)oc_uniform_below(g, (uint64_t)i);
        int64_t t = v[i - 1];
        v[i - 1] = v[j];
        v[j] = t;
    }
}

/* Exposed for pinning: raw outputs / derived sequences of make_stream(seed,stream). */
void oc_stream_raw(uint64_t seed, uint64_t stream, int64_t count, uint64_t* out) {
    oc_mt64 g;
    oc_make_stream(&g, seed, stream);
    for (int64_t k = 0; k < count; ++k) out[k] = oc_mt_next(&g);
}
void oc_uniform_below_seq(uint64_t seed, uint64_t stream, uint64_t n, int64_t count, uint64_t* out) {
    oc_mt64 g;
    oc_make_stream(&g, seed, stream);
    for (int64_t k = 0; k < count; ++k) out[k] = oc_uniform_below(&g, n);
}
void oc_normal_seq(uint64_t seed, uint64_t stream, int64_t count, double* out) {
    oc_mt64 g;
    oc_make_stream(&g, seed, stream);
    for (int64_t k = 0; k < count; ++k) out[k] = oc_standard_normal(&g);
}
void oc_shuffle_seq(uint64_t seed, uint64_t stream, int64_t n, int64_t rounds, int64_t* out) {
    oc_mt64 g;
    oc_make_stream(&g, seed, stream);
    int64_t* p = (int64_t*)malloc((size_t)n * 8);
    for (int64_t i = 0; i < n; ++i) p[i] = i;
    for (int64_t r = 0; r < rounds; ++r) {
        oc_shuffle_i64(p, n, &g);
        memcpy(out + r * n, p, (size_t)n * 8);
    }
    free(p);
}

/* ------------------------------------------------------------------ CSR */
/* Error codes: 1 + ref ErrorCode ordinal (ref/include/asyrk/error.hpp:8-33). */
enum {
    OC_OK = 0,
    OC_IndexOutOfRange = 1,
    OC_DuplicateEntry = 2,
    OC_ZeroRow = 3,
    OC_ZeroColumn = 4,
    OC_NotNormalized = 5,
    OC_DimensionMismatch = 6,
    OC_PowerIterationDiverged = 7,
    OC_NonFinite = 8,
    OC_InvalidGamma = 16,
    OC_NonPositiveData = 17,
    OC_InsufficientData = 18,
    OC_InvalidArgument = 24,
};

typedef struct {
    int64_t m, n, nnz;
    int64_t* row_ptr; /* m+1 */
    int64_t* col;     /* nnz */
    double* val;      /* nnz */
    double* row_norm; /* m */
    int normalized;
} oc_csr;

typedef struct {
    int64_t r, c;
    double v;
    int64_t ord;
} trip_t;

static int trip_cmp(const void* a, const void* b) {
    const trip_t* x = (const trip_t*)a;
    const trip_t* y = (const trip_t*)b;
    if (x->r != y->r) return x->r < y->r ? -1 : 1;
    if (x->c != y->c) return x->c < y->c ? -1 : 1;
    return x->ord < y->ord ? -1 : (x->ord > y->ord);
}

void oc_csr_free(oc_csr* A) {
    if (!A) return;
    free(A->row_ptr);
    free(A->col);
    free(A->val);
    free(A->row_norm);
    free(A);
}

/* row_norm = sqrt of the storage-order sum of squares: ref/src/csr.cpp:53-61 */
static double row_sumsq(const oc_csr* A, int64_t i) {
    double s = 0.0;
    for (int64_t k = A->row_ptr[i]; k < A->row_ptr[i + 1]; ++k) s += A->val[k] * A->val[k];
    return s;
}

/* ref/src/csr.cpp:9-63 (CsrMatrix::from_triplets) */
oc_csr* oc_csr_from_triplets(int64_t m, int64_t n, int64_t nnz, const int64_t* rows, const int64_t* cols,
                             const double* vals, int* status) {
    *status = OC_OK;
    if (m < 1 || n < 1) {
        *status = OC_InvalidArgument;
        return NULL;
    }
    for (int64_t k = 0; k < nnz; ++k)
        if (rows[k] < 0 || rows[k] >= m || cols[k] < 0 || cols[k] >= n) {
            *status = OC_IndexOutOfRange;
            return NULL;
        }
    trip_t* t = (trip_t*)malloc((size_t)(nnz ? nnz : 1) * sizeof(trip_t));
    for (int64_t k = 0; k < nnz; ++k) t[k] = (trip_t){rows[k], cols[k], vals[k], k};
    qsort(t, (size_t)nnz, sizeof(trip_t), trip_cmp);
    oc_csr* A = (oc_csr*)calloc(1, sizeof(oc_csr));
    A->m = m;
    A->n = n;
    A->row_ptr = (int64_t*)calloc((size_t)m + 1, 8);
    A->col = (int64_t*)malloc((size_t)(nnz ? nnz : 1) * 8);
    A->val = (double*)malloc((size_t)(nnz ? nnz : 1) * 8);
    int64_t w = 0;
    for (int64_t k = 0; k < nnz; ++k) {
        if (k > 0 && t[k].r == t[k - 1].r && t[k].c == t[k - 1].c) {
            *status = OC_DuplicateEntry;
            free(t);
            oc_csr_free(A);
            return NULL;
        }
        if (t[k].v != 0.0) { /* explicit zeros dropped: csr.cpp:38-42 */
            A->col[w] = t[k].c;
            A->val[w] = t[k].v;
            A->row_ptr[t[k].r + 1]++;
            ++w;
        }
    }
    free(t);
    A->nnz = w;
    for (int64_t i = 0; i < m; ++i) A->row_ptr[i + 1] += A->row_ptr[i];
    A->row_norm = (double*)malloc((size_t)m * 8);
    for (int64_t i = 0; i < m; ++i) {
        if (A->row_ptr[i + 1] == A->row_ptr[i]) {
            *status = OC_ZeroRow;
            oc_csr_free(A);
            return NULL;
        }
        A->row_norm[i] = sqrt(row_sumsq(A, i));
    }
    return A;
}

/* ref/src/csr.cpp:113-138 (normalize_rows; rows within 1e-12 of unit norm are
 * left bit-identical, others divided then their norm recomputed) + flag_normalized
 * csr.cpp:103-111. b may be NULL. Modifies A and b in place. */
int oc_normalize_rows(oc_csr* A, double* b) {
    for (int64_t i = 0; i < A->m; ++i) {
        const double nrm = A->row_norm[i];
        if (nrm == 0.0) return OC_ZeroRow;
        if (fabs(nrm - 1.0) <= 1e-12) continue;
        for (int64_t k = A->row_ptr[i]; k < A->row_ptr[i + 1]; ++k) A->val[k] /= nrm;
        if (b) b[i] /= nrm;
        A->row_norm[i] = sqrt(row_sumsq(A, i));
    }
    for (int64_t i = 0; i < A->m; ++i)
        if (fabs(A->row_norm[i] - 1.0) > 1e-12) return OC_NotNormalized;
    A->normalized = 1;
    return OC_OK;
}

void oc_csr_export(const oc_csr* A, int64_t* row_ptr, int64_t* col, double* val, double* row_norm) {
    if (row_ptr) memcpy(row_ptr, A->row_ptr, (size_t)(A->m + 1) * 8);
    if (col) memcpy(col, A->col, (size_t)A->nnz * 8);
    if (val) memcpy(val, A->val, (size_t)A->nnz * 8);
    if (row_norm) memcpy(row_norm, A->row_norm, (size_t)A->m * 8);
}
int64_t oc_csr_nnz(const oc_csr* A) { return A->nnz; }

/* Wrap existing CSR arrays (copied); row_norm recomputed as csr.cpp:53-61;
 * normalized flag set iff every norm is within 1e-12 of 1 (flag_normalized). */
oc_csr* oc_csr_from_arrays(int64_t m, int64_t n, const int64_t* row_ptr, const int64_t* col, const double* val) {
    oc_csr* A = (oc_csr*)calloc(1, sizeof(oc_csr));
    A->m = m;
    A->n = n;
    A->nnz = row_ptr[m];
    A->row_ptr = (int64_t*)malloc((size_t)(m + 1) * 8);
    A->col = (int64_t*)malloc((size_t)(A->nnz ? A->nnz : 1) * 8);
    A->val = (double*)malloc((size_t)(A->nnz ? A->nnz : 1) * 8);
    A->row_norm = (double*)malloc((size_t)m * 8);
    memcpy(A->row_ptr, row_ptr, (size_t)(m + 1) * 8);
    memcpy(A->col, col, (size_t)A->nnz * 8);
    memcpy(A->val, val, (size_t)A->nnz * 8);
    int ok = 1;
    for (int64_t i = 0; i < m; ++i) {
        A->row_norm[i] = sqrt(row_sumsq(A, i));
        if (fabs(A->row_norm[i] - 1.0) > 1e-12) ok = 0;
    }
    A->normalized = ok;
    return A;
}

/* a_i . x in storage order: ref/src/csr.cpp:65-70 */
static double row_dot(const oc_csr* A, int64_t i, const double* x) {
    double s = 0.0;
    for (int64_t k = A->row_ptr[i]; k < A->row_ptr[i + 1]; ++k) s += A->val[k] * x[A->col[k]];
    return s;
}

/* ref/src/csr.cpp:72-77 */
void oc_multiply(const oc_csr* A, const double* x, double* y) {
    for (int64_t i = 0; i < A->m; ++i) y[i] = row_dot(A, i, x);
}

/* ref/src/csr.cpp:80-92 (rows with x_i == 0 skipped) */
void oc_multiply_transpose(const oc_csr* A, const double* x, double* y) {
    for (int64_t j = 0; j < A->n; ++j) y[j] = 0.0;
    for (int64_t i = 0; i < A->m; ++i) {
        const double xi = x[i];
        if (xi == 0.0) continue;
        for (int64_t k = A->row_ptr[i]; k < A->row_ptr[i + 1]; ++k) y[A->col[k]] += A->val[k] * xi;
    }
}

/* ref/src/csr.cpp:140-160 */
void oc_residuals(const oc_csr* A, const double* x, const double* b, double* r_sq, double* grad_sq) {
    double* r = (double*)malloc((size_t)A->m * 8);
    double* g = (double*)malloc((size_t)A->n * 8);
    double s = 0.0;
    for (int64_t i = 0; i < A->m; ++i) {
        r[i] = row_dot(A, i, x) - b[i];
        s += r[i] * r[i];
    }
    oc_multiply_transpose(A, r, g);
    double gs = 0.0;
    for (int64_t j = 0; j < A->n; ++j) gs += g[j] * g[j];
    *r_sq = s;
    *grad_sq = gs;
    free(r);
    free(g);
}

/* ------------------------------------------------------------- kernels */
/* ref/include/asyrk/kaczmarz.hpp:48-60 */
static double stale_residual(const oc_csr* A, const double* x, const double* b, int64_t i) {
    return row_dot(A, i, x) - b[i];
}
/* ref/include/asyrk/kaczmarz.hpp:63-67: gamma*res/(nrm*nrm), left to right */
static double row_coef(const oc_csr* A, int64_t i, double gamma, double res) {
    const double nrm = A->row_norm[i];
    return gamma * res / (nrm * nrm);
}
/* ref/include/asyrk/kaczmarz.hpp:70-80 */
static void apply_row(const oc_csr* A, int64_t i, double c, double* x) {
    for (int64_t k = A->row_ptr[i]; k < A->row_ptr[i + 1]; ++k) x[A->col[k]] -= c * A->val[k];
}

/* ref/src/kaczmarz.cpp:63-78 */
int oc_rk_step(const oc_csr* A, const double* b, const double* x, int64_t i, double* out) {
    if (i < 0 || i >= A->m) return OC_IndexOutOfRange;
    memcpy(out, x, (size_t)A->n * 8);
    const double res = stale_residual(A, out, b, i);
    apply_row(A, i, row_coef(A, i, 1.0, res), out);
    return OC_OK;
}

/* ----------------------------------------------------------- alias table */
/* ref/src/kaczmarz.cpp:14-61 (Walker alias; small/large stacks popped from the back) */
typedef struct {
    int64_t n;
    double* prob;
    int64_t* alias;
} oc_alias;

int oc_alias_build(oc_alias* t, const double* w, int64_t n) {
    if (n == 0) return OC_InvalidArgument;
    double sum = 0.0;
    for (int64_t k = 0; k < n; ++k) {
        if (!(w[k] >= 0.0)) return OC_InvalidArgument;
        sum += w[k];
    }
    if (sum <= 0.0) return OC_InvalidArgument;
    t->n = n;
    t->prob = (double*)calloc((size_t)n, 8);
    t->alias = (int64_t*)calloc((size_t)n, 8);
    double* scaled = (double*)malloc((size_t)n * 8);
    int64_t* small = (int64_t*)malloc((size_t)n * 8);
    int64_t* large = (int64_t*)malloc((size_t)n * 8);
    int64_t ns = 0, nl = 0;
    for (int64_t k = 0; k < n; ++k) scaled[k] = w[k] * (double)n / sum;
    for (int64_t k = 0; k < n; ++k) {
        if (scaled[k] < 1.0)
            small[ns++] = k;
        else
            large[nl++] = k;
    }
    while (ns > 0 && nl > 0) {
        const int64_t s = small[--ns];
        const int64_t l = large[nl - 1];
        t->prob[s] = scaled[s];
        t->alias[s] = l;
        scaled[l] -= 1.0 - scaled[s];
        if (scaled[l] < 1.0) {
            --nl;
            small[ns++] = l;
        }
    }
    for (int64_t k = 0; k < nl; ++k) t->prob[large[k]] = 1.0;
    for (int64_t k = 0; k < ns; ++k) t->prob[small[k]] = 1.0;
    free(scaled);
    free(small);
    free(large);
    return OC_OK;
}
static void alias_free(oc_alias* t) {
    free(t->prob);
    free(t->alias);
}
/* ref/src/kaczmarz.cpp:63-69 (AliasTable::sample) */
static int64_t alias_sample(const oc_alias* t, oc_mt64* g) {
    const int64_t k = (int64_t)oc_uniform_below(g, (uint64_t)t->n);
    const double u = oc_uniform_unit(g);
    return u < t->prob[k] ? k : t->alias[k];
}

int oc_alias_sample_seq(const double* w, int64_t n, uint64_t seed, int64_t count, int64_t* out) {
    oc_alias t;
    int st = oc_alias_build(&t, w, n);
    if (st) return st;
    oc_mt64 g;
    oc_make_stream(&g, seed, 0);
    for (int64_t k = 0; k < count; ++k) out[k] = alias_sample(&t, &g);
    alias_free(&t);
    return OC_OK;
}

/* ------------------------------------------------------------- traces */
typedef struct {
    int64_t cap;
    int64_t count;
    int64_t* epoch_index;
    double* r_sq;
    double* grad_sq;
    double* dist_sq;
    double* wall;
    int64_t* updates;
    double* final_x;
} oc_trace;

typedef struct {
    int64_t row_updates;
    int64_t increments;
    double max_abs_error;
    double tolerance;
    int32_t consistent;
} oc_instrument;

static double now_s(void) {
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

/* The record lambda of rk_solve / solve_single (kaczmarz.cpp:178-199,
 * parallel.cpp:141-157). Returns OC_NonFinite on a non-finite residual. */
static int record(oc_trace* tr, const oc_csr* A, const double* x, const double* b, const double* xstar,
                  int64_t epoch, int64_t updates, double t0, double* r_sq_out) {
    double r_sq, g_sq;
    oc_residuals(A, x, b, &r_sq, &g_sq);
    if (!isfinite(r_sq) || !isfinite(g_sq)) return OC_NonFinite;
    const int64_t k = tr->count++;
    if (k < tr->cap) {
        if (tr->epoch_index) tr->epoch_index[k] = epoch;
        if (tr->r_sq) tr->r_sq[k] = r_sq;
        if (tr->grad_sq) tr->grad_sq[k] = g_sq;
        if (tr->dist_sq) {
            double d = -1.0;
            if (xstar) {
                d = 0.0;
                for (int64_t j = 0; j < A->n; ++j) {
                    const double e = x[j] - xstar[j];
                    d += e * e;
                }
            }
            tr->dist_sq[k] = d;
        }
        if (tr->wall) tr->wall[k] = now_s() - t0;
        if (tr->updates) tr->updates[k] = updates;
    }
    *r_sq_out = r_sq;
    return OC_OK;
}

/* ref/src/kaczmarz.cpp:128-227 (rk_solve). sampling: 0 uniform,
 * 1 norm_proportional, 2 shuffle (kaczmarz.hpp:89-93). */
int oc_rk_solve(const oc_csr* A, const double* b, const double* x0, int64_t max_epochs, double target,
                uint64_t seed, int sampling, const double* xstar, oc_trace* tr) {
    const int64_t m = A->m, n = A->n;
    if (sampling == 0 && !A->normalized) return OC_NotNormalized;
    if (max_epochs < 0) return OC_InvalidArgument;
    oc_mt64 g;
    oc_make_stream(&g, seed, 0);
    double* x = (double*)malloc((size_t)n * 8);
    memcpy(x, x0, (size_t)n * 8);
    oc_alias al = {0, NULL, NULL};
    int64_t* perm = NULL;
    if (sampling == 1) {
        double* w = (double*)malloc((size_t)m * 8);
        for (int64_t i = 0; i < m; ++i) w[i] = A->row_norm[i] * A->row_norm[i];
        int st = oc_alias_build(&al, w, m);
        free(w);
        if (st) {
            free(x);
            return st;
        }
    } else if (sampling == 2) {
        perm = (int64_t*)malloc((size_t)m * 8);
        for (int64_t i = 0; i < m; ++i) perm[i] = i;
    }
    tr->count = 0;
    const double t0 = now_s();
    double r_sq;
    int st = record(tr, A, x, b, xstar, 0, 0, t0, &r_sq);
    for (int64_t e = 1; st == OC_OK && e <= max_epochs && r_sq > target; ++e) {
        if (sampling == 2) oc_shuffle_i64(perm, m, &g);
        for (int64_t q = 0; q < m; ++q) {
            int64_t i;
            if (sampling == 0)
                i = (int64_t)oc_uniform_below(&g, (uint64_t)m);
            else if (sampling == 1)
                i = alias_sample(&al, &g);
            else
                i = perm[q];
            const double res = stale_residual(A, x, b, i);
            apply_row(A, i, row_coef(A, i, 1.0, res), x);
        }
        st = record(tr, A, x, b, xstar, e, e * m, t0, &r_sq);
    }
    if (tr->final_x) memcpy(tr->final_x, x, (size_t)n * 8);
    free(x);
    free(perm);
    if (sampling == 1) alias_free(&al);
    return st;
}

/* ref/src/parallel.cpp:56-80 (validate_config) + :111-210 (solve_single):
 * the threads == 1 path of solve_parallel. variant: 0 single_component,
 * 1 full_row; sampling: 0 with_replacement, 1 slice_shuffle. */
int oc_solve_single(const oc_csr* A, const double* b, const double* x0, double gamma, int64_t epochs,
                    double target, int variant, int sampling, uint64_t seed, int64_t snapshot_interval,
                    const double* xstar, oc_trace* tr, oc_instrument* rep) {
    const int64_t m = A->m, n = A->n;
    if (!A->normalized) return OC_NotNormalized;
    if (!(gamma > 0.0)) return OC_InvalidGamma;
    if (epochs < 0 || snapshot_interval < 1) return OC_InvalidArgument;
    oc_mt64 g;
    oc_make_stream(&g, seed, 0);
    double* x = (double*)malloc((size_t)n * 8);
    memcpy(x, x0, (size_t)n * 8);
    int64_t* perm = NULL;
    if (sampling == 1) {
        perm = (int64_t*)malloc((size_t)m * 8);
        for (int64_t i = 0; i < m; ++i) perm[i] = i;
    }
    double* shadow = rep ? (double*)calloc((size_t)n, 8) : NULL;
    int64_t increments = 0;
    tr->count = 0;
    const double t0 = now_s();
    double r_sq;
    int st = record(tr, A, x, b, xstar, 0, 0, t0, &r_sq);
    int64_t e = 0;
    while (st == OC_OK && e < epochs && r_sq > target) {
        const int64_t span = snapshot_interval < epochs - e ? snapshot_interval : epochs - e;
        for (int64_t s = 0; s < span; ++s) {
            if (sampling == 1) oc_shuffle_i64(perm, m, &g);
            for (int64_t q = 0; q < m; ++q) {
                const int64_t i = sampling == 1 ? perm[q] : (int64_t)oc_uniform_below(&g, (uint64_t)m);
                const double res = stale_residual(A, x, b, i);
                if (variant == 1) {
                    const double c = row_coef(A, i, gamma, res);
                    apply_row(A, i, c, x);
                    if (shadow) {
                        for (int64_t k = A->row_ptr[i]; k < A->row_ptr[i + 1]; ++k)
                            shadow[A->col[k]] -= c * A->val[k];
                        increments += A->row_ptr[i + 1] - A->row_ptr[i];
                    }
                } else {
                    const int64_t theta = A->row_ptr[i + 1] - A->row_ptr[i];
                    const int64_t pick = (int64_t)oc_uniform_below(&g, (uint64_t)theta);
                    const int64_t slot = A->row_ptr[i] + pick;
                    const int64_t t = A->col[slot];
                    /* -gamma * theta * v * res, left to right (parallel.cpp:188-190) */
                    const double delta = -gamma * (double)theta * A->val[slot] * res;
                    x[t] += delta;
                    if (shadow) {
                        shadow[t] += delta;
                        ++increments;
                    }
                }
            }
        }
        e += span;
        st = record(tr, A, x, b, xstar, e, e * m, t0, &r_sq);
    }
    if (rep) {
        rep->row_updates = e * m;
        rep->increments = increments;
        double mx = 0.0;
        for (int64_t t = 0; t < n; ++t) {
            const double d = fabs(x[t] - x0[t] - shadow[t]);
            if (d > mx) mx = d;
        }
        rep->max_abs_error = mx;
        rep->tolerance = 1e-9 * (double)(increments > 1 ? increments : 1);
        rep->consistent = mx <= rep->tolerance;
    }
    if (tr->final_x) memcpy(tr->final_x, x, (size_t)n * 8);
    free(x);
    free(perm);
    free(shadow);
    return st;
}

/* ref/src/stats.cpp:15-50 (power_iteration_lambda_max, start vector from
 * make_stream(0x5ca1ab1e, 0) standard normals). */
int oc_power_iteration(const oc_csr* A, double tol, int64_t max_iters, double* lambda_out, int64_t* iters_out) {
    const int64_t n = A->n;
    oc_mt64 g;
    oc_make_stream(&g, 0x5ca1ab1eULL, 0);
    double* v = (double*)malloc((size_t)n * 8);
    double* av = (double*)malloc((size_t)A->m * 8);
    double* w = (double*)malloc((size_t)n * 8);
    for (int64_t k = 0; k < n; ++k) v[k] = oc_standard_normal(&g);
    double s = 0.0;
    for (int64_t k = 0; k < n; ++k) s += v[k] * v[k];
    double vn = sqrt(s);
    if (vn == 0.0) v[0] = 1.0, vn = 1.0;
    for (int64_t k = 0; k < n; ++k) v[k] /= vn;
    double lambda = 0.0;
    int st = OC_PowerIterationDiverged;
    for (int64_t it = 0; it < max_iters; ++it) {
        oc_multiply(A, v, av);
        oc_multiply_transpose(A, av, w);
        double ws = 0.0;
        for (int64_t k = 0; k < n; ++k) ws += w[k] * w[k];
        const double wn = sqrt(ws);
        if (wn == 0.0) {
            *lambda_out = 0.0;
            *iters_out = it + 1;
            st = OC_OK;
            break;
        }
        double next = 0.0;
        for (int64_t k = 0; k < n; ++k) next += v[k] * w[k];
        for (int64_t k = 0; k < n; ++k) v[k] = w[k] / wn;
        const double scale = fabs(next) > 1.0 ? fabs(next) : 1.0;
        if (it > 0 && fabs(next - lambda) <= tol * scale) {
            *lambda_out = next;
            *iters_out = it + 1;
            st = OC_OK;
            break;
        }
        lambda = next;
    }
    free(v);
    free(av);
    free(w);
    return st;
}

/* ref/src/stepsize.cpp:26-36 (psi) and :59-82 (corollary_params, feasibility
 * and rho/gamma only; the rate fields need lambda_min from a dense SVD). */
double oc_psi(double mu, double lambda_max, int64_t tau, double rho, int64_t m) {
    if (tau == 0) return mu;
    return mu + 2.0 * lambda_max * (double)tau * pow(rho, (double)tau) / (double)m;
}
void oc_corollary(int64_t m, int64_t mu, double lambda_max, int64_t tau, double* rho, double* psi,
                  double* gamma, int* feasible) {
    const double e = 2.71828182845904523536;
    const double lhs = 2.0 * e * lambda_max * (double)(tau + 1) / (double)m;
    *feasible = lhs <= 1.0;
    *rho = 1.0 + lhs;
    *psi = oc_psi((double)mu, lambda_max, tau, *rho, m);
    *gamma = *feasible ? 1.0 / *psi : 0.0;
}

/* ref/src/stats.cpp:52-130 (compute_stats, exact_spectral = false): delta,
 * theta/mu (row counts), CSC (ref csr.cpp:162-185, rows ascending per
 * column), nu, column norms, frob_sq / l_max in column order, alpha, and
 * l_res = max_t ||A^T (A e_t)|| with the reference's accumulation order
 * (rows of column t ascending, each row in CSR order) and its first-touch
 * order for the sum of squares; lambda_max by power iteration.
 * d[6] = {delta, alpha, lambda_max, frob_sq, l_max, l_res}. */
int oc_compute_stats(const oc_csr* A, double tol, int64_t max_iters, int64_t* mu_out, int64_t* nu_out, double* d,
                     int64_t* theta, int64_t* zero_col) {
    if (!A->normalized) return OC_NotNormalized;
    const int64_t m = A->m, n = A->n, nnz = A->nnz;
    double delta = (double)nnz / ((double)m * (double)n);
    int64_t mu = 0, nu = 0;
    for (int64_t i = 0; i < m; ++i) {
        const int64_t l = A->row_ptr[i + 1] - A->row_ptr[i];
        if (theta) theta[i] = l;
        if (l > mu) mu = l;
    }
    int64_t* cp = (int64_t*)calloc((size_t)n + 1, 8);
    int64_t* cur = (int64_t*)malloc((size_t)n * 8);
    int64_t* crow = (int64_t*)malloc((size_t)(nnz ? nnz : 1) * 8);
    double* cval = (double*)malloc((size_t)(nnz ? nnz : 1) * 8);
    double* cn = (double*)malloc((size_t)n * 8);
    for (int64_t k = 0; k < nnz; ++k) ++cp[A->col[k] + 1];
    for (int64_t j = 0; j < n; ++j) cp[j + 1] += cp[j];
    for (int64_t j = 0; j < n; ++j) cur[j] = cp[j];
    for (int64_t i = 0; i < m; ++i)
        for (int64_t k = A->row_ptr[i]; k < A->row_ptr[i + 1]; ++k) {
            const int64_t dst = cur[A->col[k]]++;
            crow[dst] = i;
            cval[dst] = A->val[k];
        }
    double frob = 0.0, l_max = 0.0, alpha = 0.0, l_res = 0.0;
    int st = OC_OK;
    for (int64_t t = 0; t < n && st == OC_OK; ++t) {
        const int64_t cnt = cp[t + 1] - cp[t];
        if (cnt == 0) {
            if (zero_col) *zero_col = t;
            st = OC_ZeroColumn;
            break;
        }
        if (cnt > nu) nu = cnt;
        double c = 0.0;
        for (int64_t k = cp[t]; k < cp[t + 1]; ++k) c += cval[k] * cval[k];
        cn[t] = sqrt(c);
        frob += c;
        if (l_max < c) l_max = c;
    }
    if (st == OC_OK) {
        for (int64_t i = 0; i < m; ++i) {
            const double th = (double)(A->row_ptr[i + 1] - A->row_ptr[i]);
            for (int64_t k = A->row_ptr[i]; k < A->row_ptr[i + 1]; ++k) {
                const double cand = th * fabs(A->val[k]) * cn[A->col[k]];
                if (alpha < cand) alpha = cand;
            }
        }
        double* acc = (double*)calloc((size_t)n, 8);
        int64_t cap = 1024, cnt_t = 0;
        int64_t* touched = (int64_t*)malloc((size_t)cap * 8);
        for (int64_t t = 0; t < n; ++t) {
            cnt_t = 0;
            for (int64_t k = cp[t]; k < cp[t + 1]; ++k) {
                const int64_t i = crow[k];
                const double av = cval[k];
                for (int64_t kk = A->row_ptr[i]; kk < A->row_ptr[i + 1]; ++kk) {
                    const int64_t u = A->col[kk];
                    if (acc[u] == 0.0) {
                        if (cnt_t == cap) {
                            cap *= 2;
                            touched = (int64_t*)realloc(touched, (size_t)cap * 8);
                        }
                        touched[cnt_t++] = u;
                    }
                    acc[u] += av * A->val[kk];
                }
            }
            double rs = 0.0;
            for (int64_t q = 0; q < cnt_t; ++q) {
                const double x = acc[touched[q]];
                rs += x * x;
                acc[touched[q]] = 0.0;
            }
            const double r = sqrt(rs);
            if (l_res < r) l_res = r;
        }
        free(acc);
        free(touched);
    }
    free(cp);
    free(cur);
    free(crow);
    free(cval);
    free(cn);
    if (st != OC_OK) return st;
    double lam = 0.0;
    int64_t iters = 0;
    st = oc_power_iteration(A, tol, max_iters, &lam, &iters);
    if (st != OC_OK) return st;
    *mu_out = mu;
    *nu_out = nu;
    d[0] = delta;
    d[1] = alpha;
    d[2] = lam;
    d[3] = frob;
    d[4] = l_max;
    d[5] = l_res;
    return OC_OK;
}

/* ------------------------------------------------------------- delay simulator */
/* ref/src/delay_sim.cpp:71-228 (simulate), :230-270 (monte_carlo_ratios),
 * :272-338 (rate_fit). Delay kinds: 0 fixed, 1 uniform_random, 2
 * max_staleness (delay_sim.hpp:17); variant 0 single_component, 1 full_row.
 * LiveResidual (delay_sim.cpp:27-60): r = Ax - b with a running r_sq, bumped
 * column by column (CSC order, rows ascending) and recomputed at every epoch. */
typedef struct {
    int64_t ev_cap, ev_count;
    int64_t *ev_j, *ev_i, *ev_t, *ev_k;
    double* ev_step;
    int64_t hist_cap, hist_rows;
    double* history;
    int64_t probe_cap, probe_count;
    int64_t* probe_iteration;
    double* probe_r_sq;
} oc_sim_extra;

typedef struct {
    int64_t *cp, *row;
    double* val;
    double *r, r_sq;
    const double* b;
} oc_live;

static void live_recompute(oc_live* L, const oc_csr* A, const double* x) {
    oc_multiply(A, x, L->r);
    L->r_sq = 0.0;
    for (int64_t i = 0; i < A->m; ++i) {
        L->r[i] -= L->b[i];
        L->r_sq += L->r[i] * L->r[i];
    }
}

static void live_bump(oc_live* L, int64_t t, double delta) {
    for (int64_t k = L->cp[t]; k < L->cp[t + 1]; ++k) {
        const int64_t i = L->row[k];
        L->r_sq -= L->r[i] * L->r[i];
        L->r[i] += L->val[k] * delta;
        L->r_sq += L->r[i] * L->r[i];
    }
}

static void live_init(oc_live* L, const oc_csr* A, const double* b, const double* x) {
    const int64_t n = A->n, nnz = A->nnz;
    L->cp = (int64_t*)calloc((size_t)n + 1, 8);
    L->row = (int64_t*)malloc((size_t)(nnz ? nnz : 1) * 8);
    L->val = (double*)malloc((size_t)(nnz ? nnz : 1) * 8);
    L->r = (double*)malloc((size_t)A->m * 8);
    L->b = b;
    int64_t* cur = (int64_t*)malloc((size_t)n * 8);
    for (int64_t k = 0; k < nnz; ++k) ++L->cp[A->col[k] + 1];
    for (int64_t j = 0; j < n; ++j) L->cp[j + 1] += L->cp[j];
    for (int64_t j = 0; j < n; ++j) cur[j] = L->cp[j];
    for (int64_t i = 0; i < A->m; ++i)
        for (int64_t k = A->row_ptr[i]; k < A->row_ptr[i + 1]; ++k) {
            const int64_t d = cur[A->col[k]]++;
            L->row[d] = i;
            L->val[d] = A->val[k];
        }
    free(cur);
    live_recompute(L, A, x);
}

static void live_free(oc_live* L) {
    free(L->cp);
    free(L->row);
    free(L->val);
    free(L->r);
}

int oc_simulate(const oc_csr* A, const double* b, const double* x0, double gamma, int64_t tau, int kind,
                int64_t iterations, uint64_t seed, int variant, int64_t probe_every, int probe_r_sq,
                int64_t max_events, oc_trace* tr, oc_sim_extra* ex) {
    const int64_t m = A->m, n = A->n;
    if (!A->normalized) return OC_NotNormalized;
    if (gamma < 0.0) return OC_InvalidGamma;
    if (iterations < 1 || tau < 0) return OC_InvalidArgument;
    const int64_t ring_len = tau + 1;
    oc_mt64 g;
    oc_make_stream(&g, seed, 0);
    double* x = (double*)malloc((size_t)n * 8);
    double* ring = (double*)malloc((size_t)(ring_len * n) * 8);
    memcpy(x, x0, (size_t)n * 8);
    memcpy(ring, x, (size_t)n * 8);
    const int probing = probe_every > 0 && probe_r_sq;
    oc_live live;
    int have_live = probing;
    if (have_live) live_init(&live, A, b, x);
    tr->count = 0;
    ex->ev_count = 0;
    ex->probe_count = 0;
#define OC_PROBE(jj)                                                              \
    do {                                                                          \
        const int64_t q_ = ex->probe_count++;                                     \
        if (q_ < ex->probe_cap) {                                                 \
            ex->probe_iteration[q_] = (jj);                                       \
            if (ex->probe_r_sq) ex->probe_r_sq[q_] = live.r_sq;                   \
        }                                                                         \
    } while (0)
    const double t0 = now_s();
    double rs;
    int st = record(tr, A, x, b, NULL, 0, 0, t0, &rs);
    if (st == OC_OK && probing) OC_PROBE(0);
    for (int64_t j = 0; j < iterations && st == OC_OK; ++j) {
        const int64_t i = (int64_t)oc_uniform_below(&g, (uint64_t)m);
        int64_t k;
        if (kind == 1) {
            const int64_t d = (int64_t)oc_uniform_below(&g, (uint64_t)(tau + 1));
            k = j - d > 0 ? j - d : 0;
        } else {
            k = j - tau > 0 ? j - tau : 0;
        }
        const double* xr = ring + (k % ring_len) * n;
        const double res = stale_residual(A, xr, b, i);
        int64_t ev_t;
        double ev_step;
        if (variant == 0) {
            const int64_t theta = A->row_ptr[i + 1] - A->row_ptr[i];
            const int64_t pick = (int64_t)oc_uniform_below(&g, (uint64_t)theta);
            const int64_t slot = A->row_ptr[i] + pick;
            const int64_t t = A->col[slot];
            const double delta = -gamma * (double)theta * A->val[slot] * res;
            x[t] += delta;
            if (have_live) live_bump(&live, t, delta);
            ev_t = t;
            ev_step = delta;
        } else {
            const double c = row_coef(A, i, gamma, res);
            apply_row(A, i, c, x);
            if (have_live)
                for (int64_t q = A->row_ptr[i]; q < A->row_ptr[i + 1]; ++q) live_bump(&live, A->col[q], -c * A->val[q]);
            ev_t = -1;
            ev_step = c;
        }
        memcpy(ring + ((j + 1) % ring_len) * n, x, (size_t)n * 8);
        if (ex->ev_count < max_events) {
            const int64_t e = ex->ev_count++;
            if (e < ex->ev_cap) {
                ex->ev_j[e] = j;
                ex->ev_i[e] = i;
                ex->ev_t[e] = ev_t;
                ex->ev_k[e] = k;
                ex->ev_step[e] = ev_step;
            }
        }
        const int64_t done = j + 1;
        if (done % m == 0) {
            st = record(tr, A, x, b, NULL, done / m, done, t0, &rs);
            if (st != OC_OK) break;
            if (have_live) live_recompute(&live, A, x);
        }
        if (probing && done % probe_every == 0) OC_PROBE(done);
    }
    if (st == OC_OK && iterations % m != 0) st = record(tr, A, x, b, NULL, iterations / m + 1, iterations, t0, &rs);
#undef OC_PROBE
    if (st == OC_OK) {
        const int64_t kept = ring_len < iterations + 1 ? ring_len : iterations + 1;
        ex->hist_rows = kept;
        int64_t row = 0;
        for (int64_t idx = iterations - kept + 1; idx <= iterations; ++idx, ++row)
            if (row < ex->hist_cap) memcpy(ex->history + row * n, ring + (idx % ring_len) * n, (size_t)n * 8);
        if (tr->final_x) memcpy(tr->final_x, x, (size_t)n * 8);
    }
    if (have_live) live_free(&live);
    free(x);
    free(ring);
    return st;
}

int oc_monte_carlo(const oc_csr* A, const double* b, const double* x0, double gamma, int64_t tau, int kind,
                   int64_t iterations, int64_t runs, uint64_t base_seed, int variant, double* mean_r_sq,
                   double* ratios) {
    if (runs < 100) return OC_InsufficientData;
    const int64_t K = iterations;
    double* pr = (double*)malloc((size_t)(K + 1) * 8);
    int64_t* pi = (int64_t*)malloc((size_t)(K + 1) * 8);
    for (int64_t j = 0; j <= K; ++j) mean_r_sq[j] = 0.0;
    int st = OC_OK;
    for (int64_t r = 0; r < runs && st == OC_OK; ++r) {
        oc_trace tr;
        memset(&tr, 0, sizeof tr);
        oc_sim_extra ex;
        memset(&ex, 0, sizeof ex);
        ex.probe_cap = K + 1;
        ex.probe_iteration = pi;
        ex.probe_r_sq = pr;
        st = oc_simulate(A, b, x0, gamma, tau, kind, iterations, base_seed + (uint64_t)r, variant, 1, 1, 0, &tr, &ex);
        if (st == OC_OK)
            for (int64_t j = 0; j <= K; ++j) mean_r_sq[j] += pr[j];
    }
    free(pr);
    free(pi);
    if (st != OC_OK) return st;
    const double inv = 1.0 / (double)runs;
    for (int64_t j = 0; j <= K; ++j) mean_r_sq[j] *= inv;
    for (int64_t j = 0; j < K; ++j) {
        const double a = mean_r_sq[j], c = mean_r_sq[j + 1];
        ratios[j] = a == 0.0 ? (c == 0.0 ? 1.0 : INFINITY) : c / a;
    }
    return OC_OK;
}

int oc_rate_fit(const double* y, int64_t n, double stride, double* slope, double* r2) {
    if (n < 20) return OC_InsufficientData;
    if (!(stride > 0.0)) return OC_InvalidArgument;
    double* ly = (double*)malloc((size_t)n * 8);
    for (int64_t k = 0; k < n; ++k) {
        if (!(y[k] > 0.0)) {
            free(ly);
            return OC_NonPositiveData;
        }
        ly[k] = log(y[k]);
    }
    const double shift = ly[0];
    for (int64_t k = 0; k < n; ++k) ly[k] -= shift;
    double sx = 0.0, sy = 0.0;
    for (int64_t k = 0; k < n; ++k) {
        sx += (double)k;
        sy += ly[k];
    }
    const double mx = sx / (double)n, my = sy / (double)n;
    double sxx = 0.0, sxy = 0.0, syy = 0.0;
    for (int64_t k = 0; k < n; ++k) {
        const double dx = (double)k - mx, dy = ly[k] - my;
        sxx += dx * dx;
        sxy += dx * dy;
        syy += dy * dy;
    }
    *slope = sxy / sxx / stride;
    *r2 = syy == 0.0 ? 1.0 : 1.0 - (syy - sxy * sxy / sxx) / syy;
    free(ly);
    return OC_OK;
}
