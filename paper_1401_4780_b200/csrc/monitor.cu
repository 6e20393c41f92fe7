// K3 — the residual / convergence monitor (replaces residuals,
// ref/src/csr.cpp:140-160, as called by the snapshot/record lambdas of
// ref/src/parallel.cpp:244-270 and ref/src/kaczmarz.cpp:178-199) and the
// coordinator's stop logic (parallel.cpp:388-408).
//
// Pass 1 (rows):    r_i = a_i^T x - b_i
// Pass 2 (columns): g_j = sum_i a_ij r_i over the CSC copy, rows ascending
//                   (the reference's multiply_transpose order, csr.cpp:80-92),
//                   plus (x_j - x*_j)^2 when an x_star oracle is given
// Finalize:         r_sq, grad_sq, dist_sq -> trace record, stop / NonFinite
//
// r_i and g_j are always formed in the reference's floating-point order
// (serial storage-order sums of rounded products), so they are bit-identical
// to ref residuals(). exact = 1 (deterministic path) also sums r^2, g^2 and
// (x - x*)^2 serially in index order, making every trace record
// bit-identical; exact = 0 (async path) sums them as fixed-order block
// partials: deterministic run to run, within a few ulps of the reference.
#include "kernels.h"

namespace ak {

constexpr int kMonThreads = 256;

template <class X>
__device__ __forceinline__ double ldx(const void* x, long long k) {
    return (double)__ldcg(static_cast<const X*>(x) + k);
}

// ---- pass 1: one warp per row. Lanes form the products v_k * x[c_k]
// (rounded multiplies); lane 0 adds them in storage order starting from 0.0,
// then subtracts b_i — exactly the reference's row_dot(i, x) - b_i
// (csr.cpp:65-70,146), so r is bit-identical in both monitor flavours.
// fast flavour: r^2 block partials (fixed order).
template <class V, class X>
__global__ void __launch_bounds__(kMonThreads) rows_kernel(MonitorArgs a) {
    if (a.st->stop) return;
    __shared__ double red[kMonThreads / 32];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const long long warps_total = (long long)gridDim.x * (kMonThreads / 32);
    double mine = 0.0;
    for (long long i = (long long)blockIdx.x * (kMonThreads / 32) + wib; i < a.L.m; i += warps_total) {
        const RowRef r = row_ref(a.L, i);
        const V* vals = rec_vals<V>(r);
        const int32_t* cols = rec_cols<V>(r);
        double s = 0.0;
        for (int c0 = 0; c0 < r.len; c0 += 32) {
            const int k = c0 + lane;
            double p = 0.0;
            if (k < r.len) p = __dmul_rn((double)__ldg(vals + k), ldx<X>(a.x, __ldg(cols + k)));
            const int lim = min(32, r.len - c0);
            for (int t = 0; t < lim; ++t) {
                const double pt = __shfl_sync(FULL, p, t);
                s = __dadd_rn(s, pt);
            }
        }
        const double ri = __dsub_rn(s, rec_b(r));
        if (lane == 0) a.r[i] = ri;
        mine += ri * ri;
    }
    if (a.exact) return;
    if (lane == 0) red[wib] = mine;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < kMonThreads / 32; ++w) t += red[w];
        a.part[blockIdx.x] = t;
    }
}

// ---- pass 2: one thread per column over the CSC copy (rows ascending).
// exact: g_j kept for the serial finalize; fast: g^2 and dist^2 block partials.
template <class V, class X>
__global__ void __launch_bounds__(kMonThreads) cols_kernel(MonitorArgs a, int nblocks_rows) {
    if (a.st->stop) return;
    __shared__ double red_g[kMonThreads], red_d[kMonThreads];
    const long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    double g2 = 0.0, d2 = 0.0;
    if (j < a.L.n) {
        const long long e0 = __ldg(a.csc.col_ptr + j), e1 = __ldg(a.csc.col_ptr + j + 1);
        const V* cv = static_cast<const V*>(a.csc.val);
        double g = 0.0;
        for (long long e = e0; e < e1; ++e) g = __dadd_rn(g, __dmul_rn((double)__ldg(cv + e), a.r[__ldg(a.csc.row + e)]));
        if (a.exact) {
            a.g[j] = g;
        } else {
            g2 = g * g;
            if (a.x_star) {
                const double d = ldx<X>(a.x, j) - a.x_star[j];
                d2 = d * d;
            }
        }
    }
    if (a.exact) return;
    red_g[threadIdx.x] = g2;
    red_d[threadIdx.x] = d2;
    __syncthreads();
    for (int o = kMonThreads / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o) {
            red_g[threadIdx.x] += red_g[threadIdx.x + o];
            red_d[threadIdx.x] += red_d[threadIdx.x + o];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        a.part[nblocks_rows + blockIdx.x] = red_g[0];
        a.part[nblocks_rows + gridDim.x + blockIdx.x] = red_d[0];
    }
}

__device__ void commit_record(const MonitorArgs& a, double r_sq, double g_sq, double d_sq) {
    DevState* st = a.st;
    if (a.advance) {
        const long long sp = chunk_span(st);
        st->epoch += sp;
        st->updates += sp * a.m_rows;
    }
    if (!isfinite(r_sq) || !isfinite(g_sq)) {
        st->status = 8;  // ASYRK_E_NonFinite
        st->stop = 1;
    } else {
        const long long k = st->nrec;
        if (k < a.rec_cap) {
            DevRecord rc;
            rc.epoch = st->epoch;
            rc.updates = st->updates;
            rc.r_sq = r_sq;
            rc.grad_sq = g_sq;
            rc.dist_sq = a.x_star ? d_sq : -1.0;
            rc.t_ns = globaltimer_ns() - st->t0_ns;
            a.rec[k] = rc;
        }
        st->nrec = k + 1;
        if (r_sq <= st->target || st->epoch >= st->epochs_cap) st->stop = 1;
    }
    if (st->stop && a.host_flag) {
        *reinterpret_cast<volatile int*>(a.host_flag) = 1;
        __threadfence_system();
    }
}

// ---- finalize, exact: serial sums in the reference's order (residuals
// csr.cpp:147-158, dist oracle parallel.cpp:82-92). Lanes square 32 values at
// a time; lane 0 accumulates them in index order.
__device__ __forceinline__ double serial_sumsq(const double* v, const double* w, long long n, int lane) {
    double s = 0.0;
    for (long long c0 = 0; c0 < n; c0 += 32) {
        const long long k = c0 + lane;
        double q = 0.0;
        if (k < n) {
            const double d = w ? __dsub_rn(v[k], w[k]) : v[k];
            q = __dmul_rn(d, d);
        }
        const int lim = (int)min(32ll, n - c0);
        for (int t = 0; t < lim; ++t) s = __dadd_rn(s, __shfl_sync(FULL, q, t));
    }
    return s;
}

template <class X>
__global__ void finalize_exact_kernel(MonitorArgs a) {
    if (a.st->stop) return;
    const int lane = threadIdx.x & 31;
    const double rs = serial_sumsq(a.r, nullptr, a.L.m, lane);
    const double gs = serial_sumsq(a.g, nullptr, a.L.n, lane);
    double ds = 0.0;
    if (a.x_star) ds = serial_sumsq(static_cast<const double*>(a.x), a.x_star, a.L.n, lane);  // exact mode is fp64
    if (lane == 0) commit_record(a, rs, gs, ds);
}

// ---- finalize, fast: fixed-order sum of the block partials (one block)
__global__ void __launch_bounds__(kMonThreads) finalize_fast_kernel(MonitorArgs a, int nb_rows, int nb_cols) {
    if (a.st->stop) return;
    __shared__ double red[3][kMonThreads];
    double s[3] = {0.0, 0.0, 0.0};
    for (int k = threadIdx.x; k < nb_rows; k += kMonThreads) s[0] += a.part[k];
    for (int k = threadIdx.x; k < nb_cols; k += kMonThreads) {
        s[1] += a.part[nb_rows + k];
        s[2] += a.part[nb_rows + nb_cols + k];
    }
    for (int c = 0; c < 3; ++c) red[c][threadIdx.x] = s[c];
    __syncthreads();
    for (int o = kMonThreads / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o)
            for (int c = 0; c < 3; ++c) red[c][threadIdx.x] += red[c][threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) commit_record(a, red[0][0], red[1][0], red[2][0]);
}

static int sm_count() {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    }
    return sms;
}

int monitor_row_blocks(long long m) {
    const long long want = (m + (kMonThreads / 32) - 1) / (kMonThreads / 32);
    const long long cap = (long long)sm_count() * 8;
    return (int)(want < cap ? want : cap);
}
int monitor_col_blocks(long long n) { return (int)((n + kMonThreads - 1) / kMonThreads); }

template <class V, class X>
static void monitor_impl(const MonitorArgs& a, cudaStream_t s) {
    const int nbr = monitor_row_blocks(a.L.m);
    const int nbc = monitor_col_blocks(a.L.n);
    rows_kernel<V, X><<<nbr, kMonThreads, 0, s>>>(a);
    cols_kernel<V, X><<<nbc, kMonThreads, 0, s>>>(a, nbr);
    if (a.exact)
        finalize_exact_kernel<X><<<1, 32, 0, s>>>(a);
    else
        finalize_fast_kernel<<<1, kMonThreads, 0, s>>>(a, nbr, nbc);
}

void launch_monitor(const MonitorArgs& a, int precision, cudaStream_t s) {
    switch (precision) {
        case P_F32: monitor_impl<float, float>(a, s); break;
        case P_F32X64: monitor_impl<float, double>(a, s); break;
        default: monitor_impl<double, double>(a, s); break;
    }
}

// ---- power iteration pieces (ref/src/stats.cpp:15-50): y = A v and
// w = A^T y in the reference's order, fixed-order tree dots.
template <class V>
__global__ void __launch_bounds__(kMonThreads) spmv_rows_kernel(Layout L, const double* v, double* out) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= L.m) return;
    const RowRef r = row_ref(L, i);
    const V* vals = rec_vals<V>(r);
    const int32_t* cols = rec_cols<V>(r);
    double s = 0.0;
    for (int k = 0; k < r.len; ++k) s = __dadd_rn(s, __dmul_rn((double)__ldg(vals + k), v[__ldg(cols + k)]));
    out[i] = s;
}
template <class V>
__global__ void __launch_bounds__(kMonThreads) spmv_cols_kernel(CscDev C, long long n, const double* r, double* out) {
    const long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    const V* cv = static_cast<const V*>(C.val);
    double g = 0.0;
    for (long long e = C.col_ptr[j]; e < C.col_ptr[j + 1]; ++e) g = __dadd_rn(g, __dmul_rn((double)cv[e], r[C.row[e]]));
    out[j] = g;
}

void launch_spmv_rows(const Layout& L, int precision, const double* v, double* out, cudaStream_t s) {
    const unsigned nb = (unsigned)((L.m + kMonThreads - 1) / kMonThreads);
    if (precision == P_F64)
        spmv_rows_kernel<double><<<nb, kMonThreads, 0, s>>>(L, v, out);
    else
        spmv_rows_kernel<float><<<nb, kMonThreads, 0, s>>>(L, v, out);
}
void launch_spmv_cols(const CscDev& C, int precision, long long n, const double* r, double* out, cudaStream_t s) {
    const unsigned nb = (unsigned)((n + kMonThreads - 1) / kMonThreads);
    if (precision == P_F64)
        spmv_cols_kernel<double><<<nb, kMonThreads, 0, s>>>(C, n, r, out);
    else
        spmv_cols_kernel<float><<<nb, kMonThreads, 0, s>>>(C, n, r, out);
}

__global__ void __launch_bounds__(kMonThreads) dot_part_kernel(const double* a, const double* b, long long n,
                                                              double* part) {
    __shared__ double red[kMonThreads];
    double s = 0.0;
    for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (long long)gridDim.x * blockDim.x)
        s += a[k] * b[k];
    red[threadIdx.x] = s;
    __syncthreads();
    for (int o = kMonThreads / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) part[blockIdx.x] = red[0];
}
__global__ void __launch_bounds__(kMonThreads) sum_part_kernel(const double* part, int np, double* out) {
    __shared__ double red[kMonThreads];
    double s = 0.0;
    for (int k = threadIdx.x; k < np; k += kMonThreads) s += part[k];
    red[threadIdx.x] = s;
    __syncthreads();
    for (int o = kMonThreads / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = red[0];
}
void launch_dot(const double* a, const double* b, long long n, double* scratch, double* out, cudaStream_t s) {
    long long want = (n + kMonThreads - 1) / kMonThreads;
    const int nb = (int)(want < 4 * sm_count() ? (want > 0 ? want : 1) : 4 * sm_count());
    dot_part_kernel<<<nb, kMonThreads, 0, s>>>(a, b, n, scratch);
    sum_part_kernel<<<1, kMonThreads, 0, s>>>(scratch, nb, out);
}
// v = w / sqrt(ww)  (stats.cpp:37,41)
__global__ void power_update_kernel(double* v, const double* w, const double* ww, long long n) {
    const double wn = sqrt(*ww);
    for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (long long)gridDim.x * blockDim.x)
        v[k] = w[k] / wn;
}
void launch_power_update(double* v, const double* w, const double* ww, long long n, cudaStream_t s) {
    power_update_kernel<<<4 * sm_count(), kMonThreads, 0, s>>>(v, w, ww, n);
}

}  // namespace ak
